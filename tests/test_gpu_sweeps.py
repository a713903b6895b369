"""Reference test strategies that need the whole device path (C ABI, GPU):

* every-byte truncation sweep (reference tests/test_container.py:59-63) with the reference's own
  CorruptStream message and offset for each cut (tests/golden/truncation.json);
* config 5 at full size (100x500x500, 1% of blocks flipped, three stages) against the
  reference's archive / output / report hashes (tools/make_golden.py --large).
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2010_03144_b200 as F
from oracle import oracle as O
from tests.golden_util import GOLDEN, load, manifest, sha

pytestmark = pytest.mark.gpu


def _truncation():
    with open(os.path.join(GOLDEN, "truncation.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("src", sorted(_truncation()))
def test_truncation_sweep_every_byte(src):
    t = _truncation()[src]
    arch = load(src)["archive"].tobytes()
    assert len(arch) == t["len"]
    for cut, ix in enumerate(t["index"]):
        cls, msg = t["messages"][ix]
        with pytest.raises(F.FtlzError) as ei:
            F.parse(arch[:cut])
        assert (type(ei.value).__name__, str(ei.value)) == (cls, msg), cut
    # the whole archive parses and decompresses to the reference output
    out, rep = F.decompress(F.parse(arch))
    z = load(src)
    np.testing.assert_array_equal(out.values.view(np.uint32), z["output"].view(np.uint32))


def _h(obj) -> str:
    return hashlib.sha256(json.dumps(obj).encode()).hexdigest()


@pytest.fixture(scope="module")
def c5_field():
    from tools import synth

    x = synth.field("c5")
    vols = synth.block_volumes(x.shape, 10)
    return x, synth.fault_plan(len(vols), vols)


@pytest.mark.parametrize("target", ["input", "bins", "decomp"])
def test_c5_full_size_matches_reference(c5_field, target):
    """BASELINE config 5: 250 single-bit flips (1% of 25,000 blocks, bits 0..31) at one stage;
    archive, output, corrected / re-executed lists and statuses equal the reference's."""
    x, plan = c5_field
    ent = manifest()["large"]["c5"]
    assert sha(x) == ent["input_sha256"]
    assert _h(plan) == ent["plan_sha256"] and len(plan) == ent["n_faults"]
    want = ent[target]
    faults = [(target, b, e, t) for b, e, t in plan]
    stream, rc = F.compress(F.Field.from_array(x), F.ErrorBound(ent["mode"], ent["value"]), F.FtConfig(),
                            faults=faults if target != "decomp" else None)
    data = F.serialize(stream)
    assert len(data) == want["archive_len"]
    assert sha(np.frombuffer(data, np.uint8)) == want["archive_sha256"]
    r = rc.to_dict()
    assert r["status"] == want["status_c"]
    assert len(r["input_corrected"]) == want["n_input_corrected"]
    assert _h(r["input_corrected"]) == want["input_corrected_sha256"]
    assert len(r["bins_corrected"]) == want["n_bins_corrected"]
    assert _h(r["bins_corrected"]) == want["bins_corrected_sha256"]
    out, rd = F.decompress(F.parse(data), faults=faults if target == "decomp" else None)
    d = rd.to_dict()
    assert d["status"] == want["status_d"]
    assert len(d["decomp_block_reexecuted"]) == want["n_reexecuted"]
    assert _h(d["decomp_block_reexecuted"]) == want["reexecuted_sha256"]
    assert out is not None and sha(out.values) == want["output_sha256"]


# Seeded random cases through every kernel variant the library picks by geometry (2-D and 3-D
# fields, ragged blocks, edges 2..24, the warp-per-block or lane-per-block decoder, Lorenzo blocks
# fused into the regression kernel or not), random flags, bounds and faults: archive, report
# lists and reconstruction equal to the oracle's.
def _fuzz_case(seed):
    rng = np.random.default_rng(seed)
    if rng.random() < 0.3:
        dims = (1, int(rng.integers(12, 300)), int(rng.integers(12, 300)))
    else:
        dims = tuple(int(v) for v in rng.integers(8, 90, size=3))
    edge = int(rng.choice([10, 10, 10, 4, 6, 8, 12, 16, 24, 2, 3]))
    i, j, k = np.meshgrid(*[np.arange(d, dtype=np.float64) for d in dims], indexing="ij")
    kind = rng.integers(0, 3)
    if kind == 0:
        x = np.sin(0.07 * i * rng.uniform(0.5, 2)) * np.cos(0.05 * j) + 0.02 * k + rng.normal(0, 1e-3, dims)
    elif kind == 1:
        x = rng.standard_normal(dims) * rng.uniform(0.1, 10)
    else:
        x = np.exp(rng.standard_normal(dims))
    x = x.astype(np.float32)
    mode = "value_range_relative" if rng.random() < 0.7 else "absolute"
    value = float(10.0 ** rng.uniform(-5, -1.5))
    cfg = dict(block_edge=edge, protect_input=bool(rng.random() < 0.8), protect_bins=bool(rng.random() < 0.8),
               duplicate_eval=bool(rng.random() < 0.8), store_sum_dc=bool(rng.random() < 0.9))
    nb = 1
    for d in dims:
        nb *= -(-d // edge)
    vol = min(edge, dims[0]) * min(edge, dims[1]) * min(edge, dims[2])   # first block: full extent
    faults = []
    if rng.random() < 0.6:
        for _ in range(int(rng.integers(1, 6))):
            t = str(rng.choice(["input", "bins", "dup_predict", "dup_reconstruct"]))
            faults.append((t, 0, int(rng.integers(0, vol)), int(rng.integers(0, 192 if t.startswith("dup") else 32))))
    dfaults = [("decomp", 0, int(rng.integers(0, vol)), int(rng.integers(0, 32)))] if rng.random() < 0.5 else []
    return x, mode, value, cfg, faults, dfaults


@pytest.mark.parametrize("seed", range(64))
def test_random_cases_against_oracle(seed):
    x, mode, value, cfg, faults, dfaults = _fuzz_case(1000 + seed)
    try:
        want, wrep = O.compress(x, mode, value, cfg, faults=faults, threads=4)
    except O.OracleError as e:
        with pytest.raises(F.FtlzError) as ei:
            F.compress(F.Field.from_array(x), F.ErrorBound(mode, value), F.FtConfig(**cfg), faults=faults)
        assert type(ei.value).__name__ == e.cls
        assert str(ei.value) == str(e)
        return
    stream, rep = F.compress(F.Field.from_array(x), F.ErrorBound(mode, value), F.FtConfig(**cfg), faults=faults)
    data = F.serialize(stream)
    assert data == want
    rd = rep.to_dict()
    for k in ("input_corrected", "bins_corrected", "dup_mismatch_resolved"):
        assert rd[k] == wrep[k], k
    out, drep = F.decompress(F.parse(data), faults=dfaults)
    ro, rr = O.decompress(want, faults=dfaults, threads=4)
    assert drep.to_dict()["decomp_block_reexecuted"] == rr["decomp_block_reexecuted"]
    if ro is None:
        assert out is None
    else:
        np.testing.assert_array_equal(out.values.view(np.uint32), ro.view(np.uint32))


# Decompressed-data faults on several blocks of a payload-damaged archive: the re-execution
# kernels queued behind the decode are sized from the faulted blocks, the damage adds
# mismatching (or undecodable) blocks the host did not count; status, detail, re-executed list
# and output equal to the oracle's.
@pytest.mark.parametrize("seed", range(12))
def test_decomp_faults_on_damaged_payload(seed):
    rng = np.random.default_rng(7000 + seed)
    dims = (30, 40, 50) if seed % 3 else (1, 60, 70)
    i, j, k = np.meshgrid(*[np.arange(d, dtype=np.float64) for d in dims], indexing="ij")
    x = (np.sin(0.11 * i) * np.cos(0.07 * j) + 0.03 * k + rng.normal(0, 2e-3, dims)).astype(np.float32)
    stream, _ = F.compress(F.Field.from_array(x), F.ErrorBound("absolute", 1e-3))
    data = bytearray(F.serialize(stream))
    grid = F.BlockGrid(dims, 10)
    nb = grid.n_blocks
    blocks = sorted(set(int(b) for b in rng.integers(0, nb, size=int(rng.integers(1, 8)))))
    dfaults = []
    for b in blocks:
        vol = int(np.prod(grid.spec(b).extent))
        for _ in range(int(rng.integers(1, 3))):
            dfaults.append(("decomp", b, int(rng.integers(0, vol)), int(rng.integers(0, 32))))
    if seed % 4 != 3:   # damage a payload bit (seed % 4 == 3: faults only, several blocks)
        off = data.find(stream.payload[:16])
        assert off > 0
        pos = off + int(rng.integers(0, len(stream.payload)))
        data[pos] ^= 1 << int(rng.integers(0, 8))
    data = bytes(data)
    ro, rr = O.decompress(data, faults=dfaults, threads=4)
    out, rep = F.decompress(F.parse(data), faults=dfaults)
    d = rep.to_dict()
    assert d["status"] == rr["status"]
    assert d["detail"] == rr["detail"]
    assert d["decomp_block_reexecuted"] == rr["decomp_block_reexecuted"]
    if ro is None:
        assert out is None
    else:
        np.testing.assert_array_equal(out.values.view(np.uint32), ro.view(np.uint32))
        got = F.decompress_bytes(data, faults=dfaults)
        np.testing.assert_array_equal(got.view(np.uint32).ravel(), ro.view(np.uint32).ravel())
