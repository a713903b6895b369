"""Parity of the B200 path (through the C ABI) with the reference, on the GPU.

Golden fixtures come from the reference package itself (tools/make_golden.py); seeded cases
beyond them are checked against the CPU oracle (oracle/ftlz_oracle.c), which is pinned to the
reference by tests/test_oracle_golden.py.  Everything integer/byte-valued must be bit-exact:
archives, reconstructed float32 words, unpredictable words, FtReport lists, error texts.
"""

import dataclasses

import numpy as np
import pytest

import paper_2010_03144_b200 as F
from oracle import oracle as O
from tests.golden_util import faults_of, load, manifest, override_of, sha

pytestmark = pytest.mark.gpu

M = manifest()


def _cfg(d):
    d = dict(d)
    cap = d.pop("bin_capacity", None)
    if cap is not None:
        d["quant"] = F.QuantConfig(cap)
    return F.FtConfig(**d)


@pytest.mark.parametrize("name", sorted(M["cases"]))
def test_golden_compress_decompress(name):
    e = M["cases"][name]
    z = load(name)
    x = z["input"]
    faults = faults_of(e)
    cfg = _cfg(e["cfg"])
    eb = F.ErrorBound(e["mode"], e["value"])
    if "compress_error" in e:
        with pytest.raises(F.FtlzError) as ei:
            F.compress(F.Field.from_array(x), eb, cfg, predictor_override=override_of(e), faults=faults)
        assert type(ei.value).__name__ == e["compress_error"]["cls"]
        assert str(ei.value) == e["compress_error"]["msg"]
        return
    stream, rep = F.compress(F.Field.from_array(x), eb, cfg, predictor_override=override_of(e), faults=faults)
    data = F.serialize(stream)
    want = z["archive"].tobytes()
    if data != want:
        d = np.flatnonzero(np.frombuffer(data[: len(want)], np.uint8) != np.frombuffer(want[: len(data)], np.uint8))
        pytest.fail(f"archive differs: len {len(data)} vs {len(want)}, first diff at {d[:5]}")
    rd = rep.to_dict()
    for k in ("status", "input_corrected", "bins_corrected", "dup_mismatch_resolved", "detail"):
        assert rd[k] == e["compress_report"][k], k
    out, drep = F.decompress(F.parse(data), faults=faults)
    dd = drep.to_dict()
    for k in ("status", "decomp_block_reexecuted", "detail"):
        assert dd[k] == e["decompress_report"][k], k
    if "output_sha256" in e:
        assert out is not None
        np.testing.assert_array_equal(out.values.view(np.uint32), z["output"].view(np.uint32))
    else:
        assert out is None


def _corrupt_cases():
    for src, cases in sorted(M["corrupt"].items()):
        for name in sorted(cases):
            yield src, name


@pytest.mark.parametrize("src,name", list(_corrupt_cases()))
def test_golden_parse_and_sdc(src, name):
    e = M["corrupt"][src][name]
    blob = load(f"corrupt_{src}")[name].tobytes()
    if "error" in e:
        with pytest.raises(F.FtlzError) as ei:
            F.decompress(F.parse(blob))
        assert type(ei.value).__name__ == e["error"]["cls"]
        assert str(ei.value) == e["error"]["msg"]
        return
    out, rep = F.decompress(F.parse(blob))
    d = rep.to_dict()
    for k in ("status", "decomp_block_reexecuted", "detail"):
        assert d[k] == e["decompress_report"][k], k
    assert (None if out is None else sha(out.values)) == e["output_sha256"]


def _seeded(kind, dims, seed):
    rng = np.random.default_rng(seed)
    if kind == "noise":
        return rng.standard_normal(dims).astype(np.float32)
    if kind == "smooth":
        i, j, k = np.meshgrid(*[np.arange(d, dtype=np.float64) for d in dims], indexing="ij")
        return (np.sin(0.21 * i + 0.3) * np.cos(0.17 * j) + 0.05 * k
                + 1e-3 * rng.standard_normal(dims)).astype(np.float32)
    if kind == "lognormal":
        return np.exp(2.0 * rng.standard_normal(dims)).astype(np.float32)
    raise ValueError(kind)


ORACLE_CASES = [
    ("smooth", (37, 41, 29), 10, "value_range_relative", 1e-3),
    ("smooth", (64, 70, 90), 10, "value_range_relative", 1e-4),
    ("noise", (33, 20, 51), 10, "absolute", 1e-2),
    ("lognormal", (40, 40, 40), 10, "value_range_relative", 1e-3),
    ("smooth", (1, 180, 360), 10, "value_range_relative", 1e-4),
    ("smooth", (50, 50, 50), 8, "absolute", 1e-3),
    ("noise", (17, 23, 29), 5, "absolute", 1e-5),
    ("smooth", (30, 31, 32), 3, "value_range_relative", 1e-3),
    ("smooth", (48, 48, 48), 16, "value_range_relative", 1e-3),
]


@pytest.mark.parametrize("kind,dims,edge,mode,value", ORACLE_CASES)
def test_seeded_against_oracle(kind, dims, edge, mode, value):
    x = _seeded(kind, dims, seed=hash((kind, dims, edge)) % 2**31)
    cfg = {"block_edge": edge}
    want, wrep = O.compress(x, mode, value, cfg, threads=4)
    got = F.compress_bytes(x, mode, value, F.FtConfig(block_edge=edge))
    assert got == want
    out = F.decompress_bytes(got)
    ref, _ = O.decompress(want, threads=4)
    np.testing.assert_array_equal(out.view(np.uint32), ref.view(np.uint32))
    # error bound holds on every point (unpredictables are stored losslessly)
    ebv = wrep["eb"]
    assert np.max(np.abs(out.astype(np.float64) - x.astype(np.float64))) <= ebv


@pytest.mark.parametrize("cfg", [
    dict(protect_input=False, protect_bins=False, duplicate_eval=False, store_sum_dc=False),
    dict(protect_input=True, protect_bins=False, duplicate_eval=False, store_sum_dc=True),
    dict(protect_input=False, protect_bins=True, duplicate_eval=True, store_sum_dc=False),
])
def test_config_flags_against_oracle(cfg):
    x = _seeded("smooth", (40, 33, 27), seed=5)
    want, _ = O.compress(x, "absolute", 1e-3, cfg)
    got = F.compress_bytes(x, "absolute", 1e-3, F.FtConfig(**cfg))
    assert got == want


def test_payload_flip_isolation_and_sdc():
    # a flipped payload bit is detected: SDC reported, output withheld (test_pipeline.py:289-297)
    x = _seeded("noise", (20, 20, 20), seed=3)
    stream, _ = F.compress(F.Field.from_array(x), F.ErrorBound.absolute(1e-3))
    corrupted = bytearray(stream.payload)
    corrupted[len(corrupted) // 2] ^= 0xFF
    s2 = dataclasses.replace(stream, payload=bytes(corrupted))
    out, rep = F.decompress(s2)
    want, wrep = O.decompress(F.serialize(s2))
    assert out is None and rep.status == "sdc_in_compression"
    assert rep.detail == wrep["detail"]


def test_replace_roundtrip_equals_original():
    x = _seeded("smooth", (21, 22, 23), seed=8)
    stream, _ = F.compress(F.Field.from_array(x), F.ErrorBound.absolute(1e-3), F.FtConfig(block_edge=4))
    s2 = dataclasses.replace(stream)
    assert F.serialize(s2) == F.serialize(stream)
    assert F.parse(F.serialize(stream)) == stream


def test_thread_argument_is_deterministic():
    x = _seeded("smooth", (22, 18, 14), seed=18)
    a, _ = F.compress(F.Field.from_array(x), F.ErrorBound.absolute(1e-3), threads=1)
    b, _ = F.compress(F.Field.from_array(x), F.ErrorBound.absolute(1e-3), threads=8)
    assert F.serialize(a) == F.serialize(b)


# ---- BASELINE.json configurations at full size: archive and output hashes of the reference's
#      own runs (tools/make_golden.py --large), generated from the same seeded fields
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c4", "c2", "c2_1e-4", "c3"])
def test_full_size_configs_match_reference_hashes(name):
    from tools import synth

    ent = manifest()["large"][name]
    x = synth.field(name)
    assert sha(x) == ent["input_sha256"]
    mode, value = synth.CONFIGS[name]["eb"]
    data = F.compress_bytes(x, mode, value)
    assert len(data) == ent["archive_len"]
    assert sha(np.frombuffer(data, np.uint8)) == ent["archive_sha256"]
    y = F.decompress_bytes(data)
    assert sha(y) == ent["output_sha256"]


@pytest.mark.gpu
def test_slab_overlapped_decompress_with_reexecution_on_c3():
    """Large fields decode in slabs whose output downloads overlap the decode; decompressed-data
    faults force re-execution afterwards, and the result must still be the fault-free output
    (pipeline.py:708-723)."""
    from tools import synth
    x = synth.field("c3")
    data = F.compress_bytes(x, "value_range_relative", 1e-3)
    clean = F.decompress_bytes(data)
    stream = F.parse(data)
    faults = [("decomp", 5, 17, 30), ("decomp", 70000, 999, 22), ("decomp", 140607, 3, 31)]
    out, rep = F.decompress(stream, faults=faults)
    rd = rep.to_dict()
    assert rd["status"] == "corrected" and rd["decomp_block_reexecuted"] == [5, 70000, 140607]
    np.testing.assert_array_equal(out.values.view(np.uint32), clean.view(np.uint32))


def test_reused_context_buffers_do_not_leak_into_archives():
    """The device archive and workspace are reused across calls, and k_enc_pack merges the
    words it shares with neighbouring blocks (or lanes) with atomicOr into words k_enc_scan /
    k_enc_pack zeroed first.  Alternate unlike fields of one shape (noise with unstaged blocks,
    a smooth field, constant) through the same context: every archive must equal the oracle's,
    whatever the previous call left in the buffers."""
    dims = (48, 40, 36)
    rng = np.random.default_rng(17)
    noise = rng.standard_normal(dims).astype(np.float32)
    smooth = _seeded("smooth", dims, seed=3)
    const = np.full(dims, 2.5, np.float32)
    cases = [(noise, "absolute", 1e-5), (smooth, "value_range_relative", 1e-3), (noise, "absolute", 1e-2),
             (const, "absolute", 1e-3), (noise, "absolute", 1e-5), (smooth, "absolute", 1e-6)]
    for x, mode, v in cases + cases[::-1]:
        want, _ = O.compress(x, mode, v, threads=4)
        got = F.compress_bytes(x, mode, v)
        assert got == want
        out = F.decompress_bytes(got)
        ref, _ = O.decompress(want, threads=4)
        np.testing.assert_array_equal(out.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("ebv", [3e-3, 1e-3, 4e-4, 1.5e-4, 6e-5, 2.5e-5])
def test_alphabet_sizes_sort_and_merge_paths(ebv):
    """Noise at falling bounds grows the alphabet from hundreds to tens of thousands of symbols:
    the codebook's bitonic sorts cross every register / shared-memory stage split (and the
    plain network past 8,192 keys), the two-queue merge runs in shared and in global memory,
    and the decoder's long-code path is taken.  Archives and outputs equal the oracle's."""
    x = _seeded("noise", (64, 60, 56), seed=23)
    want, wrep = O.compress(x, "absolute", ebv, threads=4)
    got = F.compress_bytes(x, "absolute", ebv)
    assert got == want
    out = F.decompress_bytes(got)
    ref, _ = O.decompress(want, threads=4)
    np.testing.assert_array_equal(out.view(np.uint32), ref.view(np.uint32))


def test_parse_reuse_is_invalidated_by_another_upload():
    """parse(a) leaves a's device copy for decompress(s_a) to reuse; any other archive uploaded
    in between (decompress_bytes(b), decompress of another stream) must invalidate that, so
    decompress(s_a) still returns a's data (stale-archive reuse)."""
    xa = _seeded("smooth", (30, 20, 25), seed=1)
    xb = _seeded("smooth", (30, 20, 25), seed=2)
    a = F.compress_bytes(xa, "absolute", 1e-3)
    b = F.compress_bytes(xb, "absolute", 1e-3)
    ya = F.decompress_bytes(a)
    yb = F.decompress_bytes(b)
    sa = F.parse(a)
    F.decompress_bytes(b)
    out, _ = F.decompress(sa)
    np.testing.assert_array_equal(out.values.view(np.uint32), ya.view(np.uint32))
    sb = F.parse(b)
    out, _ = F.decompress(F.parse(a))
    np.testing.assert_array_equal(out.values.view(np.uint32), ya.view(np.uint32))
    out, _ = F.decompress(sb)
    np.testing.assert_array_equal(out.values.view(np.uint32), yb.view(np.uint32))
    reg, _ = F.decompress_region(sa, ((1, 2, 3), (20, 15, 22)))
    np.testing.assert_array_equal(reg.values.view(np.uint32), ya[1:20, 2:15, 3:22].view(np.uint32))


def test_decompress_bytes_validates_caller_output_buffer():
    x = _seeded("smooth", (12, 10, 9), seed=4)
    data = F.compress_bytes(x, "absolute", 1e-3)
    good = np.empty(x.size, np.float32)
    assert F.decompress_bytes(data, out=good) is good
    for bad in (np.empty(x.size - 1, np.float32), np.empty(x.size, np.float64),
                np.empty((x.size * 2,), np.float32)[::2]):
        with pytest.raises(ValueError):
            F.decompress_bytes(data, out=bad)
    ro = np.empty(x.size, np.float32)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        F.decompress_bytes(data, out=ro)


# Lorenzo blocks of 3-D fields with >= 4096 blocks are quantized inside k_quant_reg10 (before its
# regression blocks); every fault seam of that path against the oracle: input flips after the
# checksum (protected and not), duplicated-evaluation flips in all three rounds, ragged edges
@pytest.mark.parametrize("protect", [True, False])
def test_lorenzo_blocks_inside_the_regression_kernel(protect):
    dims = (171, 165, 158)   # 18 x 17 x 16 = 4896 blocks, ragged in every axis
    x = _seeded("smooth", dims, seed=11)
    nb = 18 * 17 * 16
    rng = np.random.default_rng(3)
    lor = sorted(int(b) for b in rng.choice(nb, 300, replace=False))
    override = {b: 0 for b in lor}   # forced Lorenzo
    faults = []
    def vol(b):
        bi, r = divmod(b, 17 * 16)
        bj, bk = divmod(r, 16)
        return min(10, 171 - 10 * bi) * min(10, 165 - 10 * bj) * min(10, 158 - 10 * bk)

    for t, b in enumerate(lor[:60]):
        el = int(rng.integers(0, vol(b)))
        if t % 3 == 0:
            faults.append(("input", b, el, int(rng.integers(0, 32))))
        elif t % 3 == 1:
            faults.append(("dup_predict", b, el, int(rng.integers(0, 192))))
        else:
            faults.append(("dup_reconstruct", b, el, int(rng.integers(0, 192))))
    # and blocks of the last (8-point) z layer, quantized by regx_block in the same kernel
    last = [b for b in range(nb) if b % 16 == 15 and b not in override][:40]
    for t, b in enumerate(last):
        el = int(rng.integers(0, vol(b)))
        kind = ("input", "dup_predict", "dup_reconstruct")[t % 3]
        faults.append((kind, b, el, int(rng.integers(0, 32 if kind == "input" else 192))))
    cfg = dict(protect_input=protect, duplicate_eval=True)
    want, wrep = O.compress(x, "value_range_relative", 1e-3, cfg, faults=faults, override=override, threads=4)
    stream, rep = F.compress(F.Field.from_array(x), F.ErrorBound("value_range_relative", 1e-3), F.FtConfig(**cfg),
                             predictor_override=override, faults=faults)
    assert F.serialize(stream) == want
    rd = rep.to_dict()
    for k in ("input_corrected", "dup_mismatch_resolved"):
        assert rd[k] == wrep[k], k
    assert rd["dup_mismatch_resolved"] and bool(rd["input_corrected"]) == protect


def test_threads_run_the_pipeline_concurrently_on_their_own_contexts():
    """Each thread owns a library context: compress and decompress calls from two threads at
    once give the sequential results bit for bit."""
    import threading

    xs = [_seeded(k, (60, 70, 80), seed=s) for k, s in (("smooth", 1), ("lognormal", 2), ("noise", 3))]
    want = [F.compress_bytes(x, "value_range_relative", 1e-3) for x in xs]
    outs = [F.decompress_bytes(w) for w in want]
    got, dec, errs = {}, {}, []

    def work(i):
        try:
            for _ in range(3):
                a = F.compress_bytes(xs[i], "value_range_relative", 1e-3)
                got[i] = a
                dec[i] = F.decompress_bytes(a)
        except Exception as ex:   # noqa: BLE001
            errs.append(ex)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(3):
        assert got[i] == want[i]
        np.testing.assert_array_equal(dec[i].view(np.uint32), outs[i].view(np.uint32))


# Lorenzo blocks of 2-D fields (1 x by x bz) are quantized and reconstructed a lane per block
# (lor2d.cu); blocks with injected faults or a failed stage (a) checksum go to the warp kernel.
@pytest.mark.parametrize("protect", [True, False])
def test_two_d_lorenzo_lane_kernels_against_oracle(protect):
    dims = (1, 233, 171)   # 24 x 18 blocks, ragged in y and z
    x = _seeded("smooth", dims, seed=21)
    nb = 24 * 18
    rng = np.random.default_rng(5)
    lor = sorted(int(b) for b in rng.choice(nb, 200, replace=False))
    override = {b: 0 for b in lor}

    def vol(b):
        bj, bk = divmod(b, 18)
        return min(10, 233 - 10 * bj) * min(10, 171 - 10 * bk)

    faults = []
    for t, b in enumerate(lor[:30]):
        el = int(rng.integers(0, vol(b)))
        kind = ("input", "dup_predict", "dup_reconstruct")[t % 3]
        faults.append((kind, b, el, int(rng.integers(0, 32 if kind == "input" else 192))))
    cfg = dict(protect_input=protect, duplicate_eval=True)
    want, wrep = O.compress(x, "value_range_relative", 1e-3, cfg, faults=faults, override=override, threads=4)
    stream, rep = F.compress(F.Field.from_array(x), F.ErrorBound("value_range_relative", 1e-3), F.FtConfig(**cfg),
                             predictor_override=override, faults=faults)
    data = F.serialize(stream)
    assert data == want
    rd = rep.to_dict()
    for k in ("input_corrected", "dup_mismatch_resolved"):
        assert rd[k] == wrep[k], k
    # decompress, clean and with decompressed-data flips on Lorenzo blocks
    ref, _ = O.decompress(want, threads=4)
    out = F.decompress_bytes(data)
    np.testing.assert_array_equal(out.view(np.uint32), ref.view(np.uint32))
    dfaults = [("decomp", b, int(rng.integers(0, vol(b))), int(rng.integers(0, 32))) for b in lor[30:60]]
    o2, r2 = F.decompress(F.parse(data), faults=dfaults)
    ro, rr = O.decompress(want, faults=dfaults, threads=4)
    assert r2.to_dict()["decomp_block_reexecuted"] == rr["decomp_block_reexecuted"]
    np.testing.assert_array_equal(o2.values.view(np.uint32), ro.view(np.uint32))


def test_warp_decoder_oversized_slices_and_reexecution():
    """Small smooth field (the warp-per-block decoder) with a few noisy blocks whose slices exceed
    its shared-memory staging (decoded by one lane from global memory); decompressed-data flips on
    those blocks are re-executed from the checkpoints that path records."""
    x = _seeded("smooth", (60, 60, 60), seed=31).astype(np.float64)
    rng = np.random.default_rng(9)
    x[0:10, 0:10, 0:20] += rng.standard_normal((10, 10, 20)) * 10.0   # blocks 0 and 1
    x[30:40, 50:60, 10:20] += rng.standard_normal((10, 10, 10)) * 10.0
    x = x.astype(np.float32)
    data = F.compress_bytes(x, "absolute", 1e-3)   # the noisy blocks: ~17.7 bits per point
    want, _ = O.compress(x, "absolute", 1e-3, threads=4)
    assert data == want
    assert len(data) * 8 <= 6 * x.size   # the field as a whole stays on the warp decoder
    ref, _ = O.decompress(want, threads=4)
    np.testing.assert_array_equal(F.decompress_bytes(data).view(np.uint32), ref.view(np.uint32))
    noisy = [0, 1, (3 * 6 + 5) * 6 + 1]
    faults = [("decomp", b, int(rng.integers(0, 1000)), int(rng.integers(0, 32))) for b in noisy]
    out, rep = F.decompress(F.parse(data), faults=faults)
    ro, rr = O.decompress(want, faults=faults, threads=4)
    assert rep.to_dict()["decomp_block_reexecuted"] == rr["decomp_block_reexecuted"] == sorted(noisy)
    np.testing.assert_array_equal(out.values.view(np.uint32), ro.view(np.uint32))


def test_block_table_of_more_than_256_super_chunks():
    """A block table longer than 256 super-chunks (4 MiB) takes the k_parse_top walk."""
    x = _seeded("lognormal", (170, 170, 150), seed=41)   # 541,875 blocks, a 4.9 MB table
    cfg = {"block_edge": 2}
    want, _ = O.compress(x, "value_range_relative", 1e-3, cfg, threads=8)
    got = F.compress_bytes(x, "value_range_relative", 1e-3, F.FtConfig(block_edge=2))
    assert got == want
    assert len(F.parse(got).records) == 85 * 85 * 75
    ref, _ = O.decompress(want, threads=8)
    np.testing.assert_array_equal(F.decompress_bytes(got).view(np.uint32), ref.view(np.uint32))
