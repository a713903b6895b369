"""Backend codec 1 (run-length pairs, encode.py:287-312) on the device, against fixtures made
by the reference itself (tools/make_golden.py --codec): the codec on raw byte vectors, codec-1
archives byte for byte, their reconstructions, and the parse errors of damaged run-length
sections (container.py:241-262).  Codec 2 (zlib) stays UnsupportedCodec on this path."""

import numpy as np
import pytest

import paper_2010_03144_b200 as F
from paper_2010_03144_b200 import container as CT
from tests.golden_util import load, manifest, sha

pytestmark = pytest.mark.gpu

M = manifest()
C1 = M.get("codec1", {})


def _cfg(d):
    return F.FtConfig(**dict(d))


def test_device_rle_matches_reference_vectors():
    z = load("rle_vectors")
    for k in sorted(n[3:] for n in z.files if n.startswith("in_")):
        src, want = z[f"in_{k}"].tobytes(), z[f"out_{k}"].tobytes()
        assert CT.rle_apply(src) == want, k
        assert CT.rle_invert(want) == src, k


@pytest.mark.parametrize("blob,msg", [(b"\x01\x02\x03", "run-length stream has odd length"),
                                      (b"\x01\x02\x00\x05", "run-length stream has zero-length run"),
                                      (b"\x02\x07" * 5000 + b"\x00\x01", "run-length stream has zero-length run")])
def test_device_rle_invert_errors(blob, msg):
    with pytest.raises(F.CorruptStream) as ei:
        CT.rle_invert(blob)
    assert str(ei.value) == msg


def test_device_rle_long_runs_and_tiles():
    # runs crossing the 8 KiB tiles of the device kernels, lengths around multiples of 255
    rng = np.random.default_rng(5)
    parts = [bytes([int(v)]) * int(n) for v, n in zip(rng.integers(0, 4, 400), rng.integers(1, 2000, 400))]
    parts.append(b"\x09" * 70000)
    data = b"".join(parts)
    from oracle import oracle as O
    want = O.rle_apply(data)
    assert CT.rle_apply(data) == want
    assert CT.rle_invert(want) == data


@pytest.mark.parametrize("name", sorted(C1))
def test_codec1_archive_and_output_match_reference(name):
    e = C1[name]
    z = load(name)
    x = z["input"]
    stream, _ = F.compress(F.Field.from_array(x), F.ErrorBound(e["mode"], e["value"]), _cfg(e["cfg"]))
    data = F.serialize(stream)
    assert len(data) == e["archive_len"]
    assert data == z["archive"].tobytes()
    assert stream.codec_id == 1
    out, rep = F.decompress(F.parse(data))
    assert rep.to_dict()["status"] == e["decompress_report"]["status"]
    np.testing.assert_array_equal(out.values.view(np.uint32), z["output"].view(np.uint32))
    # materialised fields (payload and sum_dc inverted on the device) re-serialize identically
    p = F.parse(data)
    assert len(p.payload) == (sum(r.bit_length for r in p.records) + 7) // 8
    import dataclasses
    rebuilt = dataclasses.replace(p)
    assert F.serialize(rebuilt) == data


@pytest.mark.parametrize("name,case", [(n, c) for n in sorted(C1) for c in sorted(C1[n]["corrupt"])])
def test_codec1_damaged_sections_match_reference(name, case):
    e = C1[name]["corrupt"][case]
    blob = load(name)[f"corrupt_{case}"].tobytes()
    if e["error"]:
        with pytest.raises(F.FtlzError) as ei:
            F.decompress(F.parse(blob))
        assert type(ei.value).__name__ == e["error"]["cls"]
        assert str(ei.value) == e["error"]["msg"]
        return
    out, rep = F.decompress(F.parse(blob))
    rd = rep.to_dict()
    assert rd["status"] == e["report"]["status"]
    assert rd["detail"] == e["report"]["detail"]
    assert (out is None) == (e["output_sha256"] is None)


def test_codec1_roundtrip_equals_codec0_output():
    """Size-independent property: the backend codec never changes the reconstruction."""
    from tools import synth
    x = synth.field("c1")
    eb = F.ErrorBound("value_range_relative", 1e-3)
    s0, _ = F.compress(F.Field.from_array(x), eb, F.FtConfig())
    s1, _ = F.compress(F.Field.from_array(x), eb, F.FtConfig(codec_id=1))
    d0, d1 = F.serialize(s0), F.serialize(s1)
    from oracle import oracle as O
    assert d1[5] == 1 and d0[5] == 0
    p0 = F.parse(d0)
    assert F.parse(d1).payload == p0.payload
    o0, _ = F.decompress(F.parse(d0))
    o1, _ = F.decompress(F.parse(d1))
    np.testing.assert_array_equal(o0.values.view(np.uint32), o1.values.view(np.uint32))
    assert O.rle_apply(p0.payload) in d1


def test_codec2_is_unsupported():
    x = np.zeros((8, 8, 8), np.float32) + np.arange(8, dtype=np.float32)
    with pytest.raises(F.UnsupportedCodec):
        F.compress(F.Field.from_array(x), F.ErrorBound("absolute", 1e-3), F.FtConfig(codec_id=2))


@pytest.mark.parametrize("name", sorted(C1))
def test_codec1_region_extraction_matches_full_decompress(name):
    """decompress_region (pipeline.py:726-795) on a codec-1 archive: the payload and sum_dc
    are inverted on the device by the parse, then only the intersecting blocks decode."""
    z = load(name)
    data = z["archive"].tobytes()
    full, _ = F.decompress(F.parse(data))
    dims = full.values.shape
    lo = tuple(d // 4 for d in dims)
    hi = tuple(max(l + 1, (3 * d) // 4) for l, d in zip(lo, dims))
    out, rep = F.decompress_region(F.parse(data), (lo, hi))
    assert rep.to_dict()["status"] == "clean"
    want = full.values[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]
    np.testing.assert_array_equal(out.values.view(np.uint32), want.view(np.uint32))


def test_codec1_fault_campaign_cell_matches_codec0():
    """Injected input / bins / decompressed-data flips behave the same under codec 1: the
    backend codec only changes how the payload is stored (faults.py:143-260)."""
    from paper_2010_03144_b200 import faults as FT
    f = F.synth_field("mixed", (16, 14, 12), seed=21) if hasattr(F, "synth_field") else None
    if f is None:
        x = np.random.default_rng(3).standard_normal((16, 14, 12)).astype(np.float32)
        f = F.Field.from_array(x)
    eb = F.ErrorBound.absolute(1e-3)
    for tgt in ("input", "bins", "decomp"):
        for seed in range(3):
            plan = FT.InjectionPlan(target=tgt, seed=seed)
            o0 = FT.run_trial(f, eb, F.FtConfig(block_edge=5), plan)
            o1 = FT.run_trial(f, eb, F.FtConfig(block_edge=5, codec_id=1), plan)
            assert o0.classification == o1.classification
            assert o0.corrected == o1.corrected
            assert o0.max_abs_error == o1.max_abs_error
            assert o0.bit_identical_output == o1.bit_identical_output
