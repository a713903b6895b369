"""Pin the CPU oracle (oracle/ftlz_oracle.c) against the reference's own outputs.

Every fixture in tests/golden was produced by running the reference Python package
(tools/make_golden.py).  The oracle must reproduce each archive byte-for-byte, every
report list, every decompressed word and every exception class + message.
"""

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_util import faults_of, load, manifest, override_of, sha

M = manifest()


@pytest.mark.parametrize("name", sorted(M["cases"]))
def test_oracle_compress_decompress_matches_reference(name):
    e = M["cases"][name]
    z = load(name)
    x = z["input"]
    assert sha(x) == e["input_sha256"]
    faults = faults_of(e)
    if "compress_error" in e:
        with pytest.raises(O.OracleError) as ei:
            O.compress(x, e["mode"], e["value"], e["cfg"], faults, override_of(e))
        assert ei.value.cls == e["compress_error"]["cls"]
        assert str(ei.value) == e["compress_error"]["msg"]
        return
    data, rep = O.compress(x, e["mode"], e["value"], e["cfg"], faults, override_of(e))
    assert data == z["archive"].tobytes()
    for k in ("status", "input_corrected", "bins_corrected", "dup_mismatch_resolved",
              "decomp_block_reexecuted", "detail"):
        assert rep[k] == e["compress_report"][k], k
    out, drep = O.decompress(data, faults)
    for k in ("status", "decomp_block_reexecuted", "detail"):
        assert drep[k] == e["decompress_report"][k], k
    if "output_sha256" in e:
        assert out is not None and sha(out) == e["output_sha256"]
        np.testing.assert_array_equal(out.view(np.uint32), z["output"].view(np.uint32))
    else:
        assert out is None


def _corrupt_cases():
    for src, cases in sorted(M["corrupt"].items()):
        for name in sorted(cases):
            yield src, name


@pytest.mark.parametrize("src,name", list(_corrupt_cases()))
def test_oracle_parse_and_sdc_match_reference(src, name):
    e = M["corrupt"][src][name]
    blob = load(f"corrupt_{src}")[name].tobytes()
    assert sha(np.frombuffer(blob, np.uint8)) == e["sha256"]
    if "error" in e:
        with pytest.raises(O.OracleError) as ei:
            O.decompress(blob)
        assert ei.value.cls == e["error"]["cls"]
        assert str(ei.value) == e["error"]["msg"]
        return
    out, rep = O.decompress(blob)
    for k in ("status", "decomp_block_reexecuted", "detail"):
        assert rep[k] == e["decompress_report"][k], k
    assert (None if out is None else sha(out)) == e["output_sha256"]


def test_oracle_rle_matches_reference_vectors():
    """Backend codec 1 restatement (oracle) against the reference's own _rle_apply output."""
    z = load("rle_vectors")
    names = sorted(k[3:] for k in z.files if k.startswith("in_"))
    assert len(names) >= 9
    for k in names:
        src, want = z[f"in_{k}"].tobytes(), z[f"out_{k}"].tobytes()
        assert O.rle_apply(src) == want, k
        assert O.rle_invert(want) == src, k


def test_oracle_rle_invert_errors():
    with pytest.raises(O.OracleError) as ei:
        O.rle_invert(b"\x01\x02\x03")
    assert str(ei.value) == "run-length stream has odd length"
    with pytest.raises(O.OracleError) as ei:
        O.rle_invert(b"\x01\x02\x00\x05")
    assert str(ei.value) == "run-length stream has zero-length run"


def _truncation():
    import json
    import os

    from tests.golden_util import GOLDEN

    with open(os.path.join(GOLDEN, "truncation.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("src", sorted(_truncation()))
def test_oracle_truncation_sweep_every_byte(src):
    """test_container.py:59-63: every proper prefix of an archive is a CorruptStream, with the
    reference's own message and offset for each cut."""
    t = _truncation()[src]
    arch = load(src)["archive"].tobytes()
    assert len(arch) == t["len"]
    for cut, ix in enumerate(t["index"]):
        cls, msg = t["messages"][ix]
        with pytest.raises(O.OracleError) as ei:
            O.parse_check(arch[:cut])
        assert (ei.value.cls, str(ei.value)) == (cls, msg), cut
