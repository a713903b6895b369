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
