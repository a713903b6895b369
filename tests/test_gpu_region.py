"""Region extraction (reference pipeline.py:726-810) on the device path.

Fixtures: tests/golden/manifest.json["region"], produced by running the reference's
decompress_region on clean and payload-damaged archives (tools/make_golden.py --region):
status, SDC detail, re-executed blocks and the extracted values must match.  The reference's
own properties are checked too: the whole-field region equals the full decompression, every
region equals the same slice of it, block counts follow intersecting_block_count.
"""

import numpy as np
import pytest

import paper_2010_03144_b200 as F
from tests.golden_util import load, manifest, sha

M = manifest()
pytestmark = pytest.mark.gpu


def _blob(src, name):
    if name == "clean":
        return load(src)["archive"].tobytes()
    return load(f"corrupt_{src}")[name].tobytes()


@pytest.mark.parametrize("key", sorted(M.get("region", {})))
def test_region_matches_reference(key):
    e = M["region"][key]
    src, name, _ = key.split("|")
    stream = F.parse(_blob(src, name))
    reg = tuple(tuple(v) for v in e["region"])
    out, rep = F.decompress_region(stream, reg)
    assert rep.status == e["status"]
    assert rep.detail == e["detail"]
    assert list(rep.decomp_block_reexecuted) == e["reexecuted"]
    if e["output_sha256"] is None:
        assert out is None
    else:
        assert sha(out.values) == e["output_sha256"]


def _field(shape, seed):
    rng = np.random.default_rng(seed)
    i, j, k = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    x = np.sin(i / 4.0) + np.cos(j / 3.0) * np.sin(k / 5.0) + rng.normal(0, 0.05, shape)
    return x.astype(np.float32)


def test_region_slices_equal_full_decompression():
    x = _field((64, 64, 64), 6)
    stream, _ = F.compress(F.Field.from_array(x), F.ErrorBound.absolute(1e-3), F.FtConfig.protected(block_edge=8))
    full, _ = F.decompress(stream)
    regions = {1: ((0, 0, 0), (64, 64, 64)), 2: ((0, 0, 0), (64, 64, 32)),
               4: ((0, 0, 0), (64, 32, 32)), 8: ((0, 0, 0), (32, 32, 32))}
    for frac, reg in regions.items():
        assert F.intersecting_block_count(stream, reg) == 512 // frac
        got, rep = F.decompress_region(stream, reg)
        assert rep.status == "clean"
        (x0, y0, z0), (x1, y1, z1) = reg
        want = np.ascontiguousarray(full.values[x0:x1, y0:y1, z0:z1])
        assert np.array_equal(got.values.view(np.uint32), want.view(np.uint32))
    rng = np.random.default_rng(1)
    for _ in range(20):
        lo = rng.integers(0, 63, 3)
        hi = [int(rng.integers(a + 1, 65)) for a in lo]
        reg = (tuple(int(v) for v in lo), tuple(hi))
        got, _ = F.decompress_region(stream, reg)
        want = np.ascontiguousarray(full.values[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]])
        assert np.array_equal(got.values.view(np.uint32), want.view(np.uint32)), reg


def test_region_out_of_bounds():
    x = _field((10, 10, 10), 17)
    stream, _ = F.compress(F.Field.from_array(x), F.ErrorBound.absolute(1e-3))
    for reg in (((0, 0, 0), (11, 10, 10)), ((-1, 0, 0), (5, 5, 5)), ((4, 4, 4), (4, 5, 5))):
        with pytest.raises(F.InvalidRegion):
            F.decompress_region(stream, reg)
