"""CPU-only checks of the boundary and the host-side mirror of the reference interface.

* the C-ABI library (paper_2010_03144_b200/lib/libftlz_b200.so) loads and exports every entry
  point include/ftlz_b200.h declares; its host-only entry points (no device) agree with the
  reference semantics: default config (pipeline.py:71-99), block count (core.py:133-157),
  header peek (container.py:173-200);
* host logic: Field / partition / ErrorBound / resolve_error_bound / FtConfig /
  cr_decrease_bound mirror core.py and pipeline.py, including their error behaviour;
* `serialize` of a stream rebuilt field-by-field reproduces the reference archive bytes
  (container.py:109-147), for every golden archive;
* the product path refuses to run without a CUDA device (no CPU fallback).
"""

import dataclasses
import math
import os
import re

import numpy as np
import pytest

import paper_2010_03144_b200 as F
from paper_2010_03144_b200 import _lib
from paper_2010_03144_b200.container import CompressedStream
from paper_2010_03144_b200.errors import BackendUnavailable
from tests.conftest import gpu_available
from tests.golden_util import load, manifest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = manifest()


def _header_functions():
    src = open(os.path.join(ROOT, "include", "ftlz_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ftlz_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_exactly_the_exported_list():
    assert _header_functions() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = _lib.load()
    for name in _header_functions():
        assert hasattr(L, name), name
    assert L.ftlz_abi_version() == 3


def test_default_config_matches_reference_defaults():
    L = _lib.load()
    c = _lib.Config()
    L.ftlz_default_config(c)
    d = F.FtConfig()
    assert (c.protect_input, c.protect_bins, c.duplicate_eval, c.store_sum_dc) == (1, 1, 1, 1)
    assert c.block_edge == d.block_edge == 10
    assert c.codec_id == d.codec_id == 0
    assert c.bin_capacity == d.quant.bin_capacity == 65536


@pytest.mark.parametrize("dims,e", [((64, 64, 64), 10), ((100, 500, 500), 10), ((1, 1800, 3600), 10),
                                    ((7, 9, 12), 4), ((1, 1, 1), 2), ((20, 20, 20), 64)])
def test_block_count_matches_partition(dims, e):
    L = _lib.load()
    g = F.partition(dims, e)
    assert L.ftlz_block_count(*dims, e) == g.n_blocks == len(g.blocks)
    nb = math.prod(-(-n // e) for n in dims)
    assert g.n_blocks == nb


def test_partition_geometry_and_errors():
    g = F.partition((12, 7, 25), 5)
    assert g.n_blocks == 3 * 2 * 5
    s = g.spec(g.n_blocks - 1)
    assert s.volume == 2 * 2 * 5
    with pytest.raises(F.InvalidGeometry):
        F.partition((4, 4), 2)
    with pytest.raises(F.InvalidGeometry):
        F.partition((4, 0, 4), 2)
    with pytest.raises(F.InvalidGeometry):
        F.partition((4, 4, 4), 1)


def test_error_bound_and_resolution():
    f = F.Field.from_array(np.linspace(-2, 6, 60, dtype=np.float32).reshape(3, 4, 5))
    assert F.resolve_error_bound(F.ErrorBound.absolute(0.5), f) == 0.5
    assert F.resolve_error_bound(F.ErrorBound.relative(1e-3), f) == pytest.approx(8e-3)
    with pytest.raises(F.DegenerateBound):
        F.ErrorBound("bogus", 1.0)
    with pytest.raises(F.DegenerateBound):
        F.ErrorBound.absolute(0.0)
    with pytest.raises(F.DegenerateBound):
        F.ErrorBound.absolute(float("nan"))
    const = F.Field.from_array(np.ones((2, 2, 2), np.float32))
    with pytest.raises(F.DegenerateBound):
        F.resolve_error_bound(F.ErrorBound.relative(1e-3), const)


def test_field_is_read_only_copy():
    a = np.arange(24, dtype=np.float32).reshape(2, 3, 4)
    f = F.Field.from_array(a)
    a[0, 0, 0] = 99
    assert f.values[0, 0, 0] == 0
    assert not f.values.flags.writeable
    with pytest.raises(F.InvalidGeometry):
        F.Field.from_flat(np.zeros(5), (2, 2, 2))


def test_ftconfig_variants():
    u = F.FtConfig.unprotected()
    assert not (u.protect_input or u.protect_bins or u.duplicate_eval or u.store_sum_dc)
    p = F.FtConfig.protected(block_edge=6)
    assert p.protect_input and p.block_edge == 6
    c = p._c()
    assert (c.protect_input, c.block_edge, c.bin_capacity) == (1, 6, 65536)


def test_cr_decrease_bound():
    assert F.cr_decrease_bound(1.0, 10) == 0.0
    assert F.cr_decrease_bound(5.0, 1) == pytest.approx(4 / 5 * 100)
    with pytest.raises(F.InvalidArgument):
        F.cr_decrease_bound(0.5, 3)
    with pytest.raises(F.InvalidArgument):
        F.cr_decrease_bound(2.0, 0)


def _golden_archives():
    for name, e in sorted(M["cases"].items()):
        if "compress_error" not in e:
            yield name


@pytest.mark.parametrize("name", list(_golden_archives()))
def test_peek_header_and_field_serialize_reproduce_reference_bytes(name):
    from oracle import oracle as O  # checker only

    data = load(name)["archive"].tobytes()
    L = _lib.load()
    hdr, info = _lib.Header(), _lib.Info()
    assert L.ftlz_peek_header(data, len(data), hdr, info) == 0
    si = O.parse_check(data)
    for k in ("nx", "ny", "nz", "block_edge", "eb_mode", "bin_capacity", "block_count", "codec_id"):
        assert getattr(hdr, k) == getattr(si.hdr, k), k
    assert hdr.eb_value == si.hdr.eb_value
    # lazy stream over the archive -> materialised fields -> field-by-field serialize
    s = CompressedStream._from_archive(data, {
        "payload_off": si.payload_off, "payload_len": si.payload_len, "unpred_off": si.unpred_off,
        "n_unpred": si.n_unpred, "has_sum_dc": bool(si.has_sum_dc), "sumdc_off": si.sumdc_off})
    assert F.serialize(s) is data
    rebuilt = dataclasses.replace(s, records=tuple(s.records), code_lengths=dict(s.code_lengths),
                                  payload=bytes(s.payload), unpred_words=bytes(s.unpred_words))
    assert "_archive" not in rebuilt.__dict__
    assert F.serialize(rebuilt) == data
    assert rebuilt.bit_offsets()[-1] == si.total_bits
    assert rebuilt.unpred_offsets()[-1] == si.n_unpred


@pytest.mark.parametrize("blob,code", [(b"", 5), (b"FTLZ", 5), (b"XTLZ" + bytes(51), 5)])
def test_peek_header_rejects_bad_headers(blob, code):
    L = _lib.load()
    hdr, info = _lib.Header(), _lib.Info()
    assert L.ftlz_peek_header(blob if blob else b"\x00", len(blob), hdr, info) == code
    assert info.offset == 0


@pytest.mark.skipif(gpu_available(), reason="checks the no-device behaviour")
def test_product_path_has_no_cpu_fallback():
    x = np.ones((4, 4, 4), np.float32)
    with pytest.raises(BackendUnavailable):
        F.compress_bytes(x, "absolute", 0.1)


def test_intersecting_block_count_matches_brute_force():
    L = _lib.load()
    grid = F.partition((64, 64, 64), 8)
    assert F.intersecting_block_count(grid, ((0, 0, 0), (64, 64, 64))) == 512
    assert F.intersecting_block_count(grid, ((0, 0, 0), (64, 64, 32))) == 256
    assert F.intersecting_block_count(grid, ((0, 0, 0), (64, 32, 32))) == 128
    assert F.intersecting_block_count(grid, ((0, 0, 0), (32, 32, 32))) == 64
    rng = np.random.default_rng(3)
    for _ in range(30):
        dims = tuple(int(v) for v in rng.integers(1, 40, 3))
        e = int(rng.integers(2, 9))
        g = F.partition(dims, e)
        lo = [int(rng.integers(0, d)) for d in dims]
        hi = [int(rng.integers(a + 1, d + 1)) for a, d in zip(lo, dims)]
        reg = (tuple(lo), tuple(hi))
        hits = 0
        for b in range(g.n_blocks):
            s = g.spec(b)
            (i0, j0, k0), (bx, by, bz) = s.origin, s.extent
            if (i0 < hi[0] and i0 + bx > lo[0] and j0 < hi[1] and j0 + by > lo[1]
                    and k0 < hi[2] and k0 + bz > lo[2]):
                hits += 1
        assert F.intersecting_block_count(g, reg) == hits
        r6 = np.array(lo + hi, np.int64)
        assert L.ftlz_intersecting_block_count(*dims, e, r6.ctypes.data) == hits


def test_region_validation_before_any_device_work():
    from oracle import oracle as O

    data = load("c1")["archive"].tobytes()
    si = O.parse_check(data)
    s = CompressedStream._from_archive(data, {
        "payload_off": si.payload_off, "payload_len": si.payload_len, "unpred_off": si.unpred_off,
        "n_unpred": si.n_unpred, "has_sum_dc": bool(si.has_sum_dc), "sumdc_off": si.sumdc_off})
    for reg in (((0, 0, 0), (65, 64, 64)), ((-1, 0, 0), (5, 5, 5)), ((4, 4, 4), (4, 5, 5))):
        with pytest.raises(F.InvalidRegion) as ei:
            F.decompress_region(s, reg)
        assert str(ei.value) == f"region {reg} outside dims (64, 64, 64)"


def test_fault_plan_helpers_mirror_reference():
    from paper_2010_03144_b200 import faults as FT

    assert FT.InjectionPlan("compressed_bytes").target == "bytes"
    with pytest.raises(F.InvalidInjection):
        FT.InjectionPlan("nowhere")
    buf = np.arange(4, dtype=np.float32)
    FT.inject_bitflip(buf, 2, 31)
    assert buf[2] == -2.0
    FT.inject_bitflip(buf, 2, 31)
    assert buf[2] == 2.0
    b = bytearray(b"\x00\x01")
    FT.inject_bitflip(b, 1, 1)
    assert b == bytearray(b"\x00\x03")
    s1, s2 = FT.trial_seed(7, 0, 0), FT.trial_seed(7, 0, 1)
    assert s1 != s2 and s1 == FT.trial_seed(7, 0, 0)


@pytest.mark.parametrize("dims,cut,flip", [((4096, 4096, 4096), 200, None), ((1000, 1000, 1000), 55, None),
                                           ((64, 64, 64), 70, None), ((300, 300, 300), 90, 2)])
def test_peek_header_rejects_short_record_tables_like_reference(dims, cut, flip):
    """An archive too short for the record table its dims imply is rejected by the host header
    check with the reference parse's own message and offset (container.py:212-218), before
    any buffer is sized by the claimed dims (the oracle restates the reference parse)."""
    from oracle import oracle as O

    nb = 1
    for d in dims:
        nb *= -(-d // 10)
    hdr = (b"FTLZ" + bytes([1, 0]) + b"".join(int(d).to_bytes(8, "little") for d in dims)
           + (10).to_bytes(4, "little") + bytes([1]) + np.float64(0.5).tobytes()
           + (65536).to_bytes(4, "little") + nb.to_bytes(8, "little"))
    body = bytearray((np.arange(cut, dtype=np.int64) % 7 == 0).astype(np.uint8).tobytes())
    if flip is not None and flip < len(body):
        body[flip] = 5   # a bad indicator byte inside the table
    blob = hdr + bytes(body)
    L = _lib.load()
    h, info = _lib.Header(), _lib.Info()
    assert L.ftlz_peek_header(blob, len(blob), h, info) == 0   # the 55-byte header itself is valid
    assert L.ftlz_peek_archive(blob, len(blob), h, info) == 5
    with pytest.raises(O.OracleError) as ei:
        O.parse_check(blob)
    assert ei.value.offset == info.offset
    from paper_2010_03144_b200._messages import raise_for_info

    with pytest.raises(F.FtlzError) as e2:
        raise_for_info(5, info, blob)
    assert (type(e2.value).__name__, str(e2.value)) == (ei.value.cls, str(ei.value))
