"""compress / decompress of the drop-in API (reference pipeline.py:71-142, 287-537, 645-723).

Both directions run entirely on one B200 through libftlz_b200.so: Algorithm 1 (block prep,
duplicated prediction/reconstruction, quantization, ABFT checksums, Huffman coding, archive
assembly) and Algorithm 2 (device parse, decode, reconstruction, checksum verification,
re-execution).  Fault injection uses per-call descriptors instead of the reference's global
hook registry: ``faults=[(target, block, element, bit), ...]`` with the targets of
faults.py:157-189 ("input", "bins", "decomp", "regression", "sampling") plus the duplicated-
evaluation seam ("dup_predict", "dup_reconstruct"; hooks.STAGE_DUP_EVAL).
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._messages import raise_for_info, sdc_detail
from .container import CompressedStream, _sections_from_report, serialize
from .core import DEFAULT_BLOCK_EDGE, EB_MODE_CODES, ErrorBound, Field, partition
from .errors import InvalidInjection
from .quantize import QuantConfig

STATUS_CLEAN = "clean"
STATUS_CORRECTED = "corrected"
STATUS_SDC = "sdc_in_compression"

CODEC_IDENTITY = 0

TARGETS = {"input": 0, "input_after_checksum": 0, "bins": 1, "bin_array": 1, "decomp": 2,
           "decompressed_buffer": 2, "regression": 3, "regression_fit": 3, "sampling": 4,
           "dup_predict": 5, "dup_reconstruct": 6}
# dup_* faults (STAGE_DUP_EVAL, pipeline.py:157-179): bit = 64 * (round - 1) + b flips bit b of
# the float64 value evaluation `round` (1..3) of the prediction / reconstruction returns


@dataclass(frozen=True)
class FtConfig:
    """Protection switches + geometry (pipeline.py:71-99)."""

    protect_input: bool = True
    protect_bins: bool = True
    duplicate_eval: bool = True
    store_sum_dc: bool = True
    block_edge: int = DEFAULT_BLOCK_EDGE
    codec_id: int = CODEC_IDENTITY
    quant: QuantConfig = field(default_factory=QuantConfig)

    @classmethod
    def protected(cls, **kw) -> "FtConfig":
        return cls(**kw)

    @classmethod
    def unprotected(cls, **kw) -> "FtConfig":
        return cls(protect_input=False, protect_bins=False, duplicate_eval=False,
                   store_sum_dc=False, **kw)

    def _c(self) -> _lib.Config:
        return _lib.Config(int(self.protect_input), int(self.protect_bins),
                           int(self.duplicate_eval), int(self.store_sum_dc),
                           int(self.block_edge), int(self.codec_id),
                           int(self.quant.bin_capacity), 0)


@dataclass
class FtReport:
    """Per-block fault-tolerance events of one run (pipeline.py:102-142)."""

    input_corrected: list = field(default_factory=list)
    bins_corrected: list = field(default_factory=list)
    dup_mismatch_resolved: list = field(default_factory=list)
    decomp_block_reexecuted: list = field(default_factory=list)
    sdc_in_compression: bool = False
    detail: str = ""

    @property
    def status(self) -> str:
        if self.sdc_in_compression:
            return STATUS_SDC
        if (self.input_corrected or self.bins_corrected or self.dup_mismatch_resolved
                or self.decomp_block_reexecuted):
            return STATUS_CORRECTED
        return STATUS_CLEAN

    def to_dict(self) -> dict:
        return {
            "status": self.status,
            "input_corrected": list(self.input_corrected),
            "bins_corrected": list(self.bins_corrected),
            "dup_mismatch_resolved": list(self.dup_mismatch_resolved),
            "decomp_block_reexecuted": list(self.decomp_block_reexecuted),
            "detail": self.detail,
        }


# ------------------------------------------------------------------------------------------
def _faults_c(faults):
    faults = list(faults or [])
    arr = (_lib.Fault * max(1, len(faults)))()
    for i, f in enumerate(faults):
        target, block, element, bit = f
        t = TARGETS.get(target, target) if isinstance(target, str) else int(target)
        if not isinstance(t, int):
            raise InvalidInjection(f"unknown injection target {target!r}")
        arr[i] = _lib.Fault(t, int(bit), int(block), int(element))
    return arr, len(faults)


_tls = threading.local()


def _report_buf(capacity: int) -> "_ReportBuf":
    """Per-thread report buffers, reused across calls (results are copied out by lists())."""
    cache = getattr(_tls, "reports", None)
    if cache is None:
        cache = _tls.reports = {}
    rb = cache.pop(capacity, None)
    if rb is None:
        rb = _ReportBuf(capacity)
        while len(cache) >= 4:   # bounded: keep the most recently used block counts
            cache.pop(next(iter(cache)))
    cache[capacity] = rb
    return rb


class _ReportBuf:
    def __init__(self, capacity: int):
        self.bufs = [np.zeros(max(1, capacity), np.int64) for _ in range(4)]
        self.r = _lib.Report()
        self.r.capacity = capacity
        P = C.POINTER(C.c_int64)
        (self.r.input_corrected, self.r.bins_corrected, self.r.dup_mismatch,
         self.r.reexecuted) = (b.ctypes.data_as(P) for b in self.bufs)

    def lists(self):
        r = self.r
        ns = (r.n_input_corrected, r.n_bins_corrected, r.n_dup_mismatch, r.n_reexecuted)
        return [b[:n].tolist() for b, n in zip(self.bufs, ns)]


def _check_out(out, shape):
    """A caller-supplied output array receives 4 * prod(shape) bytes straight from the device:
    it must be a writable, C-contiguous float32 array of exactly that size."""
    if not isinstance(out, np.ndarray):
        raise ValueError("out must be a numpy float32 array")
    n = int(np.prod(shape, dtype=np.int64))
    if out.dtype != np.float32 or not out.flags.c_contiguous or not out.flags.writeable or out.size != n:
        raise ValueError(f"out must be a writable C-contiguous float32 array of {n} elements "
                         f"(got {out.dtype}, {out.size} elements, contiguous={out.flags.c_contiguous}, "
                         f"writeable={out.flags.writeable})")


def compress(field: Field, eb_spec: ErrorBound, cfg: FtConfig = FtConfig(), threads: int = 1,
             predictor_override=None, faults=None) -> tuple:
    """Compress a field (pipeline.py:287-537) -> (CompressedStream, FtReport).

    `threads` is accepted for API compatibility; the device runs all blocks at once.
    Raises DegenerateBound / UncorrectableCorruption / InternalInvariantViolation like the
    reference."""
    values = field.values if isinstance(field, Field) else np.ascontiguousarray(field, np.float32)
    grid = partition(values.shape, cfg.block_edge)
    data, rep = _compress_array(values, eb_spec, cfg, predictor_override, faults, grid)
    nb = grid.n_blocks
    r = rep.r
    stream = CompressedStream._from_archive(data, _sections_from_report(r, nb, cfg.store_sum_dc, cfg.codec_id))
    ic, bc, dm, _ = rep.lists()
    return stream, FtReport(input_corrected=ic, bins_corrected=bc, dup_mismatch_resolved=dm)


def _compress_array(values, eb_spec, cfg, predictor_override, faults, grid, out=None):
    L = _lib.load()
    ctx = _lib.context()
    x = np.ascontiguousarray(values, dtype=np.float32)
    nx, ny, nz = x.shape
    nb = grid.n_blocks
    fa, nf = _faults_c(faults)
    ov = None
    if predictor_override:
        ov = np.full(nb, -1, np.int8)
        for b, k in predictor_override.items():
            ov[int(b)] = int(k)
    rep = _report_buf(nb)
    args = (ctx, x.ctypes.data, nx, ny, nz, EB_MODE_CODES[eb_spec.mode], float(eb_spec.value),
            C.byref(cfg._c()), fa, nf, ov.ctypes.data if ov is not None else None)
    if out is not None:
        # the archive goes straight from the device into the caller's buffer
        ob = np.frombuffer(out, np.uint8)
        st = L.ftlz_ctx_compress_host_to(*args, ob.ctypes.data, ob.size, C.byref(rep.r))
        if st == 9 and rep.r.archive_len > ob.size:
            raise ValueError(f"output buffer holds {ob.size} bytes, archive needs {rep.r.archive_len}")
        if st != 0:
            raise_for_info(st, rep.r.info, eb_request=(eb_spec.mode, eb_spec.value), resolved=rep.r.eb)
        return rep.r.archive_len, rep
    st = L.ftlz_ctx_compress_host(*args, C.byref(rep.r))
    if st != 0:
        raise_for_info(st, rep.r.info, eb_request=(eb_spec.mode, eb_spec.value), resolved=rep.r.eb)
    ptr = C.c_void_p()
    ln = C.c_size_t()
    L.ftlz_ctx_archive_host(ctx, C.byref(ptr), C.byref(ln))
    return C.string_at(ptr, ln.value), rep


def compress_bytes(array: np.ndarray, mode: str, value: float, cfg: FtConfig = FtConfig(),
                   out=None, faults=None):
    """array + (mode, value) -> archive bytes (north-star form of compress+serialize).
    With `out` (a writable buffer, e.g. pinned numpy memory) the archive is copied there and
    its length returned."""
    grid = partition(np.shape(array), cfg.block_edge)
    data, _ = _compress_array(array, ErrorBound(mode, value), cfg, None, faults, grid, out=out)
    return data


def decompress(stream: CompressedStream, threads: int = 1, faults=None) -> tuple:
    """Decompress (pipeline.py:645-723) -> (Field or None, FtReport).

    A block whose decompressed checksum mismatches is re-executed once; a second mismatch or
    an undecodable block withholds the output (None) and reports sdc_in_compression."""
    data = serialize(stream)
    out, rep = _decompress_bytes(data, faults, reuse=stream.__dict__.get("_parse_token"))
    return (None if out is None else Field._wrap(out)), rep


def _decompress_bytes(data, faults=None, out=None, reuse=None):
    L = _lib.load()
    ctx = _lib.context()
    hdr = _lib.Header()
    info = _lib.Info()
    if not isinstance(data, bytes):
        # any contiguous byte buffer (e.g. pinned numpy memory) is read in place
        data = np.frombuffer(data, np.uint8)
    buf = data if isinstance(data, bytes) else data.ctypes.data
    # the header checks see the whole buffer: an archive too short for its record table is
    # rejected here (reference message and offset) before anything is sized by its dims
    st = L.ftlz_peek_archive(buf, len(data), C.byref(hdr), C.byref(info))
    if st != 0:
        raise_for_info(st, info, data)
    shape = (hdr.nx, hdr.ny, hdr.nz)
    if out is None:
        out = np.empty(shape, np.float32)
    else:
        _check_out(out, shape)
    fa, nf = _faults_c(faults)
    rb = _report_buf(int(hdr.block_count))
    st = L.ftlz_ctx_decompress_host(ctx, buf, len(data), out.ctypes.data, fa, nf,
                                    1 if reuse is not None and reuse is _lib.last_parse() else 0,
                                    C.byref(rb.r))
    if st != 0:
        raise_for_info(st, rb.r.info, data)
    _, _, _, rx = rb.lists()
    sdc = bool(rb.r.sdc)
    report = FtReport(decomp_block_reexecuted=rx, sdc_in_compression=sdc,
                      detail=sdc_detail(rb.r.info) if sdc else "")
    return (None if sdc else out), report



def decompress_bytes(data: bytes, out=None, faults=None):
    """archive bytes -> float32 array (north-star form of parse+decompress).  Returns None
    when the archive fails verification (the report is then available via decompress)."""
    arr, _ = _decompress_bytes(data, faults, out=out)
    return arr


def decompress_region(stream: CompressedStream, region, threads: int = 1) -> tuple:
    """Decode only the blocks intersecting the half-open box ((x0,y0,z0),(x1,y1,z1))
    (pipeline.py:726-795) -> (Field or None, FtReport).  Values are bit-identical to the same
    slice of a full decompression; each block is verified against its sum_dc with one
    re-execution.  InvalidRegion when the box is empty or leaves the field."""
    from .errors import InvalidRegion

    (x0, y0, z0), (x1, y1, z1) = region
    nx, ny, nz = stream.dims
    if not (0 <= x0 < x1 <= nx and 0 <= y0 < y1 <= ny and 0 <= z0 < z1 <= nz):
        raise InvalidRegion(f"region {region} outside dims {stream.dims}")
    data = serialize(stream)
    L = _lib.load()
    ctx = _lib.context()
    r6 = np.array([x0, y0, z0, x1, y1, z1], np.int64)
    out = np.empty((x1 - x0, y1 - y0, z1 - z0), np.float32)
    hdr = _lib.Header()
    info = _lib.Info()
    st = L.ftlz_peek_archive(data, len(data), C.byref(hdr), C.byref(info))
    if st != 0:
        raise_for_info(st, info, data)
    rb = _report_buf(int(hdr.block_count))
    reuse = stream.__dict__.get("_parse_token")
    st = L.ftlz_ctx_decompress_region_host(ctx, data, len(data), r6.ctypes.data, out.ctypes.data,
                                           1 if reuse is not None and reuse is _lib.last_parse() else 0,
                                           C.byref(rb.r))
    if st != 0:
        raise_for_info(st, rb.r.info, data)
    _, _, _, rx = rb.lists()
    sdc = bool(rb.r.sdc)
    report = FtReport(decomp_block_reexecuted=rx, sdc_in_compression=sdc,
                      detail=sdc_detail(rb.r.info, region=True) if sdc else "")
    return (None if sdc else Field._wrap(out)), report


def intersecting_block_count(stream_or_grid, region) -> int:
    """Number of blocks a region extraction decodes (pipeline.py:798-810)."""
    from .core import BlockGrid

    grid = stream_or_grid if isinstance(stream_or_grid, BlockGrid) else partition(
        stream_or_grid.dims, stream_or_grid.block_edge)
    (x0, y0, z0), (x1, y1, z1) = region
    e = grid.block_edge
    return (-(-x1 // e) - x0 // e) * (-(-y1 // e) - y0 // e) * (-(-z1 // e) - z0 // e)


def cr_decrease_bound(r0: float, n_blocks: int) -> float:
    """(r0 - 1) / (r0 + n - 1) * 100 (pipeline.py:182-189)."""
    from .errors import InvalidArgument

    if not r0 >= 1.0:
        raise InvalidArgument(f"baseline ratio must be >= 1, got {r0}")
    if n_blocks < 1:
        raise InvalidArgument(f"block count must be >= 1, got {n_blocks}")
    return (r0 - 1.0) / (r0 + n_blocks - 1.0) * 100.0
