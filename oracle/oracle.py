"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the CPU oracle (oracle/ftlz_oracle.c).

The oracle is the checker for the B200 path: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg are the only callers.  It restates the reference
``ftlz`` 0.1.0 compress -> serialize -> parse -> decompress path in C and is pinned against
the Python reference by tests/golden/ (tools/make_golden.py) and tests/test_oracle_golden.py.

Exceptions are reported as (class name, message) pairs whose text follows the reference
modules that raise them (errors.py, core.py:188-192, pipeline.py:343,477,490,
encode.py:85-88, container.py:150-285).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libftlz_oracle.so")


class Info(C.Structure):
    _fields_ = [("code", C.c_int32), ("kind", C.c_int32), ("offset", C.c_int64),
                ("block", C.c_int64), ("a", C.c_int64), ("b", C.c_int64)]


class Config(C.Structure):
    _fields_ = [("protect_input", C.c_int32), ("protect_bins", C.c_int32),
                ("duplicate_eval", C.c_int32), ("store_sum_dc", C.c_int32),
                ("block_edge", C.c_int32), ("codec_id", C.c_int32),
                ("bin_capacity", C.c_uint32), ("reserved", C.c_int32)]


class Fault(C.Structure):
    _fields_ = [("target", C.c_int32), ("bit", C.c_int32), ("block", C.c_int64),
                ("element", C.c_int64)]


_P64 = C.POINTER(C.c_int64)


class Report(C.Structure):
    _fields_ = [("capacity", C.c_int64),
                ("input_corrected", _P64), ("bins_corrected", _P64),
                ("dup_mismatch", _P64), ("reexecuted", _P64),
                ("n_input_corrected", C.c_int64), ("n_bins_corrected", C.c_int64),
                ("n_dup_mismatch", C.c_int64), ("n_reexecuted", C.c_int64),
                ("sdc", C.c_int32), ("reserved", C.c_int32), ("info", Info),
                ("eb", C.c_double), ("archive_len", C.c_int64), ("n_blocks", C.c_int64),
                ("n_regression", C.c_int64), ("n_unpredictable", C.c_int64),
                ("n_symbols", C.c_int64), ("payload_bits", C.c_int64),
                ("max_code_len", C.c_int32), ("reserved2", C.c_int32)]


class Header(C.Structure):
    _fields_ = [("version", C.c_int32), ("codec_id", C.c_int32), ("nx", C.c_int64),
                ("ny", C.c_int64), ("nz", C.c_int64), ("block_edge", C.c_int32),
                ("eb_mode", C.c_int32), ("eb_value", C.c_double), ("bin_capacity", C.c_uint32),
                ("reserved", C.c_int32), ("block_count", C.c_int64)]


class StreamInfo(C.Structure):
    _fields_ = [("hdr", Header), ("table_off", C.c_int64), ("table_len", C.c_int64),
                ("book_off", C.c_int64), ("n_symbols", C.c_int64),
                ("payload_off", C.c_int64), ("payload_len", C.c_int64),
                ("unpred_off", C.c_int64), ("n_unpred", C.c_int64), ("sumdc_off", C.c_int64),
                ("n_regression", C.c_int64), ("total_bits", C.c_int64),
                ("max_code_len", C.c_int32), ("has_sum_dc", C.c_int32),
                ("payload_stored_len", C.c_int64), ("sumdc_stored_len", C.c_int64)]


_lib = None


def build() -> str:
    """Compile the oracle (make) if the shared object is missing or stale."""
    src = os.path.join(_HERE, "ftlz_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.oc_compress.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                  C.c_double, C.POINTER(Config), C.POINTER(Fault), C.c_int64,
                                  C.c_void_p, C.c_int32, C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_size_t), C.POINTER(Report)]
        L.oc_compress.restype = C.c_int
        L.oc_free.argtypes = [C.c_void_p]
        L.oc_rle_apply.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.oc_rle_apply.restype = C.c_int64
        L.oc_rle_invert.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.oc_rle_invert.restype = C.c_int64
        L.oc_parse.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(StreamInfo), C.POINTER(Info)]
        L.oc_parse.restype = C.c_int
        L.oc_decompress.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.POINTER(Fault),
                                    C.c_int64, C.c_int32, C.POINTER(Report)]
        L.oc_decompress.restype = C.c_int
        _lib = L
    return _lib


TARGETS = {"input": 0, "bins": 1, "decomp": 2, "regression": 3, "sampling": 4, "dup_predict": 5,
           "dup_reconstruct": 6}

_FIELD_NAMES = ["header", "block indicator", "regression coefficients", "block record",
                "codebook size", "codebook entry", "payload length", "payload",
                "unpredictable words", "checksum section lengths", "checksum section"]


class OracleError(Exception):
    """Raised with .cls = the reference exception class name, str() = reference message."""

    def __init__(self, cls: str, message: str, offset=None):
        super().__init__(message)
        self.cls = cls
        self.offset = offset


def _corrupt_message(info: Info, data: bytes) -> str:
    k, off = info.kind, info.offset
    if k == 20:
        msg = f"truncated while reading {_FIELD_NAMES[info.a]}"
    elif k == 21:
        msg = f"bad magic {bytes(data[:4])!r}"
    elif k == 22:
        msg = f"unsupported version {data[4]}"
    elif k == 23:
        dims = tuple(int.from_bytes(data[6 + 8 * i: 14 + 8 * i], "little") for i in range(3))
        msg = f"bad dims {dims}"
    elif k == 24:
        msg = f"bad block edge {int.from_bytes(data[30:34], 'little')}"
    elif k == 25:
        msg = f"bad error-bound mode {data[34]}"
    elif k == 26:
        msg = f"bad error bound {float(np.frombuffer(data[35:43], '<f8')[0])}"
    elif k == 27:
        msg = f"bad bin capacity {int.from_bytes(data[43:47], 'little')}"
    elif k == 28:
        msg = f"block count {int.from_bytes(data[47:55], 'little')} does not match dims"
    elif k == 29:
        msg = f"bad predictor indicator {info.a}"
    elif k == 30:
        msg = "codebook symbols not strictly increasing"
    elif k == 31:
        msg = f"codebook symbol {info.a} outside bin range"
    elif k == 32:
        msg = f"bad code length {info.a}"
    elif k == 33:
        msg = "empty codebook"
    elif k == 34:
        msg = "codebook violates Kraft inequality"
    elif k == 35:
        msg = "block bit lengths exceed payload"
    elif k == 36:
        msg = f"bad checksum section length {info.a}"
    elif k == 37:
        msg = "checksum section length mismatch"
    elif k == 38:
        msg = "orphan checksum payload"
    elif k == 39:
        msg = f"{info.a} trailing bytes"
    else:
        msg = f"corrupt stream kind {k}"
    return f"{msg} (offset {off})"


def raise_for(status: int, info: Info, data: bytes = b"", eb_request=None) -> None:
    if status == 0:
        return
    if status == 1:
        raise OracleError("InvalidGeometry", "invalid geometry")
    if status == 2:
        mode, value, resolved = eb_request
        raise OracleError("DegenerateBound",
                          f"resolved bound {resolved} is not positive and finite "
                          f"(mode={mode}, value={value})")
    if status == 3:
        if info.kind == 1:
            raise OracleError("UncorrectableCorruption",
                              f"input block {info.block} failed verification beyond repair")
        tag = "histogram" if info.kind == 2 else "encode"
        raise OracleError("UncorrectableCorruption",
                          f"bin array of block {info.block} failed verification beyond repair ({tag})")
    if status == 4:
        if info.kind == 4:
            raise OracleError("InternalInvariantViolation", "bin index outside quantizer range")
        raise OracleError("InternalInvariantViolation", f"code length {info.a} exceeds cap 57")
    if status == 5:
        raise OracleError("CorruptStream", _corrupt_message(info, data), info.offset)
    if status == 6:
        raise OracleError("UnsupportedCodec", f"codec {info.a} is not registered")
    raise OracleError("FtlzError", f"status {status}")


def sdc_detail(info: Info) -> str:
    k, b = info.kind, info.block
    why = {
        60: "bit slice extends past payload end",
        61: "code ran past block boundary",
        62: "bit pattern outside Huffman code space",
        63: f"block consumed {info.a} bits, expected {info.b}",
        64: f"block {b} decoded {info.a} unpredictable markers, record says {info.b}",
        65: "empty block with nonzero bit length",
    }
    if k == 66:
        return f"block {b} mismatches after re-execution"
    return f"block {b} undecodable: {why.get(k, str(k))}"


EB_MODES = {"absolute": 0, "value_range_relative": 1}


def _cfg(cfg: dict | None) -> Config:
    c = dict(protect_input=True, protect_bins=True, duplicate_eval=True, store_sum_dc=True,
             block_edge=10, codec_id=0, bin_capacity=65536)
    if cfg:
        c.update(cfg)
    return Config(int(c["protect_input"]), int(c["protect_bins"]), int(c["duplicate_eval"]),
                  int(c["store_sum_dc"]), int(c["block_edge"]), int(c["codec_id"]),
                  int(c["bin_capacity"]), 0)


def _faults(faults):
    faults = list(faults or [])
    arr = (Fault * max(1, len(faults)))()
    for i, (target, block, element, bit) in enumerate(faults):
        arr[i] = Fault(TARGETS[target] if isinstance(target, str) else int(target), int(bit),
                       int(block), int(element))
    return arr, len(faults)


def _report(nb_cap: int):
    bufs = [np.zeros(max(1, nb_cap), np.int64) for _ in range(4)]
    r = Report()
    r.capacity = nb_cap
    r.input_corrected, r.bins_corrected, r.dup_mismatch, r.reexecuted = (
        b.ctypes.data_as(_P64) for b in bufs)
    return r, bufs


def _lists(r: Report, bufs) -> dict:
    ns = [r.n_input_corrected, r.n_bins_corrected, r.n_dup_mismatch, r.n_reexecuted]
    keys = ["input_corrected", "bins_corrected", "dup_mismatch_resolved", "decomp_block_reexecuted"]
    return {k: [int(v) for v in b[:n]] for k, b, n in zip(keys, bufs, ns)}


def _status_of(lists: dict, sdc: bool) -> str:
    if sdc:
        return "sdc_in_compression"
    return "corrected" if any(lists.values()) else "clean"


def compress(values: np.ndarray, mode: str, value: float, cfg: dict | None = None,
             faults=None, override=None, threads: int = 1):
    """-> (archive bytes, report dict).  Raises OracleError like the reference raises."""
    x = np.ascontiguousarray(values, dtype=np.float32)
    if x.ndim != 3:
        raise OracleError("InvalidGeometry", f"expected 3 dimensions, got {x.ndim}")
    nx, ny, nz = x.shape
    e = (cfg or {}).get("block_edge", 10)
    nb = -(-nx // e) * -(-ny // e) * -(-nz // e) if e >= 1 else 1
    fa, nf = _faults(faults)
    ov = None
    if override:
        ov = np.full(nb, -1, np.int8)
        for b, k in override.items():
            ov[int(b)] = int(k)
    rep, bufs = _report(nb)
    out = C.c_void_p()
    n = C.c_size_t()
    st = lib().oc_compress(x.ctypes.data, nx, ny, nz, EB_MODES[mode], float(value),
                           C.byref(_cfg(cfg)), fa, nf,
                           ov.ctypes.data if ov is not None else None, int(threads),
                           C.byref(out), C.byref(n), C.byref(rep))
    if st != 0:
        raise_for(st, rep.info, eb_request=(mode, float(value), rep.eb))
    data = C.string_at(out, n.value)
    lib().oc_free(out)
    lists = _lists(rep, bufs)
    lists["decomp_block_reexecuted"] = []
    report = {"status": _status_of(lists, False), **lists, "detail": "",
              "eb": rep.eb, "n_regression": rep.n_regression,
              "n_unpredictable": rep.n_unpredictable, "n_symbols": rep.n_symbols,
              "payload_bits": rep.payload_bits, "max_code_len": rep.max_code_len}
    return data, report


def parse_check(data: bytes) -> StreamInfo:
    """Validate like container.parse; raises OracleError(CorruptStream/UnsupportedCodec)."""
    si = StreamInfo()
    info = Info()
    buf = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
    st = lib().oc_parse(buf.ctypes.data, len(data), C.byref(si), C.byref(info))
    raise_for(st, info, data)
    return si


def decompress(data: bytes, faults=None, threads: int = 1):
    """-> (float32 array or None, report dict).  Parse errors raise OracleError."""
    si = parse_check(data)
    h = si.hdr
    out = np.empty((h.nx, h.ny, h.nz), np.float32)
    fa, nf = _faults(faults)
    rep, bufs = _report(int(h.block_count))
    buf = np.frombuffer(data, np.uint8)
    st = lib().oc_decompress(buf.ctypes.data, len(data), out.ctypes.data, fa, nf, int(threads),
                             C.byref(rep))
    raise_for(st, rep.info, data)
    lists = _lists(rep, bufs)
    lists["input_corrected"] = []
    lists["bins_corrected"] = []
    lists["dup_mismatch_resolved"] = []
    sdc = bool(rep.sdc)
    report = {"status": _status_of(lists, sdc), **lists,
              "detail": sdc_detail(rep.info) if sdc else ""}
    return (None if sdc else out), report


def rle_apply(data: bytes) -> bytes:
    """Backend codec 1 apply (encode.py:287-299)."""
    data = bytes(data)
    out = (C.c_uint8 * (2 * len(data) + 2))()
    n = lib().oc_rle_apply(data or b"\x00", len(data), out)
    return bytes(memoryview(out)[:n])


def rle_invert(data: bytes) -> bytes:
    """Backend codec 1 invert (encode.py:300-311); OracleError like the reference."""
    data = bytes(data)
    n = lib().oc_rle_invert(data or b"\x00", len(data), None)
    if n == -1:
        raise OracleError("CorruptStream", "run-length stream has odd length")
    if n == -2:
        raise OracleError("CorruptStream", "run-length stream has zero-length run")
    out = (C.c_uint8 * max(1, n))()
    lib().oc_rle_invert(data or b"\x00", len(data), out)
    return bytes(memoryview(out)[:n])
