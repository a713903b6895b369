"""ctypes binding of libftlz_b200.so (include/ftlz_b200.h).

The shared library is the product: every compress / parse / decompress call of this package
goes through it.  There is no CPU fallback -- if the library or a CUDA device is missing the
first call raises :class:`BackendUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# FTLZ_LIB_PATH points at another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("FTLZ_LIB_PATH") or os.path.join(_HERE, "lib", "libftlz_b200.so")


class BackendUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is not available."""


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


# every symbol the header declares; tests check the library exports all of them
EXPORTS = [
    "ftlz_abi_version", "ftlz_last_error", "ftlz_default_config", "ftlz_peek_header", "ftlz_peek_archive",
    "ftlz_block_count", "ftlz_compress_workspace_size", "ftlz_compress_bound", "ftlz_compress",
    "ftlz_decompress_workspace_size", "ftlz_parse", "ftlz_decompress", "ftlz_ctx_create",
    "ftlz_ctx_destroy", "ftlz_ctx_stream", "ftlz_ctx_compress_device", "ftlz_ctx_compress_host",
    "ftlz_ctx_archive_device", "ftlz_ctx_archive_host", "ftlz_ctx_copy_archive",
    "ftlz_ctx_parse_host", "ftlz_ctx_decompress_host", "ftlz_ctx_decompress_device",
    "ftlz_ctx_profile", "ftlz_ctx_profile_read", "ftlz_ctx_decompress_region_host",
    "ftlz_intersecting_block_count", "ftlz_ctx_rle_host", "ftlz_ctx_compress_host_to",
]

_lib = None
_lock = threading.Lock()


def load():
    """Load the shared library and declare signatures (no device access)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise BackendUnavailable(
                f"{LIB_PATH} is missing: build it with `make -C paper_2010_03144_b200` "
                "(nvcc, sm_100a); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, sz, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t, C.c_double
        PR = C.POINTER(Report)
        PC = C.POINTER(Config)
        PF = C.POINTER(Fault)
        PH = C.POINTER(Header)
        L.ftlz_abi_version.restype = C.c_int
        L.ftlz_last_error.restype = C.c_char_p
        L.ftlz_default_config.argtypes = [PC]
        L.ftlz_peek_header.argtypes = [vp, sz, PH, C.POINTER(Info)]
        L.ftlz_peek_archive.argtypes = [vp, sz, PH, C.POINTER(Info)]
        L.ftlz_block_count.argtypes = [i64, i64, i64, i32]
        L.ftlz_block_count.restype = i64
        L.ftlz_compress_workspace_size.argtypes = [i64, i64, i64, PC]
        L.ftlz_compress_workspace_size.restype = sz
        L.ftlz_compress_bound.argtypes = [i64, i64, i64, PC]
        L.ftlz_compress_bound.restype = sz
        L.ftlz_compress.argtypes = [vp, i64, i64, i64, i32, dbl, PC, PF, i64, vp, vp, sz, vp, sz, PR, vp]
        L.ftlz_decompress_workspace_size.argtypes = [PH, sz]
        L.ftlz_decompress_workspace_size.restype = sz
        L.ftlz_parse.argtypes = [vp, sz, PH, vp, sz, C.POINTER(StreamInfo), PR, vp]
        L.ftlz_decompress.argtypes = [vp, sz, PH, vp, PF, i64, vp, sz, PR, vp]
        L.ftlz_ctx_create.argtypes = [i32]
        L.ftlz_ctx_create.restype = vp
        L.ftlz_ctx_destroy.argtypes = [vp]
        L.ftlz_ctx_stream.argtypes = [vp]
        L.ftlz_ctx_stream.restype = vp
        L.ftlz_ctx_compress_device.argtypes = [vp, vp, i64, i64, i64, i32, dbl, PC, PF, i64, vp, PR]
        L.ftlz_ctx_compress_host.argtypes = [vp, vp, i64, i64, i64, i32, dbl, PC, PF, i64, vp, PR]
        L.ftlz_ctx_compress_host_to.argtypes = [vp, vp, i64, i64, i64, i32, dbl, PC, PF, i64, vp, vp, sz, PR]
        L.ftlz_ctx_archive_device.argtypes = [vp, C.POINTER(vp), C.POINTER(sz)]
        L.ftlz_ctx_archive_host.argtypes = [vp, C.POINTER(vp), C.POINTER(sz)]
        L.ftlz_ctx_copy_archive.argtypes = [vp, vp, sz]
        L.ftlz_ctx_parse_host.argtypes = [vp, vp, sz, C.POINTER(StreamInfo), PR]
        L.ftlz_ctx_decompress_host.argtypes = [vp, vp, sz, vp, PF, i64, i32, PR]
        L.ftlz_ctx_decompress_device.argtypes = [vp, vp, sz, PH, vp, PF, i64, PR]
        L.ftlz_ctx_decompress_region_host.argtypes = [vp, vp, sz, vp, vp, i32, PR]
        L.ftlz_intersecting_block_count.argtypes = [i64, i64, i64, i32, vp]
        L.ftlz_intersecting_block_count.restype = i64
        L.ftlz_ctx_rle_host.argtypes = [vp, vp, sz, i32, vp, sz, C.POINTER(sz), C.POINTER(Info)]
        L.ftlz_ctx_profile.argtypes = [vp, i32]
        L.ftlz_ctx_profile_read.argtypes = [vp, C.c_char_p, sz, C.POINTER(dbl), C.POINTER(i64), i32]
        _lib = L
        return L


_tls = threading.local()


_free = []                 # (device, handle) of contexts released by finished threads
_free_lock = threading.Lock()


class _Context:
    """A library context (stream + device workspaces) owned by one thread.  When the thread
    ends, the context goes back to a process-wide pool and the next new thread takes it over
    with its workspaces already allocated."""

    __slots__ = ("handle", "device")

    def __init__(self, device: int):
        self.device = device
        with _free_lock:
            for i, (d, h) in enumerate(_free):
                if d == device:
                    self.handle = _free.pop(i)[1]
                    return
        L = load()
        h = L.ftlz_ctx_create(device)
        if not h:
            raise BackendUnavailable(
                "no usable CUDA device for the B200 path: " + L.ftlz_last_error().decode(errors="replace"))
        self.handle = h

    def __del__(self):
        if not sys.is_finalizing():
            with _free_lock:
                _free.append((self.device, self.handle))


def context(device: int = 0):
    """The calling thread's library context for `device` (created on first use, or taken over
    from a finished thread).  Each thread owns its stream and workspaces, so threads run
    compress / decompress calls concurrently (e.g. one thread uploading and compressing the
    next field while another decompresses and downloads the previous archive)."""
    m = getattr(_tls, "ctx", None)
    if m is None:
        m = _tls.ctx = {}
    c = m.get(device)
    if c is None:
        c = m[device] = _Context(device)
    return c.handle


def last_parse() -> object:
    """Token of the archive this thread's context most recently validated on the device."""
    return getattr(_tls, "last_parse", None)


def set_last_parse(token: object) -> None:
    _tls.last_parse = token


def last_error() -> str:
    return load().ftlz_last_error().decode(errors="replace")


def profile(enable: bool, device: int = 0) -> None:
    """Enable per-kernel CUDA-event timing in the library context (resets totals)."""
    load().ftlz_ctx_profile(context(device), 1 if enable else 0)


def profile_read(device: int = 0) -> dict:
    """{kernel: (total_ms, launches)} accumulated since profile(True)."""
    L = load()
    names = C.create_string_buffer(8192)
    ms = (C.c_double * 64)()
    cnt = (C.c_int64 * 64)()
    n = L.ftlz_ctx_profile_read(context(device), names, 8192, ms, cnt, 64)
    keys = names.value.decode().split("\n")[:max(n, 0)]
    return {k: (ms[i], int(cnt[i])) for i, k in enumerate(keys)}
