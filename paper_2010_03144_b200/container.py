"""Archive container of the drop-in API (reference container.py:1-285).

`compress` on the device already emits the serialized archive, so a CompressedStream made
by this package wraps those bytes and materialises `records`, `code_lengths`, `payload` and
`unpred_words` only when a caller reads them.  `serialize` of such a stream returns the
device bytes untouched; a stream built or modified field-by-field (e.g. with
`dataclasses.replace`) is serialized from its fields in the reference byte layout.
`parse` validates on the device (records, codebook, sections) and raises the reference
exceptions with the reference offsets.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .core import EB_MODE_CODES, EB_MODE_NAMES
from .errors import UnsupportedCodec
from ._messages import raise_for_info

MAGIC = b"FTLZ"
VERSION = 1
_HEADER = struct.Struct("<4sBBQQQIBdIQ")
_LAZY_FIELDS = ("records", "code_lengths", "payload", "unpred_words")


class _Lazy:
    __slots__ = ()

    def __repr__(self):
        return "<lazy>"


_LAZY = _Lazy()


@dataclass(frozen=True)
class BlockRecord:
    """Per-block metadata (container.py:57-71)."""

    predictor: int
    coeff_bytes: Optional[bytes]
    unpred_count: int
    bit_length: int
    sum_dc: Optional[int]

    def coeffs(self):
        from .predict import RegressionCoeffs

        if self.coeff_bytes is None:
            return None
        return RegressionCoeffs.from_array(np.frombuffer(self.coeff_bytes, "<f4"))


@dataclass(frozen=True)
class CompressedStream:
    """In-memory form of an archive (container.py:74-106)."""

    dims: tuple
    block_edge: int
    eb_mode: str
    eb_value: float
    codec_id: int
    bin_capacity: int
    records: tuple
    code_lengths: dict
    payload: bytes
    unpred_words: bytes
    stored_size: Optional[int] = field(default=None, compare=False)

    # ---------------------------------------------------------------- lazy materialisation
    def __getattribute__(self, name):
        v = object.__getattribute__(self, name)
        if v is _LAZY:
            object.__getattribute__(self, "_materialize")()
            v = object.__getattribute__(self, name)
        return v

    @classmethod
    def _from_archive(cls, data: bytes, sections: dict) -> "CompressedStream":
        (_, _, codec, nx, ny, nz, edge, mode, eb, cap, _nb) = _HEADER.unpack_from(data, 0)
        s = cls((nx, ny, nz), edge, EB_MODE_NAMES[mode], eb, codec, cap, _LAZY, _LAZY, _LAZY, _LAZY,
                stored_size=len(data))
        object.__setattr__(s, "_archive", data)
        object.__setattr__(s, "_sections", sections)
        return s

    def _materialize(self):
        data = object.__getattribute__(self, "_archive")
        sec = object.__getattribute__(self, "_sections")
        if sec is None:   # codec 1 straight from compress: section map from a device parse
            sec = _parse_sections(data)
            object.__setattr__(self, "_sections", sec)
        nb = (-(-self.dims[0] // self.block_edge) * -(-self.dims[1] // self.block_edge)
              * -(-self.dims[2] // self.block_edge))
        mv = memoryview(data)
        pos = 55
        recs = []
        has = sec["has_sum_dc"]
        c1 = object.__getattribute__(self, "codec_id") == 1
        if has and c1:   # stored as run-length pairs
            so = sec["sumdc_off"]
            sums = np.frombuffer(rle_invert(mv[so:so + sec["sumdc_stored_len"]]), "<u8", nb)
        else:
            sums = (np.frombuffer(data, "<u8", nb, sec["sumdc_off"]) if has else None)
        unpack_tail = struct.Struct("<II").unpack_from
        for b in range(nb):
            ind = data[pos]
            pos += 1
            coef = None
            if ind:
                coef = bytes(mv[pos:pos + 16])
                pos += 16
            uc, bl = unpack_tail(data, pos)
            pos += 8
            recs.append(BlockRecord(ind, coef, uc, bl, int(sums[b]) if has else None))
        nsym = struct.unpack_from("<I", data, pos)[0]
        ent = np.frombuffer(data, np.uint8, 5 * nsym, pos + 4).reshape(nsym, 5)
        syms = ent[:, :4].copy().view("<u4").reshape(-1)
        lens = ent[:, 4]
        code_lengths = {int(s): int(l) for s, l in zip(syms, lens)}
        po, pl = sec["payload_off"], sec["payload_len"]
        uo, nu = sec["unpred_off"], sec["n_unpred"]
        object.__setattr__(self, "records", tuple(recs))
        object.__setattr__(self, "code_lengths", code_lengths)
        if c1:
            object.__setattr__(self, "payload", rle_invert(mv[po:po + sec["payload_stored_len"]]))
        else:
            object.__setattr__(self, "payload", bytes(mv[po:po + pl]))
        object.__setattr__(self, "unpred_words", bytes(mv[uo:uo + 4 * nu]))

    # ---------------------------------------------------------------- reference helpers
    def bit_offsets(self) -> list:
        offs = [0] * (len(self.records) + 1)
        for i, rec in enumerate(self.records):
            offs[i + 1] = offs[i] + rec.bit_length
        return offs

    def unpred_offsets(self) -> list:
        offs = [0] * (len(self.records) + 1)
        for i, rec in enumerate(self.records):
            offs[i + 1] = offs[i] + rec.unpred_count
        return offs

    def unpred_array(self) -> np.ndarray:
        return np.frombuffer(self.unpred_words, dtype="<u4")

    def has_sum_dc(self) -> bool:
        sec = self.__dict__.get("_sections")
        if sec is not None and self.__dict__.get("_archive") is not None:
            return bool(sec["has_sum_dc"])
        return bool(self.records) and self.records[0].sum_dc is not None


def _rle(data, invert: bool) -> bytes:
    """Backend codec 1 (encode.py:287-312) run on the device for host bytes."""
    data = bytes(data)
    L = _lib.load()
    ctx = _lib.context()
    cap = max(64, (4 if invert else 2) * len(data) + 64)
    buf = data if data else b"\x00"
    while True:
        out = (C.c_uint8 * cap)()
        n = C.c_size_t()
        info = _lib.Info()
        st = L.ftlz_ctx_rle_host(ctx, buf, len(data), int(invert), out, cap, C.byref(n), C.byref(info))
        if st == 9 and n.value > cap:
            cap = n.value + 64
            continue
        if st != 0:
            raise_for_info(st, info, data)
        return bytes(memoryview(out)[:n.value])


def rle_apply(data) -> bytes:
    return _rle(data, False)


def rle_invert(data) -> bytes:
    return _rle(data, True)


def _parse_sections(data: bytes) -> dict:
    L = _lib.load()
    si = _lib.StreamInfo()
    rep = _lib.Report()
    rep.capacity = 0
    st = L.ftlz_ctx_parse_host(_lib.context(), data, len(data), C.byref(si), C.byref(rep))
    if st != 0:
        raise_for_info(st, rep.info, data)
    return _sections_from_info(si)


def _sections_from_report(rep, nb: int, store_sum_dc: bool, codec_id: int = 0):
    if codec_id == 1:
        return None   # stored lengths are only in the archive: mapped on first access
    table = 9 * nb + 16 * rep.n_regression
    book = 55 + table
    pay_off = book + 4 + 5 * rep.n_symbols + 8
    pay_len = (rep.payload_bits + 7) // 8
    unp_off = pay_off + pay_len
    return {"payload_off": pay_off, "payload_len": pay_len, "unpred_off": unp_off,
            "n_unpred": rep.n_unpredictable, "has_sum_dc": store_sum_dc,
            "sumdc_off": unp_off + 4 * rep.n_unpredictable + 16,
            "payload_stored_len": pay_len, "sumdc_stored_len": 8 * nb if store_sum_dc else 0}


def _sections_from_info(si) -> dict:
    return {"payload_off": si.payload_off, "payload_len": si.payload_len,
            "unpred_off": si.unpred_off, "n_unpred": si.n_unpred,
            "has_sum_dc": bool(si.has_sum_dc), "sumdc_off": si.sumdc_off,
            "payload_stored_len": si.payload_stored_len, "sumdc_stored_len": si.sumdc_stored_len}


def serialize(stream: CompressedStream) -> bytes:
    """Archive bytes of a stream (container.py:109-147)."""
    data = stream.__dict__.get("_archive")
    if data is not None:
        return data
    if stream.codec_id not in (0, 1):
        raise UnsupportedCodec(f"codec {stream.codec_id} is not registered")
    code = rle_apply if stream.codec_id == 1 else bytes
    out = bytearray()
    out += _HEADER.pack(MAGIC, VERSION, stream.codec_id, stream.dims[0], stream.dims[1],
                        stream.dims[2], stream.block_edge, EB_MODE_CODES[stream.eb_mode],
                        stream.eb_value, stream.bin_capacity, len(stream.records))
    pack_tail = struct.Struct("<II").pack
    for rec in stream.records:
        out.append(rec.predictor)
        if rec.predictor == 1:
            assert rec.coeff_bytes is not None and len(rec.coeff_bytes) == 16
            out += rec.coeff_bytes
        out += pack_tail(rec.unpred_count, rec.bit_length)
    out += struct.pack("<I", len(stream.code_lengths))
    for sym in sorted(stream.code_lengths):
        out += struct.pack("<IB", sym, stream.code_lengths[sym])
    stored = code(stream.payload)
    out += struct.pack("<Q", len(stored))
    out += stored
    out += stream.unpred_words
    if stream.has_sum_dc():
        raw = b"".join(rec.sum_dc.to_bytes(8, "little") for rec in stream.records)
        stored = code(raw)
        out += struct.pack("<QQ", len(raw), len(stored))
        out += stored
    else:
        out += struct.pack("<QQ", 0, 0)
    return bytes(out)


def parse(data: bytes) -> CompressedStream:
    """Validate an archive on the device; raises CorruptStream(offset) like container.py:173-285."""
    data = bytes(data)
    L = _lib.load()
    ctx = _lib.context()
    si = _lib.StreamInfo()
    rep = _lib.Report()
    rep.capacity = 0
    buf = data if len(data) else b"\x00"
    st = L.ftlz_ctx_parse_host(ctx, buf, len(data), C.byref(si), C.byref(rep))
    if st != 0:
        raise_for_info(st, rep.info, data)
    stream = CompressedStream._from_archive(data, _sections_from_info(si))
    token = object()
    _lib.set_last_parse(token)
    object.__setattr__(stream, "_parse_token", token)
    return stream
