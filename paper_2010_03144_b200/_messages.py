"""Map ftlz_info (status, kind, offset, operands) to the reference exceptions and texts
(errors.py:4-59; core.py:188-192; pipeline.py:343,477,490,565-577,673-707;
encode.py:85-88,206-255,297-312; container.py:155-285)."""

from __future__ import annotations

import numpy as np

from . import errors as E

_FIELDS = ["header", "block indicator", "regression coefficients", "block record",
           "codebook size", "codebook entry", "payload length", "payload",
           "unpredictable words", "checksum section lengths", "checksum section"]


def _corrupt(info, data: bytes) -> E.CorruptStream:
    k, off = info.kind, info.offset
    if k == 20:
        msg = f"truncated while reading {_FIELDS[info.a]}"
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
    elif k == 40:
        return E.CorruptStream("run-length stream has odd length")
    elif k == 41:
        return E.CorruptStream("run-length stream has zero-length run")
    else:
        msg = f"malformed archive (kind {k})"
    return E.CorruptStream(msg, offset=off)


def raise_for_info(status: int, info, data: bytes = b"", eb_request=None, resolved=None):
    """Raise the reference exception for a non-OK library status."""
    from . import _lib

    if status == 0:
        return
    if status == 1:
        raise E.InvalidGeometry(_lib.last_error() or "invalid geometry")
    if status == 2:
        mode, value = eb_request
        raise E.DegenerateBound(f"resolved bound {resolved} is not positive and finite "
                                f"(mode={mode}, value={value})")
    if status == 3:
        if info.kind == 1:
            raise E.UncorrectableCorruption(
                f"input block {info.block} failed verification beyond repair")
        tag = "histogram" if info.kind == 2 else "encode"
        raise E.UncorrectableCorruption(
            f"bin array of block {info.block} failed verification beyond repair ({tag})")
    if status == 4:
        if info.kind == 4:
            raise E.InternalInvariantViolation("bin index outside quantizer range")
        raise E.InternalInvariantViolation(f"code length {info.a} exceeds cap 57")
    if status == 5:
        raise _corrupt(info, data)
    if status == 6:
        raise E.UnsupportedCodec(f"codec {info.a} is not registered")
    if status == 7:
        raise E.InvalidArgument(_lib.last_error())
    if status == 9:
        raise E.InvalidArgument("capacity: " + _lib.last_error())
    if status == 10:
        raise E.InvalidRegion(_lib.last_error())
    raise E.DeviceError(_lib.last_error())


def sdc_detail(info, region: bool = False) -> str:
    """The reference's SDC detail text.  decompress (pipeline.py:673-677) prefixes decoder
    failures with "block {b} undecodable: "; decompress_region (pipeline.py:788-793) reports
    the decoder's own message."""
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
    if region:
        return why.get(k, str(k))
    return f"block {b} undecodable: {why.get(k, str(k))}"
