"""Field, error bounds and block geometry of the drop-in API (reference core.py:29-193).

Geometry here is host bookkeeping only (block ids, extents, cell <-> block maps used by
fault plans and reports); all per-point arithmetic runs on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import DegenerateBound, InvalidGeometry

Dims = tuple

BLOCK_EDGE_MIN = 2
BLOCK_EDGE_MAX = 64
DEFAULT_BLOCK_EDGE = 10

EB_ABSOLUTE = "absolute"
EB_RELATIVE = "value_range_relative"
EB_MODE_CODES = {EB_ABSOLUTE: 0, EB_RELATIVE: 1}
EB_MODE_NAMES = {v: k for k, v in EB_MODE_CODES.items()}


def _check_dims(dims):
    if len(dims) != 3:
        raise InvalidGeometry(f"expected 3 dimensions, got {len(dims)}")
    nx, ny, nz = (int(d) for d in dims)
    if nx < 1 or ny < 1 or nz < 1:
        raise InvalidGeometry(f"all dimensions must be >= 1, got {(nx, ny, nz)}")
    return (nx, ny, nz)


@dataclass(frozen=True)
class Field:
    """Dense 3D float32 field (row-major). `values` is read-only (core.py:38-74)."""

    dims: tuple
    values: np.ndarray

    @classmethod
    def from_array(cls, arr: np.ndarray) -> "Field":
        dims = _check_dims(np.shape(arr))
        vals = np.ascontiguousarray(arr, dtype=np.float32)
        if vals is arr:
            vals = arr.copy()
        vals.flags.writeable = False
        return cls(dims, vals)

    @classmethod
    def from_flat(cls, flat, dims) -> "Field":
        dims = _check_dims(dims)
        vals = np.asarray(flat, dtype=np.float32)
        if vals.size != dims[0] * dims[1] * dims[2]:
            raise InvalidGeometry(f"value count {vals.size} does not match dims {dims}")
        return cls.from_array(vals.reshape(dims))

    @classmethod
    def _wrap(cls, arr: np.ndarray) -> "Field":
        """Adopt a freshly produced array without a copy (decompression output)."""
        arr.flags.writeable = False
        return cls(tuple(int(d) for d in arr.shape), arr)

    @property
    def size(self) -> int:
        return self.values.size

    @property
    def nbytes(self) -> int:
        return self.values.size * 4

    def value_range(self) -> float:
        v = self.values
        return float(v.max()) - float(v.min())


@dataclass(frozen=True, slots=True)
class BlockSpec:
    block_index: int
    origin: tuple
    extent: tuple

    @property
    def volume(self) -> int:
        bx, by, bz = self.extent
        return bx * by * bz

    def slices(self):
        (i0, j0, k0), (bx, by, bz) = self.origin, self.extent
        return (slice(i0, i0 + bx), slice(j0, j0 + by), slice(k0, k0 + bz))


class BlockGrid:
    """Row-major block tiling (core.py:95-130).  Block specs are computed on demand so the
    512^3 grid (140,608 blocks) costs nothing until a caller asks for one."""

    def __init__(self, field_dims, block_edge):
        self.field_dims = tuple(field_dims)
        self.block_edge = int(block_edge)
        e = self.block_edge
        nx, ny, nz = self.field_dims
        self.counts = (-(-nx // e), -(-ny // e), -(-nz // e))

    @property
    def n_blocks(self) -> int:
        cx, cy, cz = self.counts
        return cx * cy * cz

    def spec(self, b: int) -> BlockSpec:
        cx, cy, cz = self.counts
        if not 0 <= b < cx * cy * cz:
            raise IndexError(b)
        e = self.block_edge
        bk = b % cz
        t = b // cz
        bj, bi = t % cy, t // cy
        org = (bi * e, bj * e, bk * e)
        ext = tuple(min(e, n - o) for n, o in zip(self.field_dims, org))
        return BlockSpec(int(b), org, ext)

    @property
    def blocks(self):
        return _BlockList(self)

    def block_of_cell(self, i, j, k):
        e = self.block_edge
        cx, cy, cz = self.counts
        index = ((i // e) * cy + (j // e)) * cz + (k // e)
        s = self.spec(index)
        li, lj, lk = i - s.origin[0], j - s.origin[1], k - s.origin[2]
        _, by, bz = s.extent
        return index, (li * by + lj) * bz + lk

    def cell_of_block(self, block_index, offset):
        s = self.spec(block_index)
        _, by, bz = s.extent
        li, rem = divmod(offset, by * bz)
        lj, lk = divmod(rem, bz)
        return (s.origin[0] + li, s.origin[1] + lj, s.origin[2] + lk)

    def extents(self) -> np.ndarray:
        """(n_blocks, 3) extents, vectorised."""
        e = self.block_edge
        ex = [np.minimum(e, n - np.arange(0, n, e)) for n in self.field_dims]
        g = np.stack(np.meshgrid(*ex, indexing="ij"), axis=-1)
        return g.reshape(-1, 3)


class _BlockList:
    def __init__(self, grid):
        self._g = grid

    def __len__(self):
        return self._g.n_blocks

    def __getitem__(self, b):
        if isinstance(b, slice):
            return [self._g.spec(i) for i in range(*b.indices(len(self)))]
        if b < 0:
            b += len(self)
        return self._g.spec(b)

    def __iter__(self):
        for b in range(len(self)):
            yield self._g.spec(b)


def partition(dims, block_edge: int = DEFAULT_BLOCK_EDGE) -> BlockGrid:
    """Row-major tiling of `dims` (core.py:133-157)."""
    dims = _check_dims(dims)
    block_edge = int(block_edge)
    if not (BLOCK_EDGE_MIN <= block_edge <= BLOCK_EDGE_MAX):
        raise InvalidGeometry(
            f"block_edge must be in [{BLOCK_EDGE_MIN}, {BLOCK_EDGE_MAX}], got {block_edge}")
    return BlockGrid(dims, block_edge)


@dataclass(frozen=True)
class ErrorBound:
    """Absolute, or relative to the value range (core.py:160-179)."""

    mode: str
    value: float

    def __post_init__(self):
        if self.mode not in (EB_ABSOLUTE, EB_RELATIVE):
            raise DegenerateBound(f"unknown error-bound mode {self.mode!r}")
        if not (self.value > 0.0) or not math.isfinite(self.value):
            raise DegenerateBound(f"error-bound value must be > 0, got {self.value}")

    @classmethod
    def absolute(cls, value: float) -> "ErrorBound":
        return cls(EB_ABSOLUTE, float(value))

    @classmethod
    def relative(cls, value: float) -> "ErrorBound":
        return cls(EB_RELATIVE, float(value))


def resolve_error_bound(spec: ErrorBound, field: Field) -> float:
    """Host utility mirroring core.py:182-193 (compression resolves on the device)."""
    resolved = spec.value if spec.mode == EB_ABSOLUTE else spec.value * field.value_range()
    if not (resolved > 0.0) or not math.isfinite(resolved):
        raise DegenerateBound(
            f"resolved bound {resolved} is not positive and finite "
            f"(mode={spec.mode}, value={spec.value})")
    return float(resolved)
