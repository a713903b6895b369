"""Quantizer geometry of the drop-in API (reference quantize.py:21-34)."""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidArgument


@dataclass(frozen=True)
class QuantConfig:
    """bin_capacity must be a power of two >= 4 (device path: <= 65536)."""

    bin_capacity: int = 65536

    def __post_init__(self):
        c = self.bin_capacity
        if c < 4 or (c & (c - 1)) != 0:
            raise InvalidArgument(f"bin_capacity must be a power of two >= 4, got {c}")

    @property
    def center(self) -> int:
        return self.bin_capacity // 2
