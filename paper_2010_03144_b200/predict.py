"""Predictor identifiers of the drop-in API (reference predict.py:17-40).  The predictors
themselves run on the device (csrc/compress.cu, csrc/decompress.cu)."""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

SAMPLE_STRIDE = 8


class PredictorKind(enum.IntEnum):
    LORENZO = 0
    REGRESSION = 1


@dataclass(frozen=True)
class RegressionCoeffs:
    """pred(i,j,k) = b0 + b1*i + b2*j + b3*k over local block coordinates."""

    b0: np.float32
    b1: np.float32
    b2: np.float32
    b3: np.float32

    @classmethod
    def from_array(cls, arr) -> "RegressionCoeffs":
        a = np.asarray(arr, dtype=np.float32)
        return cls(a[0], a[1], a[2], a[3])

    def as_array(self) -> np.ndarray:
        return np.array([self.b0, self.b1, self.b2, self.b3], dtype=np.float32)
