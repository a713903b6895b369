"""Seeded synthetic stand-ins for the BASELINE.json configs.

BASELINE.json names no public dataset; the paper's NYX / Hurricane / SCALE-LETKF fields are
not available here, so these generators produce fields of the named shapes and spectra.
All fields are built in float64 with numpy and cast to float32 once, so the bytes are
identical on every machine running the same numpy (the image pins numpy 2.3.5).

    c1  64^3  sum of 8 random sines + N(0, 1e-3)           rel 1e-3
    c2  100x500x500 Gaussian random field, P(k) ~ k^-3     rel 1e-2 and 1e-4
    c3  512^3 lognormal exp(GRF), P(k) ~ k^-2.5, std 1     rel 1e-3
    c4  1x1800x3600 latitude bands + 2D GRF (k^-3, std 5)  rel 1e-4
    c5  = c2 at rel 1e-3 with seeded 1% single-bit flips (fault_plan)
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

CONFIGS = {
    "c1": {"dims": (64, 64, 64), "eb": ("value_range_relative", 1e-3)},
    "c2": {"dims": (100, 500, 500), "eb": ("value_range_relative", 1e-2)},
    "c2_1e-4": {"dims": (100, 500, 500), "eb": ("value_range_relative", 1e-4)},
    "c3": {"dims": (512, 512, 512), "eb": ("value_range_relative", 1e-3)},
    "c4": {"dims": (1, 1800, 3600), "eb": ("value_range_relative", 1e-4)},
    "c5": {"dims": (100, 500, 500), "eb": ("value_range_relative", 1e-3)},
}


def c1() -> np.ndarray:
    rng = np.random.default_rng(0)
    shape = (64, 64, 64)
    x = np.indices(shape).reshape(3, -1).T.astype(np.float64)
    f = np.zeros(x.shape[0])
    for _ in range(8):
        a = rng.uniform(0.5, 1.0)
        n = rng.integers(1, 5, size=3)
        phi = rng.uniform(0.0, 2.0 * math.pi)
        f += a * np.sin(2.0 * math.pi * (x @ n) / 64.0 + phi)
    f += rng.normal(0.0, 1e-3, x.shape[0])
    return f.reshape(shape).astype(np.float32)


def grf(shape, alpha: float, seed: int, std: float = 1.0) -> np.ndarray:
    """Gaussian random field with isotropic power spectrum P(k) ~ |k|^-alpha."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal(shape)
    F = np.fft.rfftn(w)
    del w
    k2 = None
    for ax, n in enumerate(shape):
        f = np.fft.rfftfreq(n) if ax == len(shape) - 1 else np.fft.fftfreq(n)
        sh = [1] * len(shape)
        sh[ax] = f.size
        t = (f ** 2).reshape(sh)
        k2 = t if k2 is None else k2 + t
    with np.errstate(divide="ignore"):
        amp = np.where(k2 > 0, k2 ** (-alpha / 4.0), 0.0)  # |k|^(-alpha/2)
    F *= amp
    del amp, k2
    g = np.fft.irfftn(F, s=shape)
    del F
    g = (g - g.mean()) / g.std() * std
    return g


def c2() -> np.ndarray:
    return grf((100, 500, 500), 3.0, 2).astype(np.float32)


def c3() -> np.ndarray:
    return np.exp(grf((512, 512, 512), 2.5, 3)).astype(np.float32)


def c4() -> np.ndarray:
    rows = np.arange(1800, dtype=np.float64)
    bands = 250.0 + 40.0 * np.cos(2.0 * math.pi * rows / 1800.0 * 3.0)
    f = bands[:, None] + grf((1800, 3600), 3.0, 4, std=5.0)
    return f.reshape(1, 1800, 3600).astype(np.float32)


def field(name: str) -> np.ndarray:
    base = name.split("_")[0]
    return {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c2}[base]()


def fault_plan(nb: int, volumes, seed: int = 12345, frac: float = 0.01):
    """c5 plan: sorted 1% of blocks, one element per block, bits 0..31."""
    rng = np.random.default_rng(seed)
    k = int(math.ceil(frac * nb))
    blocks = np.sort(rng.choice(nb, k, replace=False))
    elems = [int(rng.integers(int(volumes[b]))) for b in blocks]
    bits = rng.integers(0, 32, size=len(blocks))
    return [(int(b), int(e), int(t)) for b, e, t in zip(blocks, elems, bits)]


def block_volumes(dims, edge: int = 10) -> np.ndarray:
    nx, ny, nz = dims
    ex = [np.minimum(edge, n - np.arange(0, n, edge)) for n in (nx, ny, nz)]
    return (ex[0][:, None, None] * ex[1][None, :, None] * ex[2][None, None, :]).reshape(-1)


def sha256(buf) -> str:
    return hashlib.sha256(memoryview(buf).cast("B")).hexdigest()
