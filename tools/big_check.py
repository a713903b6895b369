"""Robustness check beyond 2^31 bytes: a 1024x1024x640 field (2.7 GB) through the device path,
compared with the C oracle (OpenMP) byte for byte.  Usage (GPU box): python tools/big_check.py"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03144_b200 as F
from oracle import oracle as O

nx, ny, nz = 640, 1024, 1024
i = np.arange(nx, dtype=np.float32)[:, None, None]
j = np.arange(ny, dtype=np.float32)[None, :, None]
k = np.arange(nz, dtype=np.float32)[None, None, :]
x = (np.sin(i / 37.0) * np.cos(j / 23.0) + np.sin(k / 29.0)).astype(np.float32)
x += np.random.default_rng(1).standard_normal(x.shape, dtype=np.float32) * np.float32(1e-3)
print("field", x.shape, x.nbytes / 2**30, "GiB", flush=True)
t = time.time()
arc = F.compress_bytes(x, "value_range_relative", 1e-3)
y = F.decompress_bytes(arc)
print("device round trip", round(time.time() - t, 2), "s, archive", len(arc), flush=True)
t = time.time()
ref, _ = O.compress(x, "value_range_relative", 1e-3)
print("oracle compress", round(time.time() - t, 2), "s", flush=True)
print("archive identical:", bytes(arc) == ref)
yr, _ = O.decompress(ref)
print("output identical:", np.array_equal(y.view(np.uint32), yr.view(np.uint32)))
eb = (float(x.max()) - float(x.min())) * 1e-3
print("max err <= eb:", float(np.max(np.abs(y.astype(np.float64) - x))) <= eb)
