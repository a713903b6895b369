"""Quick GPU sanity check: one small compress/decompress vs the oracle."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2010_03144_b200 as F
from oracle import oracle as O
rng = np.random.default_rng(0)
x = (np.sin(np.arange(24*20*22).reshape(24,20,22)*0.01) + 0.01*rng.standard_normal((24,20,22))).astype(np.float32)
t = time.time()
got = F.compress_bytes(x, "absolute", 1e-3)
print("compress ok", len(got), time.time() - t, flush=True)
want, _ = O.compress(x, "absolute", 1e-3)
print("archive equal:", got == want, len(want), flush=True)
if got != want:
    a = np.frombuffer(got[:len(want)], np.uint8); b = np.frombuffer(want[:len(got)], np.uint8)
    d = np.flatnonzero(a != b); print("first diffs", d[:10])
out = F.decompress_bytes(want)
ref, _ = O.decompress(want)
print("decompress equal:", np.array_equal(out.view(np.uint32), ref.view(np.uint32)), flush=True)
