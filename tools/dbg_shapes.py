import sys, numpy as np
sys.path.insert(0, ".")
import paper_2010_03144_b200 as F
from oracle import oracle as O
rng = np.random.default_rng(1)
for dims in [(1,32,24),(1,10,24),(1,32,10),(1,10,10),(2,32,24),(1,20,20),(1,32,30),(1,32,40),(3,32,24),(10,10,24)]:
    x = (np.cumsum(rng.standard_normal(dims), axis=2)*0.1).astype(np.float32)
    try:
        got = F.compress_bytes(x, "absolute", 1e-3)
        want, _ = O.compress(x, "absolute", 1e-3)
        print(dims, "ok" if got == want else "MISMATCH", flush=True)
    except Exception as e:
        print(dims, "ERR", type(e).__name__, e, flush=True)
