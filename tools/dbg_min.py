import sys, numpy as np
sys.path.insert(0, ".")
import paper_2010_03144_b200 as F
shape = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (20, 20, 20)
rng = np.random.default_rng(0)
i, j, k = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
x = (np.sin(i / 5.0) + np.cos(j / 4.0) * np.sin(k / 3.0)).astype(np.float32)
a = F.compress_bytes(x, "value_range_relative", 1e-3)
print("ok", len(a))
