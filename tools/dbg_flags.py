import sys, numpy as np
sys.path.insert(0, ".")
import paper_2010_03144_b200 as F
from oracle import oracle as O
rng = np.random.default_rng(1)
for dims in [(1,10,24),(1,10,30),(1,10,40)]:
    x = (np.cumsum(rng.standard_normal(dims), axis=2)*0.1).astype(np.float32)
    nb = -(-dims[2]//10)
    for ov in [{1:1}, {2:1}, {0:1,1:1}, {nb-1:1}]:
        ov = {k:v for k,v in ov.items() if k < nb}
        full = {i:0 for i in range(nb)}; full.update(ov)
        s,_ = F.compress(F.Field.from_array(x), F.ErrorBound.absolute(1e-3), predictor_override=full)
        want, rep = O.compress(x, "absolute", 1e-3, None, override=full)
        print(dims, full, F.serialize(s) == want)
