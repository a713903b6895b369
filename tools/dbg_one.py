import sys, numpy as np
sys.path.insert(0, ".")
import paper_2010_03144_b200 as F
from oracle import oracle as O
rng = np.random.default_rng(1)
dims = tuple(int(v) for v in sys.argv[1:4])
x = (np.cumsum(rng.standard_normal(dims), axis=2)*0.1).astype(np.float32)
got = F.compress_bytes(x, "absolute", 1e-3)
want, rep = O.compress(x, "absolute", 1e-3)
print(len(got), len(want), rep)
a = np.frombuffer(got[:min(len(got),len(want))], np.uint8); b = np.frombuffer(want[:len(a)], np.uint8)
d = np.flatnonzero(a != b); print("diffs at", d[:20])
si = O.parse_check(want)
print("table", si.table_off, si.table_len, "book", si.book_off, "payload", si.payload_off, si.payload_len, "unp", si.unpred_off)
# per-block records
pos = 55
for blk in range(si.hdr.block_count):
    ind = want[pos]; n = 9 + 16*ind
    print(blk, "ind", ind, "want", want[pos:pos+n].hex(), "got", got[pos:pos+n].hex())
    pos += n
og, _ = O.decompress(got)
ow, _ = O.decompress(want)
diff = np.argwhere(og.view(np.uint32) != ow.view(np.uint32))
print("n diff points", len(diff), diff[:10].tolist())
print("max err got", np.max(np.abs(og.astype(np.float64) - x)), "want", np.max(np.abs(ow.astype(np.float64)-x)))
print("x[0,0,:12]", x[0,0,:12])
print("og[0,0,:12]", og[0,0,:12])
print("ow[0,0,:12]", ow[0,0,:12])
