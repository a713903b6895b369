import sys, numpy as np
sys.path.insert(0, ".")
import paper_2010_03144_b200 as F
from tests.golden_util import load, manifest, faults_of
name = sys.argv[1]
e = manifest()["cases"][name]; z = load(name)
d = dict(e["cfg"]); cfg = F.FtConfig(**d)
try:
    s, rep = F.compress(F.Field.from_array(z["input"]), F.ErrorBound(e["mode"], e["value"]), cfg, faults=faults_of(e))
    data = F.serialize(s)
    print("compress ok", len(data), data == z["archive"].tobytes(), rep.to_dict(), flush=True)
except Exception as ex:
    print("compress failed", type(ex).__name__, ex, flush=True); raise
out, drep = F.decompress(F.parse(data), faults=faults_of(e))
print("decompress", drep.to_dict())
