import sys
sys.path.insert(0, ".")
import paper_2010_03144_b200 as F
from tests.golden_util import load, manifest
from oracle import oracle as O
name = sys.argv[1]
e = manifest()["cases"][name]
x = load(name)["input"]
cfg = F.FtConfig(**{k: v for k, v in e["cfg"].items() if k != "bin_capacity"},
                 quant=F.QuantConfig(e["cfg"]["bin_capacity"]) if "bin_capacity" in e["cfg"] else F.QuantConfig())
try:
    a = F.compress_bytes(x, e["mode"], e["value"], cfg)
    ref, _ = O.compress(x, e["mode"], e["value"], e["cfg"])
    print(name, "len", len(a), len(ref), "same", bytes(a) == ref)
except Exception as ex:
    print(name, "ERR", type(ex).__name__, str(ex)[:200])
