"""Per-kernel device time of the c5 arms (fault-free, input, bins, decompressed-data flips).

    python tools/c5_profile.py        (GPU box; needs the c5 field, tools/synth.py makes it)
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2010_03144_b200 as F  # noqa: E402
from paper_2010_03144_b200 import _lib  # noqa: E402
from tools import synth  # noqa: E402

x = bench.load_field("c5")
mode, v = synth.CONFIGS["c5"]["eb"]
vols = synth.block_volumes(x.shape, 10)
plan = synth.fault_plan(len(vols), vols)
field = F.Field.from_array(x)
eb = F.ErrorBound(mode, v)
for tgt in (None, "input", "bins", "decomp"):
    faults = [(tgt, b, e, t) for b, e, t in plan] if tgt else None
    for rep in range(2):
        _lib.profile(True, 0)
        s, _ = F.compress(field, eb, F.FtConfig(), faults=faults if tgt in ("input", "bins") else None)
        data = F.serialize(s)
        F.decompress(F.parse(data), faults=faults if tgt == "decomp" else None)
        prof = _lib.profile_read(0)
        _lib.profile(False, 0)
    tot = sum(p[0] for p in prof.values())
    print(tgt, round(tot, 3), {k: (round(p[0], 3), p[1]) for k, p in prof.items() if p[0] > 0.005})
