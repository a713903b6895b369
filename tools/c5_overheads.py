"""c5 time overheads (bench.run_c5) repeated, to see the run-to-run spread of the three arms.

    python tools/c5_overheads.py [repeats]        (GPU box)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_03144_b200 as F  # noqa: E402
from paper_2010_03144_b200 import _lib  # noqa: E402

L = _lib.load()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    r = bench.run_c5(F, L, _lib, torch, 0)
    print("fault-free %.4f ms" % r["fault_free_ms"],
          {a: (round(r[a]["ms"], 4), round(100 * r[a]["time_overhead"], 2), r[a]["detected_corrected"],
               r[a]["output_bit_identical"]) for a in ("input", "bins", "decomp")})
