"""Per-kernel device time (library profiler marks) of the c5 arms through the C ABI with the
field and archive in HBM: where the fault arms' extra time goes.

    python tools/c5_device_profile.py        (GPU box)
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_03144_b200 as F  # noqa: E402
from paper_2010_03144_b200 import _lib  # noqa: E402
from tools import synth  # noqa: E402

L = _lib.load()
ctx = _lib.context(0)
x = bench.load_field("c5")
mode, v = synth.CONFIGS["c5"]["eb"]
vols = synth.block_volumes(x.shape, 10)
plan = synth.fault_plan(len(vols), vols)
nx, ny, nz = x.shape
d_x = torch.from_numpy(x).cuda()
d_o = torch.empty(x.size, dtype=torch.float32, device="cuda")
rb = F.pipeline._ReportBuf(len(vols))
cfg = F.FtConfig()
fa0, _ = F.pipeline._faults_c([])
for tgt in (None, "input", "bins", "decomp"):
    fd = F.pipeline._faults_c([(tgt, b, e, t) for b, e, t in plan]) if tgt else (fa0, 0)
    fc = fd if tgt in ("input", "bins") else (fa0, 0)
    fdd = fd if tgt == "decomp" else (fa0, 0)
    for it in range(4):
        if it == 3:
            _lib.profile(True, 0)
        L.ftlz_ctx_compress_device(ctx, d_x.data_ptr(), nx, ny, nz, 1, v, C.byref(cfg._c()), fc[0], fc[1], None,
                                   C.byref(rb.r))
        ptr, ln = C.c_void_p(), C.c_size_t()
        L.ftlz_ctx_archive_device(ctx, C.byref(ptr), C.byref(ln))
        hb = np.zeros(64, np.uint8)
        bench.ctypes_cuda().cudaMemcpy(C.c_void_p(hb.ctypes.data), C.c_void_p(ptr.value), C.c_size_t(64), 2)
        hdr, info = _lib.Header(), _lib.Info()
        L.ftlz_peek_header(hb.tobytes(), 64, C.byref(hdr), C.byref(info))
        L.ftlz_ctx_decompress_device(ctx, ptr.value, ln.value, C.byref(hdr), d_o.data_ptr(), fdd[0], fdd[1],
                                     C.byref(rb.r))
        torch.cuda.synchronize()
    prof = _lib.profile_read(0)
    _lib.profile(False, 0)
    tot = sum(p[0] for p in prof.values())
    print(tgt, round(tot, 3), {k: round(p[0], 3) for k, p in prof.items() if p[0] > 0.003})
