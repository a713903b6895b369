"""Per-kernel device time (library profiler marks) of one BASELINE config through the C ABI.

    python tools/config_profile.py c4 [c2 ...]      (GPU box; "c3:u" = FtConfig.unprotected())
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
fa0, _ = F.pipeline._faults_c([])
cfg = F.FtConfig()
for arg in sys.argv[1:]:
    name, _, flag = arg.partition(":")
    cfg = F.FtConfig.unprotected() if flag == "u" else F.FtConfig()
    x = bench.load_field(name)
    mode, v = synth.CONFIGS[name]["eb"]
    nx, ny, nz = x.shape
    d_x = torch.from_numpy(x).cuda()
    d_o = torch.empty(x.size, dtype=torch.float32, device="cuda")
    rb = F.pipeline._ReportBuf(F.partition(x.shape, 10).n_blocks)
    mcode = {"absolute": 0, "value_range_relative": 1}[mode]
    for it in range(4):
        if it == 3:
            _lib.profile(True, 0)
        L.ftlz_ctx_compress_device(ctx, d_x.data_ptr(), nx, ny, nz, mcode, v, C.byref(cfg._c()), fa0, 0, None,
                                   C.byref(rb.r))
        ptr, ln = C.c_void_p(), C.c_size_t()
        L.ftlz_ctx_archive_device(ctx, C.byref(ptr), C.byref(ln))
        hb = np.zeros(64, np.uint8)
        bench.ctypes_cuda().cudaMemcpy(C.c_void_p(hb.ctypes.data), C.c_void_p(ptr.value), C.c_size_t(64), 2)
        hdr, info = _lib.Header(), _lib.Info()
        L.ftlz_peek_header(hb.tobytes(), 64, C.byref(hdr), C.byref(info))
        L.ftlz_ctx_decompress_device(ctx, ptr.value, ln.value, C.byref(hdr), d_o.data_ptr(), fa0, 0, C.byref(rb.r))
        torch.cuda.synchronize()
    prof = _lib.profile_read(0)
    _lib.profile(False, 0)
    print(arg, {k: round(p[0], 3) for k, p in prof.items() if p[0] > 0.004})
