"""Per-stage CUDA-event times of the device-resident quantize (L2 flushed
between steps), for A/B of libraries (CQB_LIB_PATH) and debug flags:
python tools/stage_ab.py CONFIG [FLAGS ...]  -> one line per flag value."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
flags = [int(f) for f in sys.argv[2:]] or [0]
ctx = N.context(0)
lib = ctx.lib
s = torch.cuda.Stream()
ctx.check(lib.cqb_set_stream(ctx.h, C.c_void_p(s.cuda_stream)))
lib.cqb_set_profiling(ctx.h, 1)
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
idx = torch.empty(cfg.pixels, dtype=torch.uint8, device="cuda")
out = torch.empty(3 * cfg.pixels, dtype=torch.uint8, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
term = N.Termination(1, 10, 1e-4, 100)
rep = N.Report()
cent = np.zeros(768)
hist = np.zeros(100)
ms = (C.c_float * 7)()


def run(n):
    st = []
    with torch.cuda.stream(s):
        for _ in range(n):
            fl.fill_(1)
            ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, 256, C.byref(term), 1,
                                              C.c_void_p(idx.data_ptr()), C.c_void_p(out.data_ptr()), 0,
                                              cent.ctypes.data_as(C.POINTER(C.c_double)),
                                              hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
            ctx.check(lib.cqb_stage_times(ctx.h, ms, 7))
            st.append(list(ms))
    return np.median(np.array(st), axis=0)


res = {}
for r in range(2):
    for f in flags:
        lib.cqb_set_debug(ctx.h, f)
        run(2)
        res.setdefault(f, []).append(run(10))
lib_name = os.path.basename(os.environ.get("CQB_LIB_PATH", "cur"))
for f, v in res.items():
    m = np.median(np.array(v), axis=0)
    print(f"{cfg.name} {lib_name} flag {f}: total {m.sum():.4f} ms  " +
          " ".join(f"{n}={x * 1e3:.1f}us" for n, x in zip(N.STAGES, m)))
