"""Ablation timing of the WSM loop phases (diagnostic flags; results wrong on purpose)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
ctx = N.context(0)
lib = ctx.lib
img = cfg.image()
d = torch.from_numpy(img.reshape(-1)).cuda()
term = N.Termination(1, 10, 1e-4, 100)  # the bench's convergent run
rep = N.Report()
cent = np.zeros(768)
hist = np.zeros(100)
lib.cqb_set_profiling(ctx.h, 1)
for flags in [int(f) for f in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['0', '1', '16'])]:
    lib.cqb_set_debug(ctx.h, flags)
    ts = []
    for _ in range(3):
        ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, 256, C.byref(term), 1, None,
                                          None, 1, cent.ctypes.data_as(C.POINTER(C.c_double)),
                                          hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
        tl = np.zeros(800, np.uint64)
        lib.cqb_loop_timeline(ctx.h, tl.ctypes.data_as(C.POINTER(C.c_uint64)), 100)
        n = int(rep.iterations)
        tl = tl.reshape(100, 8).astype(np.int64)[:n]
        a = tl[2:-1]
        ts.append((np.mean(a[:, 2] - a[:, 1]) / 1e3, np.mean(a[:, 4] - a[:, 3]) / 1e3, np.mean(np.diff(tl[2:, 0])) / 1e3,
                   (tl[n - 1, 6] - tl[0, 0]) / 1e3, n))
    t = np.median(np.array(ts), axis=0)
    print(f"flags {flags:2d}: block0 points {t[0]:7.2f} us  barrier1 {t[1]:7.2f} us  iteration {t[2]:7.2f} us  "
          f"loop {t[3]:8.1f} us  iterations {int(t[4])}")
lib.cqb_set_debug(ctx.h, 0)
