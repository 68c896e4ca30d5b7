"""Per-iteration diagnostics of the WSM loop from the %globaltimer timeline:
python tools/loop_counts.py CONFIG [K] [debug_flags]. With debug flag
1<<19 the "active" column counts FP64 fallbacks of the FP32 screen, with
1<<20 skipped points (chunk skipping)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 256
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ctx = N.context(0)
lib = ctx.lib
lib.cqb_set_debug(ctx.h, flags)
lib.cqb_set_profiling(ctx.h, 1)
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
term = N.Termination(1, 10, 1e-4, 100)
rep = N.Report()
cent = np.zeros(3 * k)
hist = np.zeros(100)
ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, k, C.byref(term), 1, None, None, 1,
                                  cent.ctypes.data_as(C.POINTER(C.c_double)),
                                  hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
tl = np.zeros(800, np.uint64)
ctx.check(lib.cqb_loop_timeline(ctx.h, tl.ctypes.data_as(C.POINTER(C.c_uint64)), 100))
tl = tl.reshape(100, 8).astype(np.int64)[: rep.iterations]
n = int(rep.n_unique)
print(f"{cfg.name} k={k} flags={flags}: N'={n} iterations={rep.iterations} evals={rep.dist_evals}")
print(" it   iter_us  points_us  changed   count    count/N'")
for i in range(rep.iterations):
    it_us = (tl[i + 1, 0] - tl[i, 0]) / 1e3 if i + 1 < rep.iterations else float("nan")
    pts = (tl[i, 2] - tl[i, 1]) / 1e3
    ch, cnt = int(tl[i, 7]) & 0xFFFFFFFF, int(tl[i, 7]) >> 32
    print(f"{i + 1:3d} {it_us:9.2f} {pts:9.2f} {ch:9d} {cnt:9d}  {cnt / n:8.4f}")
