"""Block 0's chunk schedule in one iteration (build with -DCQB_CHUNK_STAMPS=1; diagnostic)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg2"]
ctx = N.context(0)
lib = ctx.lib
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
lib.cqb_set_profiling(ctx.h, int(sys.argv[1]) if len(sys.argv) > 1 else 30)
term = N.Termination(1, 10, 1e-4, 100)
rep = N.Report()
cent = np.zeros(768)
hist = np.zeros(100)
for _ in range(2):
    ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, 256, C.byref(term), 1, None, None, 1,
                                      cent.ctypes.data_as(C.POINTER(C.c_double)),
                                      hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
bt = np.zeros(16 * 1024, np.uint64)
lib.cqb_block_times(ctx.h, bt.ctypes.data_as(C.POINTER(C.c_uint64)), 16 * 1024)
g = 148
t0 = int(bt[0])  # block 0 iteration start (phase 0 stamp)
ch = bt[4096: 4096 + 4 * 1000].reshape(1000, 4).astype(np.int64)
ch = ch[ch[:, 1] > 0]
print("chunks", len(ch), "points phase (block 0) %.2f us" % ((int(bt[g]) - t0) / 1e3))
order = np.argsort(ch[:, 1])
for c in ch[order]:
    print("warp %2d start %6.2f end %6.2f dur %5.2f cost %3d" % (c[0], (c[1] - t0) / 1e3, (c[2] - t0) / 1e3,
                                                               (c[2] - c[1]) / 1e3, c[3]))
dur = (ch[:, 2] - ch[:, 1]) / 1e3
print("dur vs cost corr %.2f; mean dur %.2f" % (np.corrcoef(dur, ch[:, 3])[0, 1], dur.mean()))
