"""Where the WSM loop kernel's time goes outside the iterations: prologue
(initial center tables), iterations, loop exit -> map epilogue end (profiling
stamps 12-14 of cqb_block_times + the iteration timeline)."""
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
idx = torch.empty(cfg.pixels, dtype=torch.uint8, device="cuda")
out = torch.empty(3 * cfg.pixels, dtype=torch.uint8, device="cuda")
G = C.c_int()
lib.cqb_device_info(ctx.h, None, C.byref(G))
g = G.value
lib.cqb_set_profiling(ctx.h, 1)
term = N.Termination(1, 10, 1e-4, 100)
rep = N.Report()
cent = np.zeros(768)
hist = np.zeros(100)
for _ in range(3):
    ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, 256, C.byref(term), 1,
                                      C.c_void_p(idx.data_ptr()), C.c_void_p(out.data_ptr()), 1,
                                      cent.ctypes.data_as(C.POINTER(C.c_double)),
                                      hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
bt = np.zeros(16 * 1024, np.uint64)
lib.cqb_block_times(ctx.h, bt.ctypes.data_as(C.POINTER(C.c_uint64)), 16 * 1024)
tl = np.zeros(800, np.uint64)
lib.cqb_loop_timeline(ctx.h, tl.ctypes.data_as(C.POINTER(C.c_uint64)), 100)
tl = tl.reshape(100, 8).astype(np.int64)
ph = bt[: 16 * g].reshape(16, g).astype(np.int64)  # [phase][block]
entry, lexit, kexit = ph[12], ph[13], ph[14]
it = rep.iterations
t0 = entry.min()
us = lambda v: v / 1e3  # noqa: E731
print(f"iterations {it}")
print(f"kernel entry spread      {us(entry.max() - entry.min()):8.2f} us")
print(f"prologue (entry->it1)    {us(tl[0, 0] - t0):8.2f} us")
print(f"iterations (it1->exit)   {us(lexit[0] - tl[0, 0]):8.2f} us   ({us(lexit[0] - tl[0, 0]) / it:.2f} us/it)")
print(f"epilogue (exit->end) b0  {us(kexit[0] - lexit[0]):8.2f} us  max over blocks {us(kexit.max() - lexit.min()):8.2f}")
print(f"kernel total (stamps)    {us(kexit.max() - t0):8.2f} us")
