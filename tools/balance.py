"""Per-block phase timeline of WSM iteration 3 (profiling stamps)."""
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
G = C.c_int()
lib.cqb_device_info(ctx.h, None, C.byref(G))
g = G.value
lib.cqb_set_profiling(ctx.h, int(sys.argv[2]) if len(sys.argv) > 2 else 3)
lib.cqb_set_debug(ctx.h, int(os.environ.get("CQB_DEBUG", "0")))  # ablations (results wrong)
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
ph = bt[: 6 * g].reshape(6, g).astype(np.int64)
if len(sys.argv) > 3:
    np.save(sys.argv[3], bt)
t0 = ph[0].min()
names = ["iter start (after barrier2)", "points done", "flush done", "barrier1 exit", "finalize done", "tables done"]
for i, n in enumerate(names):
    v = (ph[i] - t0) / 1e3
    q = np.percentile(v, [0, 50, 90, 100])
    print(f"{n:28s} min {q[0]:6.2f} p50 {q[1]:6.2f} p90 {q[2]:6.2f} max {q[3]:6.2f}  argmax {int(np.argmax(v))}  block0 {v[0]:6.2f}")
dur = lambda a, b: (ph[b] - ph[a]) / 1e3  # noqa: E731
for a, b, n in [(0, 1, "points"), (1, 2, "flush"), (2, 3, "barrier1 wait"), (3, 4, "finalize"), (4, 5, "tables")]:
    v = dur(a, b)
    print(f"dur {n:14s} min {v.min():6.2f} p50 {np.median(v):6.2f} max {v.max():6.2f} block0 {v[0]:6.2f}")
ph = bt[: 12 * g].reshape(12, g).astype(np.int64)
rows = np.arange(1, g)  # blocks that own table rows
for a, b, n in [(3, 8, "fin: centers"), (8, 9, "fin: block0"), (9, 4, "fin: copy"), (4, 10, "tab: dist+load"),
                (10, 11, "tab: repair"), (11, 5, "tab: write")]:
    v = dur(a, b)[rows]
    print(f"sub {n:14s} min {v.min():6.2f} p50 {np.median(v):6.2f} max {v.max():6.2f}")
for a, b, n in [(3, 8, "block0 centers"), (8, 9, "block0 SSE/term"), (9, 4, "block0 copy")]:
    print(f"sub {n:16s} {dur(a, b)[0]:6.2f}")
b0 = bt[15 * g: 15 * g + 3].astype(np.int64)
t8 = int(bt[8 * g])
print(f"block0 SSE: terms {(b0[0] - t8) / 1e3:6.2f}  block_sum3 {(b0[1] - b0[0]) / 1e3:6.2f}  "
      f"decision+stores {(b0[2] - b0[1]) / 1e3:6.2f}  trailing sync {(int(bt[9 * g]) - b0[2]) / 1e3:6.2f}")
for a, b, n in []:
    v = dur(a, b)
    print(f"dur {n:14s} min {v.min():6.2f} p50 {np.median(v):6.2f} max {v.max():6.2f} block0 {v[0]:6.2f}")

wd = bt[6 * 1024: 6 * 1024 + 32 * 4].reshape(32, 4).astype(np.int64)
print("block 0 per warp: phase1 cycles, drain cycles, drains")
for w in range(32):
    print(f"  w{w:2d} p1 {wd[w,0]:7d}  p2 {wd[w,1]:7d}  drains {wd[w,2]}")

