"""A/B of a library debug flag on the device-resident quantize (CUDA events,
L2 flushed between steps): python tools/ab_debug.py CONFIG FLAG [rounds]."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
flag = int(sys.argv[2])
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
ctx = N.context(0)
lib = ctx.lib
s = torch.cuda.Stream()
ctx.check(lib.cqb_set_stream(ctx.h, C.c_void_p(s.cuda_stream)))
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
idx = torch.empty(cfg.pixels, dtype=torch.uint8, device="cuda")
out = torch.empty(3 * cfg.pixels, dtype=torch.uint8, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
term = N.Termination(1, 10, 1e-4, 100)
rep = N.Report()
cent = np.zeros(768)
hist = np.zeros(100)


def run(n):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    with torch.cuda.stream(s):
        for a, b in ev:
            fl.fill_(1)
            a.record(s)
            ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, 256, C.byref(term), 1,
                                              C.c_void_p(idx.data_ptr()), C.c_void_p(out.data_ptr()), 0,
                                              cent.ctypes.data_as(C.POINTER(C.c_double)),
                                              hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
            b.record(s)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


res = {0: [], flag: []}
for r in range(rounds):
    for f in (0, flag):
        lib.cqb_set_debug(ctx.h, f)
        run(3)
        res[f].append(run(20))
for f, v in res.items():
    print(f"flag {f}: median ms/step {np.median(v):.4f}  rounds {[round(x, 4) for x in v]}  "
          f"-> {cfg.pixels / np.median(v) / 1e3:.1f} Mpix/s")
