"""Device-resident quantize of one config, N times (profiling driver):
python tools/run_once.py CONFIG [N] [K] [debug_flags]."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
k = int(sys.argv[3]) if len(sys.argv) > 3 else 256
flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
ctx = N.context(0)
lib = ctx.lib
lib.cqb_set_debug(ctx.h, flags)
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
idx = torch.empty(cfg.pixels, dtype=torch.uint8, device="cuda")
out = torch.empty(3 * cfg.pixels, dtype=torch.uint8, device="cuda")
term = N.Termination(1, 10, 1e-4, 100)
rep = N.Report()
cent = np.zeros(3 * k)
hist = np.zeros(100)
for _ in range(n):
    ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, k, C.byref(term), 1,
                                      C.c_void_p(idx.data_ptr()), C.c_void_p(out.data_ptr()), 1,
                                      cent.ctypes.data_as(C.POINTER(C.c_double)),
                                      hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
print(f"{cfg.name} k={k}: iterations={rep.iterations} evals={rep.dist_evals} elapsed_ms={rep.elapsed_ms:.3f}")
