"""Where the e2e time goes: api.quantize vs the bare C call vs the device-resident pipeline (diagnostic)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import api, _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg2"]
img = cfg.image()
P = img.shape[0] * img.shape[1]
ctx = N.context(0)
lib = ctx.lib
pin_img = torch.from_numpy(img.reshape(-1)).pin_memory()
pin_idx = torch.empty(P, dtype=torch.uint8).pin_memory()
pin_out = torch.empty(3 * P, dtype=torch.uint8).pin_memory()
h_img = pin_img.numpy().reshape(img.shape)
h_idx = pin_idx.numpy().reshape(img.shape[:2])
h_out = pin_out.numpy().reshape(img.shape)
term = api.Termination.convergent(1e-4, 100)
t = term.native()
cent = np.zeros(768)
hist = np.zeros(100)
rep = N.Report()
u8 = C.POINTER(C.c_uint8)
f64 = C.POINTER(C.c_double)


def raw(idx=True, out=True):
    ctx.check(lib.cqb_quantize_ex(ctx.h, h_img.ctypes.data_as(u8), img.shape[1], img.shape[0], 256, C.byref(t), 1,
                                  cent.ctypes.data_as(f64), hist.ctypes.data_as(f64), 100,
                                  h_idx.ctypes.data_as(u8) if idx else None, h_out.ctypes.data_as(u8) if out else None,
                                  None, C.byref(rep)))


def timeit(f, n=20):
    for _ in range(3):
        f()
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3


print("api.quantize          %.3f ms" % timeit(lambda: api.quantize(h_img, 256, term, 1, out_index=h_idx, out_mapped=h_out)))
print("raw C idx+rgb         %.3f ms" % timeit(lambda: raw(True, True)))
print("raw C idx only        %.3f ms" % timeit(lambda: raw(True, False)))
print("raw C no outputs      %.3f ms" % timeit(lambda: raw(False, False)))
d = torch.from_numpy(img.reshape(-1)).cuda()
dcent = np.zeros(768)


def dev():
    ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), P, 256, C.byref(t), 1, None, None, 1,
                                      dcent.ctypes.data_as(f64), hist.ctypes.data_as(f64), 100, C.byref(rep)))


print("device-resident       %.3f ms" % timeit(dev))
lib.cqb_set_debug(ctx.h, 65536)  # staging copies + D2H copies (no zero-copy)
print("[no zero-copy] api.quantize  %.3f ms" % timeit(lambda: api.quantize(h_img, 256, term, 1, out_index=h_idx, out_mapped=h_out)))
print("[no zero-copy] raw C idx+rgb %.3f ms" % timeit(lambda: raw(True, True)))
lib.cqb_set_debug(ctx.h, 0)
print("api.quantize (again)  %.3f ms" % timeit(lambda: api.quantize(h_img, 256, term, 1, out_index=h_idx, out_mapped=h_out)))
