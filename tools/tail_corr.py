import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_1011_0093_b200 import _native as N
from paper_1011_0093_b200.configs import CONFIGS
cfg = CONFIGS[sys.argv[1]]
ctx = N.context(0); lib = ctx.lib
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
G = C.c_int(); lib.cqb_device_info(ctx.h, None, C.byref(G)); g = G.value
term = N.Termination(1, 10, 1e-4, 100); rep = N.Report(); cent = np.zeros(768); hist = np.zeros(100)
durs = []; sms = None
for it in [10, 20, 30, 40, 50]:
    lib.cqb_set_profiling(ctx.h, it)
    ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, 256, C.byref(term), 1, None, None, 1,
                                      cent.ctypes.data_as(C.POINTER(C.c_double)), hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
    bt = np.zeros(16 * 1024, np.uint64)
    lib.cqb_block_times(ctx.h, bt.ctypes.data_as(C.POINTER(C.c_uint64)), 16 * 1024)
    ph = bt[: 8 * g].reshape(8, g).astype(np.int64)
    durs.append((ph[2] - ph[0]) / 1e3)  # points + flush from iteration start
    sms = ph[6]
D = np.array(durs)
print("per-iteration: mean, max, argmax block, argmax sm")
for i, v in enumerate(D):
    print(f"  {v.mean():7.2f} {v.max():7.2f} {int(v.argmax()):4d} {int(sms[v.argmax()]):4d}  spread {v.max()-v.min():5.2f}")
z = (D - D.mean(1, keepdims=True)) / D.std(1, keepdims=True)
print("corr of block z-scores between iterations:")
print(np.round(np.corrcoef(z), 2))
zm = z.mean(0)
o = np.argsort(zm)[::-1][:10]
print("slowest blocks (mean z):", [(int(b), int(sms[b]), round(float(zm[b]), 2)) for b in o])
