import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_1011_0093_b200 import _native as N
from paper_1011_0093_b200.configs import CONFIGS
cfg = CONFIGS['cfg2']; ctx = N.context(0); lib = ctx.lib
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
lib.cqb_set_profiling(ctx.h, 1)
term = N.Termination(1, 10, 1e-4, 100); rep = N.Report(); cent = np.zeros(768); hist = np.zeros(100)
for _ in range(3):
    ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, 256, C.byref(term), 1, None, None, 1,
              cent.ctypes.data_as(C.POINTER(C.c_double)), hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
bt = np.zeros(16 * 1024, np.uint64)
lib.cqb_block_times(ctx.h, bt.ctypes.data_as(C.POINTER(C.c_uint64)), 16 * 1024)
s = bt[14 * 1024: 14 * 1024 + 11].astype(np.int64)
print('prep stamps (us from start):', np.round((s - s[0]) / 1e3, 2).tolist())
pb = (bt[13 * 1024: 13 * 1024 + 148].astype(np.int64) - s[0]) / 1e3
print('phase B end per block: min %.2f p50 %.2f p90 %.2f max %.2f argmax %d' % (pb.min(), np.median(pb), np.percentile(pb, 90), pb.max(), pb.argmax()))
print('raw', bt[13 * 1024: 13 * 1024 + 4], bt[14 * 1024: 14 * 1024 + 2])
