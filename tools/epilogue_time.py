"""Time of the loop kernel's parts outside the iterations (per-block %globaltimer stamps):
python tools/epilogue_time.py CONFIG -> entry..loop exit, loop exit..kernel exit (the fused map epilogue)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_1011_0093_b200 import _native as N
from paper_1011_0093_b200.configs import CONFIGS
cfg = CONFIGS[sys.argv[1]]
ctx = N.context(0); lib = ctx.lib
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
idx = torch.empty(cfg.pixels, dtype=torch.uint8, device="cuda")
out = torch.empty(3 * cfg.pixels, dtype=torch.uint8, device="cuda")
G = C.c_int(); lib.cqb_device_info(ctx.h, None, C.byref(G)); g = G.value
term = N.Termination(1, 10, 1e-4, 100); rep = N.Report(); cent = np.zeros(768); hist = np.zeros(100)
for rnd in range(3):
    lib.cqb_set_profiling(ctx.h, 5)
    ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d.data_ptr()), cfg.pixels, 256, C.byref(term), 1,
                                      C.c_void_p(idx.data_ptr()), C.c_void_p(out.data_ptr()), 0,
                                      cent.ctypes.data_as(C.POINTER(C.c_double)), hist.ctypes.data_as(C.POINTER(C.c_double)), 100, C.byref(rep)))
    bt = np.zeros(16 * 1024, np.uint64)
    lib.cqb_block_times(ctx.h, bt.ctypes.data_as(C.POINTER(C.c_uint64)), 16 * 1024)
    ph = bt[: 16 * g].reshape(16, g).astype(np.int64)
    t0 = ph[12].min()
    print(f"entry..loop exit {(ph[13].max() - t0) / 1e3:9.1f} us   loop exit..kernel exit {(ph[14].max() - ph[13].max()) / 1e3:7.1f} us   "
          f"iterations {rep.iterations}")
