"""Single-image grid-size sweep and concurrent multi-image throughput on one GPU.

usage: python tools/batch_probe.py [cfg] [reps]
"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS, gmm_image  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
lib = N.load_library()
term = N.Termination(1, 10, 1e-4, 100)
_f64p = C.POINTER(C.c_double)


def mk(grid):
    h = C.c_void_p()
    assert lib.cqb_create(0, C.byref(h)) == 0
    lib.cqb_set_grid_limit(h, grid)
    return h


def run(ctxs, imgs, sync_each=False):
    reps_ = []
    cent = np.zeros(768)
    hist = np.zeros(100)
    rep = N.Report()
    for h, d in zip(ctxs, imgs):
        rc = lib.cqb_quantize_device(h, C.c_void_p(d.data_ptr()), d.numel() // 3, 256, C.byref(term), 1, None, None,
                                     0, None, None, 0, None)
        assert rc == 0, lib.cqb_last_error(h)
    for h in ctxs:
        assert lib.cqb_fetch_results(h, cent.ctypes.data_as(_f64p), hist.ctypes.data_as(_f64p), 100, C.byref(rep)) == 0
        reps_.append(rep.iterations)
    return reps_


H, W = cfg.height, cfg.width
for grid in (148, 128, 111, 96, 74, 37):
    ctx = [mk(grid)]
    d = [torch.from_numpy(cfg.image().reshape(-1)).cuda()]
    run(ctx, d)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        it = run(ctx, d)
    dt = (time.perf_counter() - t) / reps
    print(f"single image grid {grid:3d}: {dt * 1e3:7.3f} ms/image  {H * W / dt / 1e6:8.1f} Mpix/s  iters {it}")
    lib.cqb_destroy(ctx[0])
for B in (1, 2, 3, 4, 6, 8):
    g = 148 // B
    ctxs = [mk(g) for _ in range(B)]
    imgs = [torch.from_numpy(gmm_image(W, H, 256, 1000 + i).reshape(-1)).cuda() for i in range(B)]
    run(ctxs, imgs)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        it = run(ctxs, imgs)
    dt = (time.perf_counter() - t) / reps
    print(f"concurrent {B} images grid {g:3d}: {dt * 1e3:7.3f} ms/batch  {B * H * W / dt / 1e6:8.1f} Mpix/s agg  iters {it}")
    for h in ctxs:
        lib.cqb_destroy(h)
