"""A/B of the host-buffer quantize (cqb_quantize_ex) with and without the
overlapped chunked transfers (debug flag 1 << 19 turns them off): wall ms per
call with pinned host buffers, outputs compared.

    python tools/e2e_ab.py cfg4 [steps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import api  # noqa: E402
from paper_1011_0093_b200.api import context  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS, EPSILON, HARD_CAP  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
k = cfg.ks[-1] if hasattr(cfg, "ks") else 256
img = cfg.image()
P = img.shape[0] * img.shape[1]
pin_img = torch.from_numpy(img.reshape(-1)).pin_memory()
h_img = pin_img.numpy().reshape(img.shape)
term = api.Termination.convergent(EPSILON, HARD_CAP)
ctx = context(0)
res = {}
for flag in (0, 1 << 19, 0, 1 << 19):
    ctx.lib.cqb_set_debug(ctx.h, flag)
    pin_idx = torch.empty(P, dtype=torch.uint8).pin_memory()
    pin_out = torch.empty(3 * P, dtype=torch.uint8).pin_memory()
    h_idx = pin_idx.numpy().reshape(img.shape[:2])
    h_out = pin_out.numpy().reshape(img.shape)
    q = api.quantize(h_img, k, term, 1, out_index=h_idx, out_mapped=h_out)
    ts = []
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q = api.quantize(h_img, k, term, 1, out_index=h_idx, out_mapped=h_out)
        ts.append(time.perf_counter() - t0)
    res.setdefault(flag, []).append(np.median(ts) * 1e3)
    out = (q.palette.copy(), h_idx.copy(), h_out.copy(), q.report.dist_evals, q.report.iterations)
    if flag == 0:
        ref = out
    else:
        assert all(np.array_equal(a, b) for a, b in zip(ref, out)), "outputs differ"
for flag, v in res.items():
    print(f"{cfg.name} {'overlap' if flag == 0 else 'serial '}: median ms/call {['%.3f' % x for x in v]}"
          f" -> {P / min(v) / 1e3:.1f} Mpix/s")
ctx.lib.cqb_set_debug(ctx.h, 0)
