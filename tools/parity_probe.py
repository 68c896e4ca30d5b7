"""Re-run the randomized parity cases and print evaluation counts per debug flag (diagnostic)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1011_0093_b200 import api, _native as N  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
import test_gpu_parity as T  # noqa: E402

port = Oracle("port")
ctx = N.context(0)
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rng = np.random.default_rng(100 + seed)
for ci, img in enumerate(T._random_cases(12, seed)):
    P = img.shape[0] * img.shape[1]
    h = port.build_histogram(img)
    n = len(h.keys)
    k = int(rng.integers(1, min(n, 256) + 1))
    mode = int(rng.integers(0, 2))
    term = api.Termination.convergent(1e-4, 100) if mode else api.Termination.fixed(int(rng.integers(1, 12)))
    iters = 10 if mode else term.max_iters
    o = port.run_wsm(h.keys, h.counts, P, k, mode=mode, max_iters=iters, eps=1e-4, cap=100, seed=7)
    res = []
    for fl in (0, 1, 16, 32, 128, 256, 16 | 128):
        ctx.lib.cqb_set_debug(ctx.h, fl)
        q = api.quantize(img, k, term, seed=7)
        res.append((fl, q.report.iterations, q.report.dist_evals, float(np.abs(q.palette - o.centers).max())))
    ctx.lib.cqb_set_debug(ctx.h, 0)
    bad = any(r[2] != o.dist_evals or r[1] != o.iterations for r in res if r[0] != 1)
    print(ci, img.shape, "n", n, "k", k, "mode", mode, "oracle", o.iterations, o.dist_evals, "BAD" if bad else "ok")
    if bad:
        for r in res:
            print("   flags", r)
