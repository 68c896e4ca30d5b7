"""e2e throughput of api.quantize (pinned host buffers) with N concurrent
host callers and a library debug flag: python tools/e2e_inflight.py CONFIG
INFLIGHT FLAGS [steps]."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import api  # noqa: E402
from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
inflight, flags = int(sys.argv[2]), int(sys.argv[3])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 12
img = cfg.image()
P = cfg.pixels
term = api.Termination.convergent(1e-4, 100)
bufs = []
for _ in range(inflight):
    a = torch.from_numpy(img.reshape(-1)).pin_memory()
    b = torch.empty(3 * P, dtype=torch.uint8).pin_memory()
    bufs.append((a, b, a.numpy().reshape(img.shape), b.numpy().reshape(img.shape)))


def work(j, n):
    torch.cuda.set_device(0)
    ctx = N.context(0)
    ctx.lib.cqb_set_debug(ctx.h, flags)
    for _ in range(n):
        api.quantize(bufs[j][2], 256, term, 1, index_map=False, out_mapped=bufs[j][3])


with ThreadPoolExecutor(inflight) as ex:
    list(ex.map(lambda j: work(j, 2), range(inflight)))
    res = []
    for r in range(3):
        t0 = time.perf_counter()
        list(ex.map(lambda j: work(j, steps // inflight), range(inflight)))
        res.append(time.perf_counter() - t0)
n = steps // inflight * inflight
t = float(np.median(res))
print(f"{cfg.name} inflight {inflight} flags {flags}: {t / n * 1e3:.3f} ms/image  {P * n / t / 1e6:.1f} Mpix/s")
