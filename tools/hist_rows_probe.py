"""Wall time of the row-sharded histogram steps on one GPU (calls are
synchronous): cqb_hist_rows for rank 0 of W, cqb_hist_merge of owner 0's
inputs from all W row shards: python tools/hist_rows_probe.py CONFIG W."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import _native as N  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402
from paper_1011_0093_b200.distributed import DeviceHistBackend  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
W = int(sys.argv[2])
ctx = N.context(0)
be = DeviceHistBackend(ctx)
d = torch.from_numpy(cfg.image().reshape(-1)).cuda()
P = cfg.pixels
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    runs = [be.rows(d, P, W, r) for r in range(W)]
    t1 = time.perf_counter()
    parts = [loc[sum(c[:0]): sum(c[:1])] for loc, c in runs]
    recv = torch.cat(parts)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    own = be.merge(recv, W)
    t3 = time.perf_counter()
print(f"{cfg.name} W={W}: hist_rows per rank {(t1 - t0) / W * 1e3:.3f} ms (local samples {runs[0][0].shape[0]}), "
      f"merge of owner 0 ({recv.shape[0]} in -> {own.shape[0]} out) {(t3 - t2) * 1e3:.3f} ms")

# the Morton-range split: every pixel, one range of bins per rank
for rep in range(3):
    t0 = time.perf_counter()
    own = [be.range(d, P, W, r) for r in range(W)]
    t1 = time.perf_counter()
print(f"{cfg.name} W={W}: hist_range per rank {(t1 - t0) / W * 1e3:.3f} ms (rank 0 owns {own[0].shape[0]} samples)")
