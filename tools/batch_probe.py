"""Config 5 lanes sweep: aggregate Mpixel/s of cqb_quantize_batch vs lanes.

usage: python tools/batch_probe.py [n_images] [lanes,...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1011_0093_b200 import api  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lanes_list = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "3", "4", "5", "6", "8"])]
cfg = CONFIGS["cfg5"]
imgs = [torch.from_numpy(cfg.image(i).reshape(-1)).cuda() for i in range(n)]
term = api.Termination.convergent(1e-4, 100)
for lanes in lanes_list:
    api.quantize_batch_device(imgs, 256, term, 1, lanes=lanes)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(2):
        _, reps = api.quantize_batch_device(imgs, 256, term, 1, lanes=lanes)
    dt = (time.perf_counter() - t) / 2
    print(f"lanes {lanes}: {dt * 1e3:8.2f} ms/batch  {n * cfg.pixels / dt / 1e6:8.1f} Mpix/s  "
          f"iters {[r.iterations for r in reps[:6]]}", flush=True)
