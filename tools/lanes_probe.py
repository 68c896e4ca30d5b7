import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1011_0093_b200 import api
from paper_1011_0093_b200.configs import CONFIGS
cfg = CONFIGS["cfg5"]
imgs = [torch.from_numpy(cfg.image(i).reshape(-1)).cuda() for i in range(16)]
term = api.Termination.convergent(1e-4, 100)
for lanes in (1, 2, 4, 6, 8, 12, 16):
    try:
        api.quantize_batch_device(imgs, 256, term, 1, lanes=lanes)
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(3): api.quantize_batch_device(imgs, 256, term, 1, lanes=lanes)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
        print(lanes, f"{dt*1e3:.2f} ms  {16*cfg.pixels/dt/1e6:.0f} Mpix/s")
    except Exception as e:
        print(lanes, "ERR", e)
