import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1011_0093_b200 import api
from paper_1011_0093_b200.configs import gmm_image
found = 0
for seed in range(200):
    for comp, k in ((3, 32), (6, 64), (12, 128), (4, 48)):
        img = gmm_image(48, 40, comp, seed)
        h = api.build_histogram(img)
        if h.size() < k:
            continue
        q = api.quantize(img, k, api.Termination.convergent(1e-4, 100), seed=seed)
        if q.report.empty_events > 0:
            print("EMPTY", seed, comp, k, q.report.empty_events, q.report.iterations, flush=True)
            found += 1
    if found >= 6:
        break
print("done", found)
