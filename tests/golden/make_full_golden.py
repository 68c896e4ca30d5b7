"""Full-size golden summaries of every BASELINE.json config, from the
UNMODIFIED reference (oracle/_ref: the colorq headers compiled in place).

For each (config, image, K) case the reference runs its own hot path as the
CLI composes it (tools/colorq.cpp:96-102): build_histogram
(histogram.hpp:65-99) -> run_wsm with convergent(1e-4, 100) and init seed 1
(kmeans.hpp:394-404) -> map_pixels (image_ops.hpp:18-51) -> mse
(metrics.hpp:18-29). The summary keeps, bit for bit (floats as float.hex):
N', a SHA-256 of the first-occurrence histogram, the palette, iterations,
dist_evals, SSE and sse_history, MSE, and SHA-256 digests of the mapped raster
and of the index map. The reference has no index map; it is taken from the
C port's map_pixels on the reference palette, after checking that the port's
mapped raster equals the reference's byte for byte.

The images come from paper_1011_0093_b200/configs.py (seeded PCG64, the same
on every machine), so the GPU tests regenerate them and compare against this
file without touching /root/reference. Regenerate with
    python tests/golden/make_full_golden.py          (~2 min, all cores)
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1011_0093_b200.configs import CONFIGS, EPSILON, HARD_CAP, INIT_SEED  # noqa: E402

OUT = os.path.join(HERE, "full_configs.json")

# (config, image index, K): every config at each of its K; config 5 on its
# first four images (each a distinct seed, 1000 + i)
CASES = ([("cfg1", 0, 32), ("cfg2", 0, 64), ("cfg2", 0, 256), ("cfg3", 0, 256), ("cfg4", 0, 256)]
         + [("cfg5", i, k) for k in (64, 256) for i in range(4)])


def case_id(cfg: str, index: int, k: int) -> str:
    return f"{cfg}_i{index}_k{k}" if cfg == "cfg5" else f"{cfg}_k{k}"


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def histogram_digest(keys: np.ndarray, counts: np.ndarray) -> str:
    return sha(keys.astype("<u4"), counts.astype("<u4"))


def run_case(cfg_name: str, index: int, k: int) -> dict:
    ref, port = Oracle("reference"), Oracle("port")
    cfg = CONFIGS[cfg_name]
    img = cfg.image(index)
    P = cfg.pixels
    t0 = time.time()
    h = ref.build_histogram(img)
    r = ref.run_wsm(h.keys, h.counts, P, k, mode=1, eps=EPSILON, cap=HARD_CAP, seed=INIT_SEED)
    mapped, _ = ref.map_pixels(img, r.centers)
    m = ref.mse(img, mapped)
    t1 = time.time()
    pmapped, idx = port.map_pixels(img, r.centers)
    assert np.array_equal(pmapped, mapped), "port map_pixels disagrees with the reference"
    return {
        "config": cfg_name, "image": index, "k": k, "pixels": P, "n_unique": int(len(h.keys)),
        "histogram_sha256": histogram_digest(h.keys, h.counts),
        "iterations": int(r.iterations), "dist_evals": int(r.dist_evals),
        "sse": float(r.sse).hex(), "sse_history": [float(x).hex() for x in r.sse_history],
        "palette": [float(x).hex() for x in r.centers.reshape(-1)],
        "mse": float(m).hex(),
        "mapped_sha256": sha(mapped), "index_sha256": sha(idx),
        "reference_seconds": round(t1 - t0, 2),
    }


def main():
    out = {"generator": "tests/golden/make_full_golden.py", "oracle": "oracle/_ref (reference headers, g++ -O2)",
           "termination": f"convergent(eps={EPSILON}, cap={HARD_CAP})", "init_seed": INIT_SEED, "cases": {}}
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        futs = {ex.submit(run_case, *c): case_id(*c) for c in CASES}
        for f in cf.as_completed(futs):
            name = futs[f]
            out["cases"][name] = f.result()
            c = out["cases"][name]
            print(f"{name}: N'={c['n_unique']} iters={c['iterations']} evals={c['dist_evals']} "
                  f"mse={float.fromhex(c['mse']):.4f} ({c['reference_seconds']} s)", flush=True)
    out["cases"] = dict(sorted(out["cases"].items()))
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
