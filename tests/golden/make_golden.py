"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Runs oracle/_ref/libcolorq_ref.so (the reference colorq headers compiled in
place by oracle/Makefile) on small seeded inputs and stores its outputs as
.npz fixtures. Regenerate with:  python tests/golden/make_golden.py
Needs /root/reference only at build time of oracle/_ref; the fixtures are
committed so the tests never read /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1011_0093_b200.configs import gmm_image, uniform_image, value_noise_image  # noqa: E402

CASES = {
    # name: (image factory, k, mode, max_iters, seed)
    "gmm64x48_k8_fixed12": (lambda: gmm_image(64, 48, 12, 101), 8, 0, 12, 3),
    "gmm96x64_k16_conv": (lambda: gmm_image(96, 64, 16, 7), 16, 1, 0, 1),
    "gmm128x64_k32_conv": (lambda: gmm_image(128, 64, 32, 8), 32, 1, 0, 5),
    "noise128_k24_conv": (lambda: value_noise_image(128, 128, 13, cells=(64, 32, 16, 8)), 24, 1, 0, 2),
    "uniform96x80_k64_fixed6": (lambda: uniform_image(96, 80, 14), 64, 0, 6, 9),
}


def main():
    ref = Oracle("reference")
    for name, (make, k, mode, iters, seed) in CASES.items():
        img = make()
        P = img.shape[0] * img.shape[1]
        h = ref.build_histogram(img)
        init = ref.init_centers(h.keys, k, seed)
        r = ref.run_wsm(h.keys, h.counts, P, k, mode=mode, max_iters=iters, eps=1e-4, cap=100, seed=seed,
                        trajectory=True)
        mapped, _ = ref.map_pixels(img, r.centers)
        m = ref.mse(img, mapped)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"), image=img, k=k, mode=mode, max_iters=iters, seed=seed,
            keys=h.keys, counts=h.counts, weights=h.weights, init_centers=init, centers=r.centers,
            iterations=r.iterations, sse=r.sse, dist_evals=r.dist_evals, sse_history=r.sse_history,
            trajectory=r.trajectory, mapped=mapped, mse=m)
        print(f"{name}: P={P} N'={len(h.keys)} iters={r.iterations} evals={r.dist_evals} mse={m:.4f}")
    # hash / prime known answers (histogram_test.cpp:16-44) and a raw mt19937_64 stream
    np.savez_compressed(
        os.path.join(HERE, "kat.npz"),
        mt64_seed1=ref.mt64_stream(1, 64), mt64_seed5489=ref.mt64_stream(5489, 16),
        next_prime_in=np.array([2, 10, 131072, 786433], np.uint64),
        next_prime_out=np.array([ref._f("next_prime")(int(x)) for x in (2, 10, 131072, 786433)], np.uint64))


if __name__ == "__main__":
    main()
