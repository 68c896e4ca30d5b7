"""CPU-only: pin the oracle before trusting it.

* the C restatement (oracle/wsm_oracle.c, "port") against the golden vectors
  generated from the unmodified reference (tests/golden/*.npz);
* the port against the reference compiled in place (oracle/_ref) on fresh
  seeded inputs, bit for bit;
* the reference's own known-answer unit tests for the hot path
  (histogram_test.cpp, kmeans_test.cpp, imageio_test.cpp, metrics_test.cpp),
  restated against the port.
"""
import glob
import os

import numpy as np
import pytest

from paper_1011_0093_b200.configs import CONFIGS, gmm_image, uniform_image, value_noise_image

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*_*.npz")))
GOLDEN = [g for g in GOLDEN if not g.endswith("kat.npz")]


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(g)[:-4] for g in GOLDEN])
def test_port_matches_golden(path, port):
    g = np.load(path)
    img = g["image"]
    P = img.shape[0] * img.shape[1]
    h = port.build_histogram(img)
    np.testing.assert_array_equal(h.keys, g["keys"])
    np.testing.assert_array_equal(h.counts, g["counts"])
    np.testing.assert_array_equal(h.weights, g["weights"])
    k, seed = int(g["k"]), int(g["seed"])
    np.testing.assert_array_equal(port.init_centers(h.keys, k, seed), g["init_centers"])
    r = port.run_wsm(h.keys, h.counts, P, k, mode=int(g["mode"]), max_iters=int(g["max_iters"]), eps=1e-4, cap=100,
                     seed=seed, trajectory=True)
    assert r.iterations == int(g["iterations"])
    assert r.dist_evals == int(g["dist_evals"])
    np.testing.assert_array_equal(r.centers, g["centers"])
    np.testing.assert_array_equal(r.sse_history, g["sse_history"])
    np.testing.assert_array_equal(r.trajectory, g["trajectory"])
    mapped, idx = port.map_pixels(img, r.centers)
    np.testing.assert_array_equal(mapped, g["mapped"])
    assert port.mse(img, mapped) == float(g["mse"])


def test_port_known_answer_vectors(port):
    kat = np.load(os.path.join(os.path.dirname(__file__), "golden", "kat.npz"))
    np.testing.assert_array_equal(port.mt64_stream(1, 64), kat["mt64_seed1"])
    np.testing.assert_array_equal(port.mt64_stream(5489, 16), kat["mt64_seed5489"])
    # C++ [rand.predef]: the 10000th draw of a default-seeded mt19937_64
    assert int(port.mt64_stream(5489, 10000)[-1]) == 9981545732273789042
    assert kat["next_prime_out"].tolist() == [2, 11, 131101, 786433]


@pytest.mark.parametrize("make,k,mode", [
    (lambda: gmm_image(80, 60, 20, 31), 12, 1),
    (lambda: gmm_image(77, 33, 9, 32), 5, 0),
    (lambda: uniform_image(64, 64, 33), 128, 1),
    (lambda: value_noise_image(96, 96, 34, cells=(48, 24, 12, 6)), 40, 1),
    (lambda: CONFIGS["cfg1"].image(), 32, 1),
])
def test_port_matches_reference(make, k, mode, port, ref):
    img = make()
    P = img.shape[0] * img.shape[1]
    hp, hr = port.build_histogram(img), ref.build_histogram(img)
    np.testing.assert_array_equal(hp.keys, hr.keys)
    np.testing.assert_array_equal(hp.counts, hr.counts)
    np.testing.assert_array_equal(hp.weights, hr.weights)
    a = port.run_wsm(hp.keys, hp.counts, P, k, mode=mode, max_iters=7, eps=1e-4, cap=100, seed=11, trajectory=True)
    b = ref.run_wsm(hr.keys, hr.counts, P, k, mode=mode, max_iters=7, eps=1e-4, cap=100, seed=11, trajectory=True)
    assert a.iterations == b.iterations and a.dist_evals == b.dist_evals
    np.testing.assert_array_equal(a.centers, b.centers)
    np.testing.assert_array_equal(a.trajectory, b.trajectory)
    np.testing.assert_array_equal(a.sse_history, b.sse_history)
    mp, _ = port.map_pixels(img, a.centers)
    mr, _ = ref.map_pixels(img, b.centers)
    np.testing.assert_array_equal(mp, mr)
    assert port.mse(img, mp) == ref.mse(img, mr)


def test_reference_hash_known_answers(ref):
    # histogram_test.cpp:16-44 — the universal hash is the reference design
    # (SPEC.md:138); pinned here for completeness of the oracle.
    h = ref._f("universal_hash")
    assert h(12, 200, 9, 7, 0, 0, 0) == 0
    assert h(255, 255, 255, 7, 1, 1, 1) == 765 % 7
    rng = np.random.default_rng(99)
    for _ in range(50):
        m = int(ref._f("next_prime")(int(2 + rng.integers(0, 5000000))))
        a = [int(rng.integers(0, m)) for _ in range(3)]
        c = [int(v) for v in rng.integers(0, 256, 3)]
        assert h(*c, m, *a) == (a[0] * c[0] + a[1] * c[1] + a[2] * c[2]) % m
    # hash parameters never change colors, counts or order (histogram_test.cpp:99-108)
    img = gmm_image(40, 40, 60, 23)
    a = ref.build_histogram(img, 100, 1)
    b = ref.build_histogram(img, 5000, 999)
    np.testing.assert_array_equal(a.keys, b.keys)
    np.testing.assert_array_equal(a.counts, b.counts)


def test_histogram_known_answers(port):
    # histogram_test.cpp:46-61
    h1 = port.build_histogram(np.array([[4, 5, 6]], np.uint8))
    assert len(h1.keys) == 1 and h1.weights[0] == 1.0 and h1.counts[0] == 1
    img = np.array([[0, 0, 0], [0, 0, 0], [255, 255, 255], [0, 0, 0]], np.uint8)
    h = port.build_histogram(img)
    assert h.keys.tolist() == [0, 0xFFFFFF]
    assert h.weights.tolist() == [0.75, 0.25]
    with pytest.raises(ValueError):
        port.build_histogram(np.zeros((0, 3), np.uint8))


def test_sort_means_boundary_and_k1(ref):
    # kmeans_test.cpp:82-100 — prev = 1, d = 4 exactly: skipped without evaluation
    keys = np.array([1 << 16], np.uint32)
    counts = np.array([1], np.uint32)
    lab, sse, evals, D, order = ref.sort_means_step(keys, counts, 1, np.array([[0.0, 0, 0], [2.0, 0, 0]]),
                                                    np.zeros(1, np.int32))
    assert D[0, 1] == 4.0 and lab[0] == 0 and evals == 1 and sse == 1.0
    # kmeans_test.cpp:102-111 — k = 1: N evaluations
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 1 << 24, 64, dtype=np.uint32)
    keys = np.unique(keys)
    _, _, evals, _, _ = ref.sort_means_step(keys, np.ones_like(keys), len(keys), np.array([[10.0, 20, 30]]),
                                            np.zeros(len(keys), np.int32))
    assert evals == len(keys)


def test_midpoint_quirk(ref, port):
    """assign_sort_means != assign_naive at an exact midpoint with t < p
    (SURVEY.md §8(c) divergence 1): the label oracle is sort-means."""
    keys = np.array([10 << 16, 20 << 16, 30 << 16, 0], np.uint32)
    counts = np.ones(4, np.uint32)
    C = np.array([[10.0, 0, 0], [30.0, 0, 0], [200.0, 0, 0]])
    lab, _, evals, _, _ = ref.sort_means_step(keys, counts, 4, C, np.array([1, 1, 1, 0], np.int32))
    assert lab.tolist() == [0, 1, 1, 0] and evals == 5
    X = np.array([[10.0, 0, 0], [20.0, 0, 0], [30.0, 0, 0], [0.0, 0, 0]])
    naive = np.zeros(4, np.int32)
    port._f("assign_naive")(X.ctypes.data_as(port._f("assign_naive").argtypes[0]), 4,
                            C.ctypes.data_as(port._f("assign_naive").argtypes[2]), 3,
                            naive.ctypes.data_as(port._f("assign_naive").argtypes[4]))
    assert naive.tolist() == [0, 0, 1, 0]


def test_update_centers_known_answers(port, ref):
    # kmeans_test.cpp:177-192: weighted mean 63.75; equal weights -> midpoint 127.5
    keys = np.array([0, 0xFFFFFF], np.uint32)
    out = ref.update_centers(keys, np.array([3, 1], np.uint32), 4, np.zeros(2, np.int32), np.array([[1.0, 1, 1]]))
    assert out[0, 0] == pytest.approx(63.75, rel=1e-12)
    out = port.update_centers(keys, np.array([1, 1], np.uint32), 2, np.zeros(2, np.int32), np.array([[1.0, 1, 1]]))
    assert out[0].tolist() == [127.5, 127.5, 127.5]
    # kmeans_test.cpp:194-208: the empty cluster is re-seeded at the farthest point
    keys = np.array([0, 10 << 16, 200 << 16], np.uint32)
    prev = np.array([[5.0, 0, 0], [999.0, 999, 999]])
    for o in (port, ref):
        nxt = o.update_centers(keys, np.array([3, 3, 4], np.uint32), 10, np.zeros(3, np.int32), prev)
        assert nxt[1].tolist() == [200.0, 0.0, 0.0]


def test_map_and_mse_known_answers(port, ref):
    img = gmm_image(16, 16, 4, 3)
    out, idx = port.map_pixels(img, np.zeros((1, 3)))
    assert not out.any() and not idx.any()  # imageio_test.cpp:91-97
    h = port.build_histogram(img)
    out, _ = port.map_pixels(img, h.colors)
    np.testing.assert_array_equal(out, img)  # imageio_test.cpp:99-105
    black = np.zeros((8, 8, 3), np.uint8)
    white = np.full((8, 8, 3), 255, np.uint8)
    assert port.mse(black, white) == 195075.0 == ref.mse(black, white)  # metrics_test.cpp:14-24
    rng = np.random.default_rng(11)
    pal = rng.uniform(0, 255, (8, 3))
    a, _ = port.map_pixels(img, pal)
    b, _ = ref.map_pixels(img, pal)
    np.testing.assert_array_equal(a, b)
    with pytest.raises(ValueError):
        port.map_pixels(img, np.zeros((0, 3)))


def test_run_wsm_invariants(port):
    img = gmm_image(64, 64, 20, 15)
    h = port.build_histogram(img)
    r = port.run_wsm(h.keys, h.counts, 4096, 16, mode=0, max_iters=12, seed=4)
    assert r.iterations == 12
    assert np.all(np.diff(r.sse_history) <= 1e-9)  # kmeans_test.cpp:250-257
    r = port.run_wsm(h.keys, h.counts, 4096, len(h.keys), mode=1, seed=1)
    assert r.iterations == 1 and r.sse == 0.0  # kmeans_test.cpp:242-248
    with pytest.raises(ValueError):
        port.run_wsm(h.keys, h.counts, 4096, len(h.keys) + 1, mode=1)


# --------------------------------------------------------------------------- full-size pin
# The port against the reference's own full convergent runs on the BASELINE
# configs (tests/golden/full_configs.json, generated from oracle/_ref by
# tests/golden/make_full_golden.py): the largest inputs the GPU tests check.
FULL = os.path.join(os.path.dirname(__file__), "golden", "full_configs.json")


@pytest.mark.parametrize("case", ["cfg2_k256", "cfg2_k64", "cfg3_k256", "cfg4_k256", "cfg5_i3_k256"])
def test_port_matches_reference_full_configs(case, port):
    import hashlib
    import json

    g = json.load(open(FULL))["cases"][case]
    img = CONFIGS[g["config"]].image(g["image"])
    P = g["pixels"]
    h = port.build_histogram(img)
    dig = hashlib.sha256(h.keys.astype("<u4").tobytes() + h.counts.astype("<u4").tobytes()).hexdigest()
    assert len(h.keys) == g["n_unique"] and dig == g["histogram_sha256"]
    r = port.run_wsm(h.keys, h.counts, P, g["k"], mode=1, eps=1e-4, cap=100, seed=1)
    assert r.iterations == g["iterations"]
    assert r.dist_evals == g["dist_evals"]
    np.testing.assert_array_equal(r.centers.reshape(-1), np.array([float.fromhex(x) for x in g["palette"]]))
    np.testing.assert_array_equal(r.sse_history, np.array([float.fromhex(x) for x in g["sse_history"]]))
    mapped, idx = port.map_pixels(img, r.centers)
    assert hashlib.sha256(mapped.tobytes()).hexdigest() == g["mapped_sha256"]
    assert hashlib.sha256(idx.tobytes()).hexdigest() == g["index_sha256"]
    assert port.mse(img, mapped) == float.fromhex(g["mse"])
