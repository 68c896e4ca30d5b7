"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): histogram / unique colors / weights / labels /
dist_evals / map / MSE bit-exact; centers and SSE within 1e-6 relative
(bit-exact centers expected whenever P is a power of two — SURVEY.md §8(c)).
"""
import os
import subprocess

import numpy as np
import pytest

from paper_1011_0093_b200 import api
from paper_1011_0093_b200.configs import CONFIGS, gmm_image, uniform_image, value_noise_image

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CENTER_RTOL = 1e-6  # BASELINE.json tolerance for centers / MSE
SSE_RTOL = 1e-9     # moment-form SSE vs sequential FP64 sum


def _cases():
    return {
        "gmm96x64": lambda: gmm_image(96, 64, 16, 7),            # P = 6144 (2^11 * 3)
        "gmm128x64": lambda: gmm_image(128, 64, 32, 8),          # P = 8192 (power of two)
        "gmm101x77": lambda: gmm_image(101, 77, 24, 9),          # tail pixels, odd P
        "noise256": lambda: value_noise_image(256, 256, 11, cells=(64, 32, 16, 8)),
        "uniform256": lambda: uniform_image(256, 256, 12),
        "cfg1": lambda: CONFIGS["cfg1"].image(),
        "cfg2": lambda: CONFIGS["cfg2"].image(),
    }


CASES = _cases()


@pytest.fixture(scope="module")
def images():
    return {k: f() for k, f in CASES.items()}


def _pow2(n):
    return n & (n - 1) == 0


# --------------------------------------------------------------------------- histogram
@pytest.mark.parametrize("case", list(CASES))
def test_histogram_bit_exact(case, images, port):
    img = images[case]
    h = api.build_histogram(img)
    o = port.build_histogram(img)
    assert h.size() == len(o.keys)
    np.testing.assert_array_equal(h.keys, o.keys)       # first-occurrence order
    np.testing.assert_array_equal(h.counts, o.counts)
    np.testing.assert_array_equal(h.weights, o.weights)  # count * (1/P), bit-exact
    flat = img.reshape(-1, 3).astype(np.uint32)
    keys = (flat[:, 0] << 16) | (flat[:, 1] << 8) | flat[:, 2]
    np.testing.assert_array_equal(keys[h.first_index], h.keys)
    assert np.all(np.diff(h.first_index.astype(np.int64)) > 0)


def test_histogram_known_answers():
    # histogram_test.cpp:46-61
    h1 = api.build_histogram(np.array([[[4, 5, 6]]], np.uint8))
    assert h1.size() == 1 and h1.weights[0] == 1.0 and h1.counts[0] == 1
    img = np.array([[[0, 0, 0], [0, 0, 0]], [[255, 255, 255], [0, 0, 0]]], np.uint8)
    h = api.build_histogram(img)
    assert h.size() == 2
    assert tuple(h.colors[0]) == (0, 0, 0)
    assert h.weights[0] == 0.75 and h.weights[1] == 0.25
    with pytest.raises(ValueError):
        api.build_histogram(np.zeros((0, 3), np.uint8))


@pytest.mark.parametrize("n", [1, 15, 16, 17, 4095, 4096, 4097, 70001])
def test_histogram_ragged_sizes(n, port):
    rng = np.random.default_rng(n)
    img = rng.integers(0, 4, size=(n, 3), dtype=np.uint8) * 60  # heavy repeats + runs
    img[: n // 3] = img[0]
    h = api.build_histogram(img)
    o = port.build_histogram(img)
    np.testing.assert_array_equal(h.keys, o.keys)
    np.testing.assert_array_equal(h.counts, o.counts)


def test_histogram_permutation_and_repeat(port):
    img = gmm_image(64, 64, 8, 3)
    a = api.build_histogram(img)
    perm = np.random.default_rng(3).permutation(img.reshape(-1, 3))
    b = api.build_histogram(perm)
    assert dict(zip(a.keys.tolist(), a.counts.tolist())) == dict(zip(b.keys.tolist(), b.counts.tolist()))
    # table is returned to zero: a second call sees identical results
    c = api.build_histogram(img)
    np.testing.assert_array_equal(a.counts, c.counts)
    np.testing.assert_array_equal(a.keys, c.keys)


def test_histogram_all_colors():
    # every 24-bit color exactly once, in key order -> N' = 2^24
    keys = np.arange(1 << 24, dtype=np.uint32)
    img = np.stack([(keys >> 16) & 255, (keys >> 8) & 255, keys & 255], 1).astype(np.uint8)
    h = api.build_histogram(img)
    assert h.size() == 1 << 24
    np.testing.assert_array_equal(h.keys, keys)
    assert np.all(h.counts == 1)


# --------------------------------------------------------------------------- WSM loop
def _run_both(img, k, port, term=("conv", 1e-4, 100), seed=1, traj=True):
    h = api.build_histogram(img)
    P = img.shape[0] * img.shape[1]
    if term[0] == "conv":
        t = api.Termination.convergent(term[1], term[2])
        o = port.run_wsm(h.keys, h.counts, P, k, mode=1, eps=term[1], cap=term[2], seed=seed, trajectory=traj)
    else:
        t = api.Termination.fixed(term[1])
        o = port.run_wsm(h.keys, h.counts, P, k, mode=0, max_iters=term[1], seed=seed, trajectory=traj)
    g = api.run_wsm(h, k, t, seed, trajectory=traj, labels=True)
    return h, g, o, P


@pytest.mark.parametrize("case,k", [("gmm96x64", 8), ("gmm128x64", 16), ("gmm101x77", 32), ("noise256", 64),
                                    ("uniform256", 256), ("cfg1", 32), ("cfg2", 64), ("cfg2", 256)])
def test_run_wsm_matches_oracle(case, k, images, port):
    img = images[case]
    h, g, o, P = _run_both(img, k, port)
    assert g.report.iterations == o.iterations
    np.testing.assert_allclose(g.report.sse_history, o.sse_history, rtol=SSE_RTOL)
    if _pow2(P):
        np.testing.assert_array_equal(g.palette, o.centers)
        np.testing.assert_array_equal(g.trajectory, o.trajectory)
        assert g.report.dist_evals == o.dist_evals
    else:
        np.testing.assert_allclose(g.palette, o.centers, rtol=CENTER_RTOL)
        np.testing.assert_allclose(g.trajectory, o.trajectory, rtol=CENTER_RTOL)
        # the ~1e-13 center differences never move a break decision here: exact
        assert g.report.dist_evals == o.dist_evals


def test_run_wsm_fixed_and_seeds(images, port):
    for seed in (1, 2, 99):
        h, g, o, P = _run_both(images["gmm128x64"], 12, port, term=("fixed", 9), seed=seed)
        assert g.report.iterations == 9 == o.iterations
        np.testing.assert_array_equal(g.palette, o.centers)
        assert g.report.dist_evals == o.dist_evals


def test_run_wsm_k_equals_n_and_k1(port):
    img = gmm_image(16, 16, 4, 3)
    h = api.build_histogram(img)
    r = api.run_wsm(h, h.size(), api.Termination.convergent(), 1)
    assert r.report.iterations == 1 and r.report.sse == 0.0  # kmeans_test.cpp:242-248
    r1 = api.run_wsm(h, 1, api.Termination.fixed(1), 1)
    assert r1.report.dist_evals == h.size()  # kmeans_test.cpp:102-111
    with pytest.raises(ValueError):
        api.run_wsm(h, h.size() + 1, api.Termination.fixed(2), 1)  # kmeans.hpp:54-56


def test_teacher_forced_iterations(images, port, ref):
    """Per-iteration labels and evals given the oracle's centers."""
    img = images["gmm128x64"]
    k = 16
    h = api.build_histogram(img)
    P = img.shape[0] * img.shape[1]
    o = port.run_wsm(h.keys, h.counts, P, k, mode=0, max_iters=10, seed=5, trajectory=True, labels=True)
    init = port.init_centers(h.keys, k, 5)
    pairs = k * (k - 1) // 2
    for it in range(1, 11):
        C_in = init if it == 1 else o.trajectory[it - 2]
        lab_in = np.zeros(h.size(), np.int32) if it == 1 else o.label_trajectory[it - 2]
        nxt, lab, rep = api.wsm_iterate(h, C_in, lab_in, api.Termination.fixed(1), dense_first=(it == 1))
        np.testing.assert_array_equal(lab, o.label_trajectory[it - 1])
        np.testing.assert_array_equal(nxt, o.trajectory[it - 1])
        _, sse, evals, _, _ = ref.sort_means_step(h.keys, h.counts, P, C_in, lab_in)
        assert rep.dist_evals == pairs + evals
        assert rep.sse == pytest.approx(sse, rel=SSE_RTOL)


def test_empty_cluster_reseed(port, ref):
    """update_centers' empty-cluster branch (kmeans.hpp:272-294)."""
    img = gmm_image(64, 64, 6, 21)
    h = api.build_histogram(img)
    P = 64 * 64
    rng = np.random.default_rng(0)
    C_in = h.colors[rng.choice(h.size(), 8, replace=False)].copy()
    C_in[2] = (999.0, 999.0, 999.0)   # owns nothing
    C_in[5] = (-500.0, 0.0, 0.0)      # owns nothing
    lab0 = np.zeros(h.size(), np.int32)
    lab_ref, _, _, _, _ = ref.sort_means_step(h.keys, h.counts, P, C_in, lab0)
    nxt_ref = ref.update_centers(h.keys, h.counts, P, lab_ref, C_in)
    nxt, lab, rep = api.wsm_iterate(h, C_in, lab0, api.Termination.fixed(1))
    np.testing.assert_array_equal(lab, lab_ref)
    np.testing.assert_array_equal(nxt, nxt_ref)
    assert rep.empty_events == 2


def test_midpoint_tie_quirk(ref):
    """Sort-means keeps p when x is the exact midpoint and t < p."""
    keys = np.array([(10 << 16), (20 << 16), (30 << 16), (0 << 16)], np.uint32)  # r = 10, 20, 30, 0
    counts = np.ones(4, np.uint32)
    h = api.ColorHistogram(keys, counts, counts / 4.0, 4)
    C_in = np.array([[10.0, 0, 0], [30.0, 0, 0], [200.0, 0, 0]])
    lab_in = np.array([1, 1, 1, 0], np.int32)  # x = 20 is the midpoint of c0 = 10 and c1 = 30, starts at p = 1
    lab_ref, sse, evals, _, _ = ref.sort_means_step(keys, counts, 4, C_in, lab_in)
    _, lab, rep = api.wsm_iterate(h, C_in, lab_in, api.Termination.fixed(1))
    np.testing.assert_array_equal(lab, lab_ref)
    assert lab[1] == 1  # not the naive lowest index 0
    assert rep.dist_evals == 3 + evals


# --------------------------------------------------------------------------- map + mse
@pytest.mark.parametrize("k", [1, 7, 64, 256])
def test_map_pixels_matches_oracle(k, images, port):
    img = images["noise256"]
    rng = np.random.default_rng(k)
    pal = rng.uniform(-3.0, 258.0, size=(k, 3))
    pal[0] = (12.5, 99.5, 200.49999)  # half-way rounding (lround: away from zero)
    out, idx, err = api.map_pixels_indexed(img, pal)
    ref_out, ref_idx = port.map_pixels(img, pal)
    np.testing.assert_array_equal(out, ref_out)
    np.testing.assert_array_equal(idx, ref_idx)
    assert err / (img.size // 3) == port.mse(img, ref_out)


def test_map_pixels_edge_cases(port):
    img = gmm_image(16, 16, 4, 3)
    np.testing.assert_array_equal(api.map_pixels(img, np.zeros((1, 3))), np.zeros_like(img))
    h = api.build_histogram(img)
    np.testing.assert_array_equal(api.map_pixels(img, h.colors), img)  # imageio_test.cpp:99-105
    with pytest.raises(ValueError):
        api.map_pixels(img, np.zeros((0, 3)))
    pal = np.array([[10.0, 10, 10], [10.0, 10, 10], [200.0, 0, 0]])  # duplicate entries: lowest index wins
    _, idx, _ = api.map_pixels_indexed(img, pal)
    assert not np.any(idx == 1)


def test_mse_known_answers(port):
    black = np.zeros((8, 8, 3), np.uint8)
    white = np.full((8, 8, 3), 255, np.uint8)
    assert api.mse(black, white) == 195075.0
    a = gmm_image(31, 17, 5, 4)
    b = gmm_image(31, 17, 5, 5)
    assert api.mse(a, b) == port.mse(a, b) == api.mse(b, a)
    with pytest.raises(ValueError):
        api.mse(black, np.zeros((4, 4, 3), np.uint8))


# --------------------------------------------------------------------------- end to end
@pytest.mark.parametrize("case,k", [("gmm96x64", 16), ("gmm101x77", 8), ("cfg1", 32), ("cfg2", 256), ("cfg2", 64),
                                    ("uniform256", 64)])
def test_quantize_end_to_end(case, k, images, port):
    img = images[case]
    q = api.quantize(img, k, api.Termination.convergent(1e-4, 100), seed=1)
    h = port.build_histogram(img)
    P = img.shape[0] * img.shape[1]
    o = port.run_wsm(h.keys, h.counts, P, k, mode=1, eps=1e-4, cap=100, seed=1)
    assert q.report.iterations == o.iterations
    assert q.report.n_unique == len(h.keys)
    ref_out, ref_idx = port.map_pixels(img, o.centers)
    if _pow2(P):
        np.testing.assert_array_equal(q.palette, o.centers)
        np.testing.assert_array_equal(q.mapped, ref_out)
        np.testing.assert_array_equal(q.index_map, ref_idx)
        assert q.report.mse == port.mse(img, ref_out)
    else:
        np.testing.assert_allclose(q.palette, o.centers, rtol=CENTER_RTOL)
        assert q.report.mse == pytest.approx(port.mse(img, ref_out), rel=CENTER_RTOL)
    # self-consistency of the fused outputs
    mine, my_idx = port.map_pixels(img, q.palette)
    np.testing.assert_array_equal(q.mapped, mine)
    np.testing.assert_array_equal(q.index_map, my_idx)
    assert q.report.mse == port.mse(img, q.mapped)


def test_quantize_batch_lanes(port):
    """Config 5 path: several images in flight (cqb_quantize_batch). Each
    image's palette, iterations, dist_evals, MSE, index map and mapped raster
    equal the single-image call and the oracle."""
    import torch

    imgs = [gmm_image(128, 64, 24, 300 + i) for i in range(7)]  # P = 8192: bit-exact centers
    dev = [torch.from_numpy(im.reshape(-1)).cuda() for im in imgs]
    idx = [torch.empty(im.shape[0] * im.shape[1], dtype=torch.uint8, device="cuda") for im in imgs]
    out = [torch.empty(im.size, dtype=torch.uint8, device="cuda") for im in imgs]
    term = api.Termination.convergent(1e-4, 100)
    for lanes in (3, 4):
        pal, reps = api.quantize_batch_device(dev, 16, term, seed=1, lanes=lanes, index_out=idx, mapped_out=out)
        for i, im in enumerate(imgs):
            q = api.quantize(im, 16, term, seed=1)
            np.testing.assert_array_equal(pal[i], q.palette)
            assert reps[i].iterations == q.report.iterations
            assert reps[i].dist_evals == q.report.dist_evals
            assert reps[i].mse == q.report.mse
            np.testing.assert_array_equal(idx[i].cpu().numpy(), q.index_map.reshape(-1))
            np.testing.assert_array_equal(out[i].cpu().numpy(), q.mapped.reshape(-1))
    h = port.build_histogram(imgs[5])
    o = port.run_wsm(h.keys, h.counts, 8192, 16, mode=1, eps=1e-4, cap=100, seed=1)
    np.testing.assert_array_equal(pal[5], o.centers)
    assert reps[5].iterations == o.iterations and reps[5].dist_evals == o.dist_evals


def test_generate_palette_api(images):
    img = images["gmm96x64"]
    a = api.generate_palette(img, api.MethodParams("wsm-c"), 16, 1)
    b = api.generate_palette(img, api.MethodParams("wsm-c"), 16, 1)
    np.testing.assert_array_equal(a.palette, b.palette)  # cli_test.cpp:123-130 determinism
    assert a.report.method == "wsm-c"
    with pytest.raises(api.UnknownMethodError):
        api.generate_palette(img, api.MethodParams("mc"), 16, 1)
    with pytest.raises(ValueError):
        api.generate_palette(img, api.MethodParams("wsm"), 0, 1)


def test_cpp_shim():
    exe = os.path.join(ROOT, "build", "shim_test")
    assert os.path.exists(exe), "build/shim_test missing (run make)"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


# --------------------------------------------------------------------------- full-size properties
@pytest.mark.slow
def test_cfg4_properties(port):
    img = CONFIGS["cfg4"].image()
    P = img.shape[0] * img.shape[1]
    h = api.build_histogram(img)
    o = port.build_histogram(img)
    np.testing.assert_array_equal(h.keys, o.keys)
    np.testing.assert_array_equal(h.counts, o.counts)
    assert int(h.counts.sum(dtype=np.uint64)) == P
    q = api.quantize(img, 256, api.Termination.convergent(1e-4, 100), seed=1)
    assert q.report.n_unique == h.size()
    hist = np.array(q.report.sse_history)
    assert np.all(np.diff(hist) <= 1e-9 * hist[:-1])  # SSE nonincreasing
    # mapping is idempotent and consistent with the palette
    again, idx2, _ = api.map_pixels_indexed(q.mapped, q.palette)
    np.testing.assert_array_equal(again, q.mapped)
    assert q.report.mse == pytest.approx(api.mse(img, q.mapped), rel=0, abs=0)


@pytest.mark.slow
def test_cfg3_full_size(port):
    """Config 3 (4096^2 value noise, ~2.6M unique colors) at full size:
    histogram bit-exact, three fixed iterations against the oracle (exact:
    P is a power of two), and the convergent run's size-independent
    properties (nonincreasing SSE, idempotent mapping, exact MSE)."""
    img = CONFIGS["cfg3"].image()
    P = img.shape[0] * img.shape[1]
    h = api.build_histogram(img)
    o = port.build_histogram(img)
    np.testing.assert_array_equal(h.keys, o.keys)
    np.testing.assert_array_equal(h.counts, o.counts)
    q3 = api.quantize(img, 256, api.Termination.fixed(3), seed=1, index_map=False, mapped=False)
    r3 = port.run_wsm(o.keys, o.counts, P, 256, mode=0, max_iters=3, seed=1)
    np.testing.assert_array_equal(q3.palette, r3.centers)
    assert q3.report.dist_evals == r3.dist_evals
    q = api.quantize(img, 256, api.Termination.convergent(1e-4, 100), seed=1)
    hist = np.array(q.report.sse_history)
    assert np.all(np.diff(hist) <= 1e-9 * hist[:-1])
    again, _, _ = api.map_pixels_indexed(q.mapped, q.palette)
    np.testing.assert_array_equal(again, q.mapped)
    assert q.report.mse == api.mse(img, q.mapped)


@pytest.mark.slow
@pytest.mark.parametrize("k", [64, 256])
def test_cfg5_image_matches_oracle(k, port):
    """Config 5's first image (1024^2 GMM-256, seed 1000) through the batch
    path equals the oracle's full convergent run (P is a power of two)."""
    import torch

    img = CONFIGS["cfg5"].image(0)
    P = img.shape[0] * img.shape[1]
    d = torch.from_numpy(img.reshape(-1)).cuda()
    pal, reps = api.quantize_batch_device([d], k, api.Termination.convergent(1e-4, 100), seed=1, lanes=1)
    h = port.build_histogram(img)
    o = port.run_wsm(h.keys, h.counts, P, k, mode=1, eps=1e-4, cap=100, seed=1)
    assert reps[0].iterations == o.iterations and reps[0].dist_evals == o.dist_evals
    np.testing.assert_array_equal(pal[0], o.centers)


# --------------------------------------------------------------------------- §8(f) f3: KM / KM-C
@pytest.mark.parametrize("case,k,mode", [("gmm128x64", 16, 1), ("gmm128x64", 8, 0), ("gmm96x64", 12, 1),
                                         ("gmm101x77", 8, 1)])
def test_run_km_full_matches_reference(case, k, mode, images, ref):
    """run_km_full (kmeans.hpp:409-426): exhaustive assignment over every
    PIXEL (weight 1/P each) on the device point-set kernels; the P*k
    evaluations per iteration are performed, and the per-cluster sums follow
    the reference's pixel order, so the centers are bit-exact for any P."""
    img = images[case]
    P = img.shape[0] * img.shape[1]
    term = api.Termination.convergent(1e-4, 100) if mode else api.Termination.fixed(7)
    q = api.run_km_full(img, k, term, seed=2)
    o = ref.run_km_full(img, k, mode=mode, max_iters=7, eps=1e-4, cap=100, seed=2)
    assert q.report.iterations == o["iterations"]
    assert q.report.dist_evals == o["dist_evals"] == o["iterations"] * P * k
    np.testing.assert_array_equal(q.palette, o["centers"])
    np.testing.assert_allclose(q.report.sse_history, o["sse_history"], rtol=1e-12)
    g = api.generate_palette(img, api.MethodParams("km-c" if mode else "km", iters=7), k, 2)
    np.testing.assert_array_equal(g.palette, q.palette)
    assert g.report.method == ("km-c" if mode else "km")


# --------------------------------------------------------------------------- §8(f) f4: FKM / FKM-C
@pytest.mark.parametrize("case,k,kp,mode", [("gmm128x64", 16, 8, 1), ("gmm128x64", 24, 4, 0), ("gmm96x64", 12, 8, 1),
                                            ("gmm128x64", 8, 8, 1)])
def test_run_fkm_matches_reference(case, k, kp, mode, images, ref):
    """run_fkm (fast_variants.hpp:20-81) through generate_palette's FKM branch:
    centers, iterations, SSE history and dist_evals (P*k, then P*k' per
    iteration, plus the center-table pairs)."""
    img = images[case]
    P = img.shape[0] * img.shape[1]
    mp = api.MethodParams("fkm-c" if mode else "fkm", iters=6, k_prime=kp)
    q = api.generate_palette(img, mp, k, 4)
    o = ref.run_fkm(img, k, kp, mode=mode, max_iters=6, eps=1e-4, seed=4)
    assert q.report.method == mp.id
    assert q.report.iterations == o["iterations"]
    assert q.report.dist_evals == o["dist_evals"]
    np.testing.assert_array_equal(q.palette, o["centers"])  # pixel-order sums: bit-exact for any P
    np.testing.assert_allclose(q.report.sse_history, o["sse_history"], rtol=1e-12)
    with pytest.raises(api.CqbInvalidArgument):
        api.run_fkm(img, 4, 8)  # k_prime > k (fast_variants.hpp:26)


# --------------------------------------------------------------------------- randomized + large-path parity
def _random_cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for c in range(n):
        kind = c % 4
        w, h = int(rng.integers(1, 140)), int(rng.integers(1, 90))
        if kind == 0:
            img = gmm_image(w, h, int(rng.integers(1, 20)), int(rng.integers(0, 10**6)))
        elif kind == 1:
            img = uniform_image(w, h, int(rng.integers(0, 10**6)))
        elif kind == 2:  # few colors, many duplicates
            pal = rng.integers(0, 256, (int(rng.integers(1, 9)), 3), dtype=np.uint8)
            img = pal[rng.integers(0, pal.shape[0], w * h)].reshape(h, w, 3)
        else:  # a single color
            img = np.broadcast_to(rng.integers(0, 256, 3, dtype=np.uint8), (h, w, 3)).copy()
        out.append(img)
    return out


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_quantize_random_images_match_oracle(seed, port):
    """Randomized images (ragged sizes down to 1 pixel, duplicates, a single
    color) through the full device pipeline - fused small-image prep, loop
    with longest-first chunk order and cell candidates, map epilogue -
    against the oracle: iterations, dist_evals, palette, index map, MSE."""
    rng = np.random.default_rng(100 + seed)
    for img in _random_cases(12, seed):
        P = img.shape[0] * img.shape[1]
        h = port.build_histogram(img)
        n = len(h.keys)
        k = int(rng.integers(1, min(n, 256) + 1))
        mode = int(rng.integers(0, 2))
        term = api.Termination.convergent(1e-4, 100) if mode else api.Termination.fixed(int(rng.integers(1, 12)))
        iters = 10 if mode else term.max_iters
        q = api.quantize(img, k, term, seed=7)
        o = port.run_wsm(h.keys, h.counts, P, k, mode=mode, max_iters=iters, eps=1e-4, cap=100, seed=7)
        assert q.report.iterations == o.iterations, (img.shape, k, mode)
        assert q.report.dist_evals == o.dist_evals, (img.shape, k, mode)
        assert q.report.n_unique == n
        if _pow2(P):
            np.testing.assert_array_equal(q.palette, o.centers)
        else:
            np.testing.assert_allclose(q.palette, o.centers, rtol=CENTER_RTOL, atol=1e-9)
        mine, my_idx = port.map_pixels(img, q.palette)
        np.testing.assert_array_equal(q.mapped, mine)
        np.testing.assert_array_equal(q.index_map, my_idx)
        assert q.report.mse == port.mse(img, q.mapped)


def test_quantize_large_path_matches_oracle(port):
    """P >= 2M pixels takes the dense-table path (4-slice K1, full 128 MiB
    compaction, bitmap scan + rank kernels, PPT=2 loop): a 2048x1024 GMM image
    in fixed-iteration mode against the oracle (bit-exact: P is a power of 2)."""
    img = gmm_image(2048, 1024, 64, 55)
    P = img.shape[0] * img.shape[1]
    q = api.quantize(img, 64, api.Termination.fixed(3), seed=2)
    h = port.build_histogram(img)
    o = port.run_wsm(h.keys, h.counts, P, 64, mode=0, max_iters=3, seed=2)
    assert q.report.n_unique == len(h.keys)
    assert q.report.iterations == 3 and q.report.dist_evals == o.dist_evals
    np.testing.assert_array_equal(q.palette, o.centers)
    mine, my_idx = port.map_pixels(img, q.palette)
    np.testing.assert_array_equal(q.index_map, my_idx)
    assert q.report.mse == port.mse(img, q.mapped)


@pytest.mark.parametrize("case,k", [("cfg2", 256), ("gmm101x77", 8)])
def test_quantize_pinned_outputs_zero_copy(case, k, images, port):
    """Pinned host outputs take the zero-copy path (the map kernel writes them
    over PCIe, results published by one kernel): index map, mapped raster,
    error image and report equal the pageable-buffer path and the oracle."""
    import torch

    img = images[case]
    h, w = img.shape[:2]
    term = api.Termination.convergent(1e-4, 100)
    ref = api.quantize(img, k, term, seed=1, error=True)  # pageable numpy outputs: device buffers + D2H
    pin_idx = torch.empty(h * w, dtype=torch.uint8).pin_memory().numpy().reshape(h, w)
    pin_out = torch.empty(h * w * 3, dtype=torch.uint8).pin_memory().numpy().reshape(h, w, 3)
    pin_idx[:] = 7
    pin_out[:] = 7
    for _ in range(2):  # twice: the staging block and the outputs are rewritten, not stale
        q = api.quantize(img, k, term, seed=1, out_index=pin_idx, out_mapped=pin_out, error=True)
        np.testing.assert_array_equal(q.palette, ref.palette)
        np.testing.assert_array_equal(pin_idx, ref.index_map)
        np.testing.assert_array_equal(pin_out, ref.mapped)
        np.testing.assert_array_equal(q.error, ref.error)
        assert q.report.mse == ref.report.mse and q.report.iterations == ref.report.iterations
        assert q.report.dist_evals == ref.report.dist_evals
        assert list(q.report.sse_history) == list(ref.report.sse_history)
    mine, my_idx = port.map_pixels(img, q.palette)
    np.testing.assert_array_equal(pin_out, mine)


def test_quantize_overlapped_transfers(port):
    """Large images through cqb_quantize_ex: the H2D copy in 8 slices with K1
    counting each slice as it lands, and the outputs copied back per map slice
    on a second stream. Ragged size (not a multiple of 16 x 8 pixels), pinned
    and pageable outputs, error image; equal to the serial path (debug flag
    1 << 19) and to the oracle."""
    import torch

    img = gmm_image(1531, 1373, 64, 77)  # 2.1M pixels: the dense path
    h, w = img.shape[:2]
    term = api.Termination.fixed(4)
    ctx = api.context(0)
    ctx.lib.cqb_set_debug(ctx.h, 1 << 19)
    try:
        ser = api.quantize(img, 64, term, seed=3, error=True)
    finally:
        ctx.lib.cqb_set_debug(ctx.h, 0)
    pin_img = torch.from_numpy(img.reshape(-1).copy()).pin_memory().numpy().reshape(img.shape)
    pin_out = torch.empty(h * w * 3, dtype=torch.uint8).pin_memory().numpy().reshape(h, w, 3)
    for src, out in ((img, None), (pin_img, pin_out)):
        q = api.quantize(src, 64, term, seed=3, error=True, out_mapped=out)
        np.testing.assert_array_equal(q.palette, ser.palette)
        np.testing.assert_array_equal(q.index_map, ser.index_map)
        np.testing.assert_array_equal(q.mapped, ser.mapped)
        np.testing.assert_array_equal(q.error, ser.error)
        assert q.report.dist_evals == ser.report.dist_evals and q.report.mse == ser.report.mse
    hh = port.build_histogram(img)
    o = port.run_wsm(hh.keys, hh.counts, h * w, 64, mode=0, max_iters=4, seed=3)
    assert q.report.n_unique == len(hh.keys) and q.report.dist_evals == o.dist_evals
    np.testing.assert_allclose(q.palette, o.centers, rtol=CENTER_RTOL)
    mine, my_idx = port.map_pixels(img, q.palette)
    np.testing.assert_array_equal(q.index_map, my_idx)
    np.testing.assert_array_equal(q.mapped, mine)


def test_quantize_concurrent_callers(port):
    """Host threads streaming images through the C ABI concurrently (one
    context each): a call that starts while another is in flight skips the
    sliced H2D/K1 overlap (one copy, 4-pass K1). Every caller's outputs equal
    the single-caller run and the oracle's map of its palette."""
    from concurrent.futures import ThreadPoolExecutor

    imgs = [gmm_image(1531, 1373, 64, 90 + i) for i in range(3)]  # dense path, ragged
    term = api.Termination.fixed(3)
    solo = [api.quantize(im, 64, term, seed=5, error=True) for im in imgs]

    def run(j):
        return [api.quantize(imgs[j], 64, term, seed=5, error=True) for _ in range(2)]

    with ThreadPoolExecutor(3) as ex:
        outs = list(ex.map(run, range(3)))
    for j, rs in enumerate(outs):
        for q in rs:
            np.testing.assert_array_equal(q.palette, solo[j].palette)
            np.testing.assert_array_equal(q.index_map, solo[j].index_map)
            np.testing.assert_array_equal(q.mapped, solo[j].mapped)
            np.testing.assert_array_equal(q.error, solo[j].error)
            assert q.report.dist_evals == solo[j].report.dist_evals and q.report.mse == solo[j].report.mse
    mine, my_idx = port.map_pixels(imgs[0], solo[0].palette)
    np.testing.assert_array_equal(solo[0].index_map, my_idx)


@pytest.mark.parametrize("k", [7, 255, 256])
def test_coarse_map_table_matches_lut_path(k, port):
    """Large images map through the coarse 4x4x8-cell table (pure cells from
    shared memory, byte 255 = gather from the LUT; with K = 256 the pure cells
    of index 255 gather too). Index map, mapped raster and error image equal
    the per-pixel LUT path (debug flag 1 << 21) and the oracle's map."""
    img = value_noise_image(2048, 1024, 11)
    term = api.Termination.fixed(2)
    ctx = api.context(0)
    ctx.lib.cqb_set_debug(ctx.h, 1 << 21)
    try:
        lut = api.quantize(img, k, term, seed=4, error=True)
    finally:
        ctx.lib.cqb_set_debug(ctx.h, 0)
    q = api.quantize(img, k, term, seed=4, error=True)
    np.testing.assert_array_equal(q.palette, lut.palette)
    np.testing.assert_array_equal(q.index_map, lut.index_map)
    np.testing.assert_array_equal(q.mapped, lut.mapped)
    np.testing.assert_array_equal(q.error, lut.error)
    assert q.report.mse == lut.report.mse
    mine, my_idx = port.map_pixels(img, q.palette)
    np.testing.assert_array_equal(q.index_map, my_idx)
    np.testing.assert_array_equal(q.mapped, mine)
