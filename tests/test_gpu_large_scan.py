"""GPU parity of the large-image loop's difference-form scan (scan_f32e).

Images of P >= 2M pixels run k_wsm_loop<2, ...>: candidates evaluated as
w + a.m from WsmState::rowE (kmeans.hpp:211-236 is the scan it replaces),
moving samples' moment deltas queued per warp, and - for sparse sample sets,
N' < P/2 - the longest-first chunk order. The full BASELINE configs are in
test_gpu_full_configs.py; these cases aim at what those do not reach: exact
ties between candidates (lattice colors, where the FP32 certificate must hand
the point to the FP64 scan and its lexicographic tie rule), every FP32 screen
switched off, and both chunk orders on the same image.
"""
import numpy as np
import pytest

from paper_1011_0093_b200 import api
from paper_1011_0093_b200.configs import gmm_image, value_noise_image

pytestmark = pytest.mark.gpu

DBG_NO_F32 = 1 << 17          # wsm.cuh: FP64 scans only
DBG_NO_SCHED_LARGE = 1 << 24  # wsm.cuh: large path without the longest-first order


def _lattice_image(w, h, step, seed):
    """Colors on the lattice {0, step, 2 step, ...}^3, i.i.d. per pixel: centers
    and points sit at symmetric positions, so equal distances are common."""
    rng = np.random.default_rng(seed)
    levels = np.arange(0, 256, step, dtype=np.uint8)
    return levels[rng.integers(0, len(levels), size=(h, w, 3))]


def _check_against_oracle(img, k, term_args, seed, port):
    P = img.shape[0] * img.shape[1]
    mode, a, b = term_args
    if mode == "conv":
        term = api.Termination.convergent(a, b)
        kw = dict(mode=1, eps=a, cap=b)
    else:
        term = api.Termination.fixed(a)
        kw = dict(mode=0, max_iters=a)
    q = api.quantize(img, k, term, seed=seed)
    h = port.build_histogram(img)
    o = port.run_wsm(h.keys, h.counts, P, k, seed=seed, **kw)
    assert q.report.n_unique == len(h.keys)
    assert q.report.iterations == o.iterations
    assert q.report.dist_evals == o.dist_evals
    np.testing.assert_array_equal(q.palette, o.centers)  # P is a power of two: bit-exact
    np.testing.assert_allclose(q.report.sse_history, o.sse_history, rtol=1e-9)
    _, idx = port.map_pixels(img, q.palette)
    np.testing.assert_array_equal(q.index_map, idx)
    return q


@pytest.mark.parametrize("step,k", [(16, 64), (32, 16), (8, 256)])
def test_lattice_colors_with_ties(step, k, port):
    """Lattice colors: candidates at exactly equal distance from a point are the
    rule, not the exception; a tie never certifies in FP32 and the FP64 scan's
    (distance, index) order decides, as in the reference."""
    img = _lattice_image(2048, 1024, step, 1234 + step)
    _check_against_oracle(img, k, ("conv", 1e-4, 100), 3, port)


def test_two_colors_and_one_color(port):
    """Degenerate sample sets on the large path: N' = 2 with K = 2 (every row has
    one entry) and N' = 1 with K = 1 (rows are all tail)."""
    img = np.zeros((1024, 2048, 3), np.uint8)
    img[::2, :, :] = (10, 200, 30)
    _check_against_oracle(img, 2, ("fixed", 3, 0), 1, port)
    img[:] = (7, 7, 7)
    _check_against_oracle(img, 1, ("fixed", 2, 0), 1, port)


def test_fp32_screen_off_is_identical(port):
    """The FP32 screen (difference form included) only ever decides what it can
    certify: with it switched off (FP64 scans only) every output is the same."""
    img = gmm_image(2048, 1024, 48, 77)
    term = api.Termination.convergent(1e-4, 100)
    ctx = api.context(0)
    ctx.lib.cqb_set_debug(ctx.h, DBG_NO_F32)
    try:
        ref = api.quantize(img, 128, term, seed=5)
    finally:
        ctx.lib.cqb_set_debug(ctx.h, 0)
    q = api.quantize(img, 128, term, seed=5)
    assert q.report.iterations == ref.report.iterations
    assert q.report.dist_evals == ref.report.dist_evals
    np.testing.assert_array_equal(q.palette, ref.palette)
    np.testing.assert_array_equal(q.report.sse_history, ref.report.sse_history)
    np.testing.assert_array_equal(q.index_map, ref.index_map)
    assert q.report.mse == ref.report.mse


def test_chunk_order_does_not_change_results(port):
    """A sparse sample set (N' < P/2) takes the longest-first chunk order; the
    order only affects timing (exact integer sums, per-point labels)."""
    img = value_noise_image(2048, 1024, 21)
    P = img.shape[0] * img.shape[1]
    term = api.Termination.convergent(1e-4, 100)
    ctx = api.context(0)
    ctx.lib.cqb_set_debug(ctx.h, DBG_NO_SCHED_LARGE)
    try:
        plain = api.quantize(img, 256, term, seed=9)
    finally:
        ctx.lib.cqb_set_debug(ctx.h, 0)
    q = api.quantize(img, 256, term, seed=9)
    assert q.report.n_unique * 2 < P  # the case this test is about
    assert q.report.iterations == plain.report.iterations
    assert q.report.dist_evals == plain.report.dist_evals
    np.testing.assert_array_equal(q.palette, plain.palette)
    np.testing.assert_array_equal(q.report.sse_history, plain.report.sse_history)
    np.testing.assert_array_equal(q.index_map, plain.index_map)
    h = port.build_histogram(img)
    o = port.run_wsm(h.keys, h.counts, P, 256, mode=1, eps=1e-4, cap=100, seed=9)
    assert q.report.iterations == o.iterations and q.report.dist_evals == o.dist_evals
    np.testing.assert_array_equal(q.palette, o.centers)
