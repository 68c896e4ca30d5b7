"""The point-set API (kmeans.hpp's span<const Vec3> overloads) on the device
against the UNMODIFIED reference (oracle/_ref): init_centers, assign_sort_means
/ assign_naive, update_centers (with empty-cluster reseeds), weighted_sse and
run_wsm_points, real-valued points and weights, k up to 1024.

Bar: chosen centers, memberships, dist_evals and updated centers bit-exact
(update_centers reproduces the reference's sequential per-cluster sums);
weighted SSE within 1e-12 relative (fixed-order tree sum vs the reference's
sequential sum)."""
import numpy as np
import pytest

from paper_1011_0093_b200 import api

pytestmark = pytest.mark.gpu
SSE_RTOL = 1e-12


def _instance(n, seed, clusters=12, dup=0):
    rng = np.random.default_rng(seed)
    means = rng.uniform(0, 255, (clusters, 3))
    X = means[rng.integers(0, clusters, n)] + rng.normal(0, 9.0, (n, 3))
    if dup:  # repeated points (the reseed's taken-by-value rule)
        X[-dup:] = X[:dup]
    W = rng.uniform(0.1, 3.0, n)
    return X, W / W.sum()


@pytest.mark.parametrize("n,k,seed", [(50, 1, 3), (500, 7, 1), (3000, 64, 9), (4000, 300, 2), (2048, 1024, 5)])
def test_init_centers_matches_reference(n, k, seed, ref):
    X, _ = _instance(n, seed)
    np.testing.assert_array_equal(api.init_centers(X, k, seed), ref.init_centers_points(X, k, seed))


def test_init_centers_errors():
    X, _ = _instance(10, 1)
    with pytest.raises(ValueError):
        api.init_centers(X, 11, 1)  # kmeans.hpp:55-56
    with pytest.raises(ValueError):
        api.init_centers(X, 0, 1)


@pytest.mark.parametrize("n,k,seed", [(1000, 5, 1), (5000, 40, 2), (3000, 400, 3)])
def test_assign_matches_reference(n, k, seed, ref):
    X, W = _instance(n, seed)
    rng = np.random.default_rng(seed + 100)
    C = X[rng.choice(n, k, replace=False)] + rng.normal(0, 0.5, (k, 3))
    m0 = rng.integers(0, k, n).astype(np.int32)
    m, sse, ev = api.assign_points(X, W, C, m0)
    rm, rsse, rev, audited = ref.points_assign(X, W, C, m0)
    np.testing.assert_array_equal(m, rm)
    assert ev == rev
    assert sse == pytest.approx(rsse, rel=SSE_RTOL)
    assert audited > 0  # the reference's pruning fired on this instance
    nm, nsse, nev = api.assign_points(X, W, C, naive=True)
    rnm, rnsse, rnev, _ = ref.points_assign(X, W, C, np.zeros(n, np.int32), naive=True)
    np.testing.assert_array_equal(nm, rnm)
    np.testing.assert_array_equal(nm, m)  # sort-means = exhaustive (ties to the lowest index)
    assert nev == rnev == n * k
    assert nsse == pytest.approx(rnsse, rel=SSE_RTOL)


@pytest.mark.parametrize("n,k,seed", [(2000, 16, 4), (6000, 200, 6)])
def test_update_centers_bit_exact_with_empty_clusters(n, k, seed, ref):
    X, W = _instance(n, seed, dup=40)
    rng = np.random.default_rng(seed)
    m = rng.integers(0, k, n).astype(np.int32)
    m[m % 5 == 3] = 0  # clusters 3, 8, 13, ... left empty
    prev = rng.uniform(0, 255, (k, 3))
    got = api.update_centers(X, W, m, prev)
    np.testing.assert_array_equal(got, ref.points_update(X, W, m, prev))
    assert api.weighted_sse(X, W, got, m) == pytest.approx(ref.points_sse(X, W, got, m), rel=SSE_RTOL)


@pytest.mark.parametrize("n,k,mode,seed", [(3000, 8, 1, 1), (5000, 32, 1, 2), (4000, 16, 0, 3), (3000, 320, 0, 4)])
def test_run_wsm_points_matches_reference(n, k, mode, seed, ref):
    X, W = _instance(n, seed)
    term = api.Termination.convergent(1e-4, 100) if mode else api.Termination.fixed(6)
    g = api.run_wsm_points(X, W, k, term, seed=seed)
    o = ref.run_wsm_points(X, W, k, mode=mode, max_iters=6, eps=1e-4, cap=100, seed=seed)
    assert g.report.iterations == o.iterations
    assert g.report.dist_evals == o.dist_evals
    np.testing.assert_array_equal(g.palette, o.centers)
    np.testing.assert_allclose(g.report.sse_history, o.sse_history, rtol=SSE_RTOL)


def test_run_wsm_on_a_real_valued_histogram_takes_the_point_path(ref):
    """run_wsm with weights that are not count/total (kmeans.hpp:394-404
    accepts any ColorHistogram): the shim routes it to the point-set path;
    here through the Python API the same way."""
    X, W = _instance(2500, 11)
    Xr = np.round(X).clip(0, 255)
    g = api.run_wsm_points(Xr, W, 24, api.Termination.convergent(1e-4, 100), seed=3)
    o = ref.run_wsm_points(Xr, W, 24, mode=1, eps=1e-4, cap=100, seed=3)
    assert g.report.iterations == o.iterations and g.report.dist_evals == o.dist_evals
    np.testing.assert_array_equal(g.palette, o.centers)
