"""GPU: the sharded device path (cqb_shard_* + cqb_finalize_moments) run as W
virtual shards on one GPU equals the oracle / single-GPU run — the exactness
that makes the N-GPU run bit-identical (integer moments, fixed finalize)."""
import os

import numpy as np
import pytest

from paper_1011_0093_b200 import api
from paper_1011_0093_b200.configs import gmm_image, uniform_image
from paper_1011_0093_b200.distributed import DeviceShardBackend, run_wsm_sharded

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shards", [1, 2, 4, 7])
def test_device_shards_match_oracle(shards, port):
    img = gmm_image(128, 64, 24, 8)  # P = 8192
    h = port.build_histogram(img)
    ref = port.run_wsm(h.keys, h.counts, 8192, 16, mode=1, seed=1, trajectory=True)
    res = run_wsm_sharded(DeviceShardBackend(), img, 16, shards=shards)
    assert res.iterations == ref.iterations
    np.testing.assert_array_equal(res.centers, ref.centers)
    assert res.dist_evals == ref.dist_evals
    np.testing.assert_allclose(res.sse_history, ref.sse_history, rtol=1e-9)


def test_device_shards_k256_uniform(port):
    img = uniform_image(256, 256, 21)  # P = 65536, N' ~ 65K, K = 256
    single = api.quantize(img, 256, api.Termination.convergent(1e-4, 100), seed=1, index_map=False, mapped=False)
    res = run_wsm_sharded(DeviceShardBackend(), img, 256, shards=3)
    assert res.iterations == single.report.iterations
    np.testing.assert_array_equal(res.centers, single.palette)
    assert res.dist_evals == single.report.dist_evals


# --------------------------------------------------------------------------- in-kernel exchange
def _sharded_run(img, k, world, term=None, seed=1):
    """cqb_quantize_sharded with `world` emulated ranks (block groups of one
    cooperative launch; world = 0: the one-process X = 1 kernel, exchanging
    with itself). Returns (centers, report, sse_history, index map, mapped)."""
    import torch

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import PeerShardedQuantizer

    term = term or api.Termination.convergent(1e-4, 100)
    P = img.shape[0] * img.shape[1]
    ctx = _native.Context(0)
    q = PeerShardedQuantizer(ctx=ctx, emulate=world)
    d_img = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
    d_idx = torch.empty(P, dtype=torch.uint8, device="cuda")
    d_rgb = torch.empty(3 * P, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    lo, hi = q.enqueue(d_img.data_ptr(), P, k, term, seed, d_idx.data_ptr(), d_rgb.data_ptr())
    assert (lo, hi) == (0, P)
    centers, rep, hist = q.fetch()
    out = (centers, rep, hist, d_idx.cpu().numpy().reshape(img.shape[:2]), d_rgb.cpu().numpy().reshape(img.shape))
    ctx.close()
    return out


@pytest.mark.parametrize("world", [0, 1, 2, 3, 8])
@pytest.mark.parametrize("case", ["gmm", "uniform"])
def test_in_kernel_exchange_matches_single_gpu(world, case):
    """The sharded loop with the moment exchange inside the kernel gives the
    single-GPU quantize bit for bit: palette, iterations, SSE history,
    dist_evals, index map, mapped raster and MSE (exact integer moments)."""
    img = gmm_image(384, 256, 48, 5) if case == "gmm" else uniform_image(1024, 2048, 9)  # small / large paths
    k = 64 if case == "gmm" else 256
    single = api.quantize(img, k, api.Termination.convergent(1e-4, 100), seed=1)
    centers, rep, hist, idx, mapped = _sharded_run(img, k, world)
    np.testing.assert_array_equal(centers, single.palette)
    assert rep.iterations == single.report.iterations
    assert rep.dist_evals == single.report.dist_evals
    assert rep.n_unique == single.report.n_unique
    np.testing.assert_array_equal(hist, np.asarray(single.report.sse_history))
    np.testing.assert_array_equal(idx, single.index_map)
    np.testing.assert_array_equal(mapped, single.mapped)
    assert rep.mse == single.report.mse


def test_in_kernel_exchange_fixed_iterations_and_repeat():
    """Fixed termination, and two calls in a row on one context (the exchange
    counters carry over between launches)."""
    import torch

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import PeerShardedQuantizer

    img = gmm_image(256, 128, 24, 11)
    term = api.Termination.fixed(7)
    single = api.quantize(img, 32, term, seed=3)
    ctx = _native.Context(0)
    q = PeerShardedQuantizer(ctx=ctx, emulate=4)
    d_img = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
    torch.cuda.synchronize()
    for _ in range(3):
        q.enqueue(d_img.data_ptr(), img.shape[0] * img.shape[1], 32, term, 3)
        centers, rep, _ = q.fetch()
        np.testing.assert_array_equal(centers, single.palette)
        assert rep.iterations == 7 and rep.dist_evals == single.report.dist_evals
    ctx.close()


@pytest.mark.parametrize("seed,comp,k", [(0, 3, 32), (28, 12, 128), (43, 6, 64)])
@pytest.mark.parametrize("world", [2, 5])
def test_in_kernel_exchange_empty_cluster_reseed(seed, comp, k, world, port):
    """Runs whose trajectory empties clusters (found by tools/find_empty.py):
    the reseed candidates go through the exchange, and the result equals the
    single-GPU run and the oracle."""
    img = gmm_image(48, 40, comp, seed)
    single = api.quantize(img, k, api.Termination.convergent(1e-4, 100), seed=seed)
    assert single.report.empty_events > 0
    centers, rep, hist, idx, mapped = _sharded_run(img, k, world, seed=seed)
    np.testing.assert_array_equal(centers, single.palette)
    assert rep.empty_events == single.report.empty_events
    assert rep.iterations == single.report.iterations and rep.dist_evals == single.report.dist_evals
    np.testing.assert_array_equal(idx, single.index_map)
    h = port.build_histogram(img)
    ref = port.run_wsm(h.keys, h.counts, 48 * 40, k, mode=1, eps=1e-4, cap=100, seed=seed)
    assert rep.iterations == ref.iterations
    np.testing.assert_allclose(centers, ref.centers, rtol=1e-12, atol=0)


@pytest.mark.slow
def test_in_kernel_exchange_cfg4_full_size():
    """Config 4 (4096^2 uniform, 10.6M unique colors) with 8 emulated ranks:
    the same palette, iteration count, dist_evals, MSE and index map as the
    one-rank run."""
    from paper_1011_0093_b200.configs import CONFIGS

    img = CONFIGS["cfg4"].image()
    single = api.quantize(img, 256, api.Termination.convergent(1e-4, 100), seed=1)
    centers, rep, hist, idx, mapped = _sharded_run(img, 256, 8)
    np.testing.assert_array_equal(centers, single.palette)
    assert rep.iterations == single.report.iterations and rep.dist_evals == single.report.dist_evals
    assert rep.mse == single.report.mse
    np.testing.assert_array_equal(idx, single.index_map)


def test_in_kernel_exchange_dead_peer_fails_instead_of_hanging():
    """A rank that stops publishing (debug flag: emulated rank 1 goes silent
    at iteration 3) makes the others give up after the 5 s exchange timeout:
    the call fails with CQB_ERR_NCCL, the kernel exits, and the context still
    quantizes afterwards."""
    import time

    import torch

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import PeerShardedQuantizer

    img = gmm_image(128, 64, 16, 3)
    ctx = _native.Context(0)
    q = PeerShardedQuantizer(ctx=ctx, emulate=2)
    d_img = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
    torch.cuda.synchronize()
    ctx.check(ctx.lib.cqb_set_debug(ctx.h, 32768))
    ctx.check(ctx.lib.cqb_xch_set_timeout(ctx.h, 1.0))
    t0 = time.time()
    q.enqueue(d_img.data_ptr(), img.shape[0] * img.shape[1], 16, api.Termination.convergent(1e-4, 100), 1)
    with pytest.raises(_native.CqbError) as e:
        q.fetch()
    assert e.value.code == _native.CQB_ERR_NCCL
    assert time.time() - t0 < 30
    ctx.check(ctx.lib.cqb_set_debug(ctx.h, 0))
    # the failed exchange is reset: the same windows are refused until set up again
    with pytest.raises(_native.CqbInvalidArgument):
        q.enqueue(d_img.data_ptr(), img.shape[0] * img.shape[1], 16, api.Termination.convergent(1e-4, 100), 1)
    ctx.check(ctx.lib.cqb_xch_set_timeout(ctx.h, 5.0))
    single = api.quantize(img, 16, api.Termination.convergent(1e-4, 100), seed=1)
    q2 = PeerShardedQuantizer(ctx=ctx, emulate=2)  # fresh windows after a failed exchange
    q2.enqueue(d_img.data_ptr(), img.shape[0] * img.shape[1], 16, api.Termination.convergent(1e-4, 100), 1)
    centers, rep, _ = q2.fetch()
    np.testing.assert_array_equal(centers, single.palette)
    ctx.close()


@pytest.mark.parametrize("world", [3, 8])
def test_in_kernel_exchange_edge_cases(world, port):
    """Fewer unique colors than ranks (empty shards), k = 1, k = N', a
    single-color image, a ragged pixel count: the emulated ranks give the
    single-GPU result."""
    rng = np.random.default_rng(world)
    cases = []
    few = rng.integers(0, 256, (5, 3), dtype=np.uint8)
    cases.append((few[rng.integers(0, 5, 17 * 3)].reshape(17, 3, 3), 3))   # N' = 5 < 8 ranks, P = 51
    cases.append((few[rng.integers(0, 5, 40 * 8)].reshape(40, 8, 3), 1))   # k = 1
    cases.append((few[rng.integers(0, 5, 16 * 16)].reshape(16, 16, 3), 5))  # k = N'
    cases.append((np.full((9, 7, 3), 200, np.uint8), 1))                    # one color
    cases.append((gmm_image(61, 37, 9, 4), 24))                             # ragged P
    for img, k in cases:
        single = api.quantize(img, k, api.Termination.convergent(1e-4, 100), seed=1)
        centers, rep, hist, idx, mapped = _sharded_run(img, k, world)
        np.testing.assert_array_equal(centers, single.palette)
        assert rep.iterations == single.report.iterations and rep.dist_evals == single.report.dist_evals
        np.testing.assert_array_equal(idx, single.index_map)
        np.testing.assert_array_equal(mapped, single.mapped)
        assert rep.mse == single.report.mse


def _ipc_worker(rank, port, q):
    import os

    import torch.distributed as dist

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import PeerShardedQuantizer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        ctx = _native.Context(0)
        qz = PeerShardedQuantizer(ctx=ctx)  # cqb_xch_window + handle all-gather + cqb_xch_open of the peer
        dist.barrier()
        ctx.close()  # closes the peer mapping, frees the window
        dist.barrier()
        q.put((rank, qz.world, qz.rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, 0, 0, repr(e)))
    finally:
        dist.destroy_process_group()


def test_ipc_windows_open_across_processes():
    """The real multi-process setup path (no kernels): two processes on this
    GPU create their exchange windows, all-gather the IPC handles and map
    each other's window. (Running the X = 1 loop itself needs one GPU per
    rank: kernels that wait on each other must not share a GPU.)"""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    outs = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [o[3] for o in outs] == ["ok", "ok"], outs
    assert [(o[1], o[2]) for o in outs] == [(2, 0), (2, 1)]


def test_exchange_argument_errors():
    """cqb_xch_* / cqb_quantize_sharded argument checks (invalid argument, not a crash)."""
    import ctypes as C

    from paper_1011_0093_b200 import _native

    ctx = _native.Context(0)
    lib = ctx.lib
    t = api.Termination.convergent(1e-4, 100).native()
    assert lib.cqb_quantize_sharded(ctx.h, None, 16, 4, C.byref(t), 1, None, None, None) == _native.CQB_ERR_INVALID_ARGUMENT
    assert lib.cqb_xch_emulate(ctx.h, 0) == _native.CQB_ERR_INVALID_ARGUMENT
    assert lib.cqb_xch_emulate(ctx.h, 9) == _native.CQB_ERR_INVALID_ARGUMENT
    h = (C.c_ubyte * _native.IPC_HANDLE_BYTES)()
    assert lib.cqb_xch_window(ctx.h, 2, 2, h) == _native.CQB_ERR_INVALID_ARGUMENT
    assert lib.cqb_xch_window(ctx.h, 2, 0, h) == _native.CQB_OK
    # the peer window is not mapped yet: refused, no launch
    import torch

    d = torch.zeros(48, dtype=torch.uint8, device="cuda")
    rc = lib.cqb_quantize_sharded(ctx.h, d.data_ptr(), 16, 4, C.byref(t), 1, None, None, None)
    assert rc == _native.CQB_ERR_INVALID_ARGUMENT and b"not mapped" in lib.cqb_last_error(ctx.h)
    ctx.close()


# --------------------------------------------------------------------------- pixel-row sharded histogram
def _morton_np(keys):
    def spread(v):
        v = v.astype(np.uint64) & 0xFF
        v = (v | (v << 8)) & 0x0000F00F
        v = (v | (v << 4)) & 0x000C30C3
        v = (v | (v << 2)) & 0x00249249
        return v
    k = keys.astype(np.uint64)
    return (spread(k >> 16) << 2) | (spread(k >> 8) << 1) | spread(k)


def _full_triplets(img):
    px = img.reshape(-1, 3).astype(np.uint32)
    keys = (px[:, 0] << 16) | (px[:, 1] << 8) | px[:, 2]
    u, first, counts = np.unique(keys, return_index=True, return_counts=True)
    o = np.argsort(_morton_np(u), kind="stable")
    return np.stack([u[o], counts[o], first[o]], 1).astype(np.uint32)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("case", ["gmm", "uniform", "ragged"])
def test_row_sharded_histogram_matches_full(world, case):
    """cqb_hist_rows (K1 over one rank's pixel rows with global pixel indices,
    occupancy compaction, owner split) + cqb_hist_merge (count sum, first-pixel
    min, owner-range compaction), W ranks emulated in one process: the owners'
    lists concatenated are the whole image's Morton-ordered histogram, entry
    for entry."""
    import torch

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import DeviceHistBackend, sharded_histogram_emulated

    img = {"gmm": lambda: gmm_image(384, 256, 48, 5), "uniform": lambda: uniform_image(2048, 2048, 9),
           "ragged": lambda: gmm_image(1531, 1373, 64, 77)}[case]()
    P = img.shape[0] * img.shape[1]
    ctx = _native.Context(0)
    try:
        d = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
        got = sharded_histogram_emulated(DeviceHistBackend(ctx), d, P, world).cpu().numpy().view(np.uint32)
    finally:
        ctx.close()
    np.testing.assert_array_equal(got, _full_triplets(img))


@pytest.mark.parametrize("world", [0, 2, 8])
def test_quantize_from_row_sharded_histogram(world):
    """cqb_quantize_sharded_samples after the row-sharded histogram (world 0:
    no exchange, the single-GPU pipeline from the given histogram; W: the
    emulated in-kernel exchange) gives the single-GPU quantize bit for bit:
    palette, iterations, dist_evals, MSE, index map and mapped raster."""
    import torch

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import (DeviceHistBackend, PeerShardedQuantizer,
                                                  sharded_histogram_emulated)

    img = uniform_image(1024, 2048, 12)
    k = 256
    term = api.Termination.convergent(1e-4, 100)
    single = api.quantize(img, k, term, seed=1)
    P = img.shape[0] * img.shape[1]
    ctx = _native.Context(0)
    try:
        d_img = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
        d_idx = torch.empty(P, dtype=torch.uint8, device="cuda")
        d_rgb = torch.empty(3 * P, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        if world:
            q = PeerShardedQuantizer(ctx=ctx, emulate=world)
            lo, hi = q.enqueue_rows(d_img, P, k, term, 1, d_idx.data_ptr(), d_rgb.data_ptr())
            centers, rep, hist = q.fetch()
        else:
            import ctypes as C

            samples = sharded_histogram_emulated(DeviceHistBackend(ctx), d_img, P, 4)
            rng = np.zeros(2, np.uint64)
            t = term.native()
            ctx.check(ctx.lib.cqb_quantize_sharded_samples(ctx.h, d_img.data_ptr(), P, samples.data_ptr(),
                                                           samples.shape[0], k, C.byref(t), 1, d_idx.data_ptr(),
                                                           d_rgb.data_ptr(), rng.ctypes.data_as(C.POINTER(C.c_uint64))))
            centers = np.zeros(3 * k)
            hist = np.zeros(term.iteration_budget)
            rep = _native.Report()
            ctx.check(ctx.lib.cqb_fetch_results(ctx.h, centers.ctypes.data_as(C.POINTER(C.c_double)),
                                                hist.ctypes.data_as(C.POINTER(C.c_double)), term.iteration_budget,
                                                C.byref(rep)))
            centers = centers.reshape(k, 3)
            lo, hi = int(rng[0]), int(rng[1])
        assert (lo, hi) == (0, P)
        np.testing.assert_array_equal(centers, single.palette)
        assert rep.iterations == single.report.iterations and rep.dist_evals == single.report.dist_evals
        assert rep.mse == single.report.mse and rep.n_unique == single.report.n_unique
        np.testing.assert_array_equal(d_idx.cpu().numpy().reshape(img.shape[:2]), single.index_map)
        np.testing.assert_array_equal(d_rgb.cpu().numpy().reshape(img.shape), single.mapped)
    finally:
        ctx.close()


def test_hist_rows_argument_errors():
    import torch

    from paper_1011_0093_b200 import _native

    ctx = _native.Context(0)
    try:
        d = torch.zeros(3 * 64, dtype=torch.uint8, device="cuda")
        out = torch.empty((64, 3), dtype=torch.int32, device="cuda")
        n = np.zeros(1, np.uint64)
        cnt = np.zeros(16, np.uint64)
        u64 = lambda a: a.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_uint64))  # noqa: E731
        for world, rank, cap in ((0, 0, 64), (2, 2, 64), (9, 0, 64), (1, 0, 63)):
            rc = ctx.lib.cqb_hist_rows(ctx.h, d.data_ptr(), 64, world, rank, out.data_ptr(), cap, u64(n), u64(cnt))
            assert rc == _native.CQB_ERR_INVALID_ARGUMENT, (world, rank, cap)
        assert ctx.lib.cqb_hist_rows(ctx.h, d.data_ptr(), 64, 1, 0, out.data_ptr(), 64, u64(n), u64(cnt)) == 0
        assert int(n[0]) == 1 and int(cnt[0]) == 1
    finally:
        ctx.close()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("case", ["gmm", "uniform", "ragged"])
def test_morton_range_histogram_matches_full(world, case):
    """cqb_hist_range (every pixel counted into one rank's Morton range of
    whole compaction tiles, L2-sized passes, range-only compaction), W ranks
    emulated in one process: the owner lists concatenated are the whole
    image's Morton-ordered histogram, entry for entry."""
    import torch

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import DeviceHistBackend, sharded_histogram_morton_emulated

    img = {"gmm": lambda: gmm_image(384, 256, 48, 5), "uniform": lambda: uniform_image(2048, 2048, 9),
           "ragged": lambda: gmm_image(1531, 1373, 64, 77)}[case]()
    P = img.shape[0] * img.shape[1]
    ctx = _native.Context(0)
    try:
        d = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
        got = sharded_histogram_morton_emulated(DeviceHistBackend(ctx), d, P, world).cpu().numpy().view(np.uint32)
    finally:
        ctx.close()
    np.testing.assert_array_equal(got, _full_triplets(img))


@pytest.mark.parametrize("world", [2, 8])
def test_quantize_from_morton_range_histogram(world):
    """The Morton-range histogram feeding the emulated in-kernel exchange:
    bit-identical to the single-GPU quantize."""
    import torch

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import PeerShardedQuantizer

    img = uniform_image(1024, 2048, 13)
    k = 256
    term = api.Termination.convergent(1e-4, 100)
    single = api.quantize(img, k, term, seed=1)
    P = img.shape[0] * img.shape[1]
    ctx = _native.Context(0)
    try:
        d_img = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
        d_idx = torch.empty(P, dtype=torch.uint8, device="cuda")
        d_rgb = torch.empty(3 * P, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        q = PeerShardedQuantizer(ctx=ctx, emulate=world)
        lo, hi = q.enqueue_rows(d_img, P, k, term, 1, d_idx.data_ptr(), d_rgb.data_ptr(), split="morton")
        centers, rep, hist = q.fetch()
        assert (lo, hi) == (0, P)
        np.testing.assert_array_equal(centers, single.palette)
        assert rep.iterations == single.report.iterations and rep.dist_evals == single.report.dist_evals
        assert rep.mse == single.report.mse
        np.testing.assert_array_equal(d_idx.cpu().numpy().reshape(img.shape[:2]), single.index_map)
        np.testing.assert_array_equal(d_rgb.cpu().numpy().reshape(img.shape), single.mapped)
    finally:
        ctx.close()


@pytest.mark.parametrize("split", ["rows", "morton"])
def test_sharded_histogram_edge_cases(split):
    """Both histogram splits on the edges: one pixel, fewer 16-pixel chunks than
    ranks (empty row shards), one color everywhere, and every one of the 2^24
    colors once (every Morton range full)."""
    import torch

    from paper_1011_0093_b200 import _native
    from paper_1011_0093_b200.distributed import (DeviceHistBackend, sharded_histogram_emulated,
                                                  sharded_histogram_morton_emulated)

    fn = sharded_histogram_emulated if split == "rows" else sharded_histogram_morton_emulated
    rng = np.random.default_rng(3)
    allc = np.arange(1 << 24, dtype=np.uint32)
    rng.shuffle(allc)
    cases = [
        rng.integers(0, 256, (1, 1, 3), dtype=np.uint8),
        rng.integers(0, 256, (1, 17, 3), dtype=np.uint8),
        np.full((64, 48, 3), 77, np.uint8),
        np.stack([(allc >> 16) & 255, (allc >> 8) & 255, allc & 255], 1).astype(np.uint8).reshape(4096, 4096, 3),
    ]
    ctx = _native.Context(0)
    try:
        for img in cases:
            P = img.shape[0] * img.shape[1]
            d = torch.zeros(3 * P + 16, dtype=torch.uint8, device="cuda")  # (16-B aligned)
            d[: 3 * P] = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
            for world in (1, 3, 8):
                got = fn(DeviceHistBackend(ctx), d, P, world).cpu().numpy().view(np.uint32)
                np.testing.assert_array_equal(got, _full_triplets(img))
    finally:
        ctx.close()


def test_sharded_histogram_over_nccl_world1(tmp_path):
    """The NCCL leg of the sharded histograms (TensorExchange: all-to-all and
    all-gather of CUDA int32 triplets) in a one-rank NCCL process group (a
    subprocess): both splits return the full histogram. The multi-rank logic
    of the same code runs over gloo in tests/test_distributed.py."""
    import subprocess
    import sys
    import textwrap

    code = textwrap.dedent("""
        import os, sys, numpy as np, torch, torch.distributed as dist
        sys.path.insert(0, os.getcwd())
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29000 + os.getpid() % 1000))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        from paper_1011_0093_b200 import _native
        from paper_1011_0093_b200.configs import gmm_image
        from paper_1011_0093_b200.distributed import (DeviceHistBackend, TensorExchange, sharded_histogram,
                                                      sharded_histogram_morton)
        img = gmm_image(1531, 1373, 64, 77)
        P = img.shape[0] * img.shape[1]
        d = torch.from_numpy(np.ascontiguousarray(img).reshape(-1)).cuda()
        ctx = _native.Context(0)
        for name, fn in (("rows", sharded_histogram), ("morton", sharded_histogram_morton)):
            got = fn(DeviceHistBackend(ctx), d, P, TensorExchange()).cpu().numpy().view(np.uint32)
            np.save(os.path.join(sys.argv[1], name + ".npy"), got)
        ctx.close()
        dist.destroy_process_group()
        print("ok")
    """)
    r = subprocess.run([sys.executable, "-c", code, str(tmp_path)], capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
    ref = _full_triplets(gmm_image(1531, 1373, 64, 77))
    for name in ("rows", "morton"):
        np.testing.assert_array_equal(np.load(tmp_path / (name + ".npy")), ref)
