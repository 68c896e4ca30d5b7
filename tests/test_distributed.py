"""CPU-only: the multi-GPU host logic (paper_1011_0093_b200/distributed.py).

World-size-2 `gloo` process groups on 127.0.0.1 run the sharded driver with a
CPU stand-in backend (numpy + the oracle's primitive functions, test
infrastructure only). The sharded trajectory must equal the single-process
oracle run: iterations, centers (bit-exact for power-of-two P), dist_evals,
SSE history — including the empty-cluster reseed exchanged via allgather.
"""
import ctypes as C
import os
import socket
import time

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1011_0093_b200.configs import gmm_image
from paper_1011_0093_b200.distributed import LocalCollective, pair_evals, run_wsm_sharded, shard_range

_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)


def _morton(keys):
    def spread(v):
        v = v.astype(np.uint64) & 0xFF
        v = (v | (v << 8)) & 0x0000F00F
        v = (v | (v << 4)) & 0x000C30C3
        v = (v | (v << 2)) & 0x00249249
        return v
    k = keys.astype(np.uint64)
    return (spread(k >> 16) << 2) | (spread(k >> 8) << 1) | spread(k)


class FakeShardBackend:
    """CPU stand-in for DeviceShardBackend (test infrastructure)."""

    def __init__(self, init_override=None):
        from oracle.oracle import Oracle

        self.o = Oracle("port")
        self.init_override = init_override

    def prepare(self, img, k, seed):
        h = self.o.build_histogram(img)
        order = np.argsort(_morton(h.keys), kind="stable")
        self.keys = h.keys[order]
        self.counts = h.counts[order].astype(np.uint64)
        self.rank = order.astype(np.uint32)  # first-occurrence rank of each Morton-ordered sample
        self.X = np.stack([(self.keys >> 16) & 255, (self.keys >> 8) & 255, self.keys & 255], 1).astype(np.float64)
        self.labels = np.zeros(len(self.keys), np.int32)
        self.k = k
        self.total = img.shape[0] * img.shape[1]
        C0 = self.o.init_centers(h.keys, k, seed) if self.init_override is None else self.init_override.copy()
        return len(self.keys), self.total, C0

    def step(self, lo, hi, centers, first):
        k = self.k
        Cc = np.ascontiguousarray(centers, np.float64)
        D = np.zeros(k * k)
        order = np.zeros(k * k, np.int32)
        f = self.o._f
        f("center_tables")(Cc.ctypes.data_as(_f64p), k, D.ctypes.data_as(_f64p), order.ctypes.data_as(_i32p))
        X = np.ascontiguousarray(self.X[lo:hi])
        W = np.ones(hi - lo)
        lab = np.ascontiguousarray(self.labels[lo:hi])
        sse = np.zeros(1)
        ev = np.zeros(1, np.uint64)
        f("assign_sort_means")(X.ctypes.data_as(_f64p), W.ctypes.data_as(_f64p), hi - lo, Cc.ctypes.data_as(_f64p), k,
                               D.ctypes.data_as(_f64p), order.ctypes.data_as(_i32p), lab.ctypes.data_as(_i32p),
                               sse.ctypes.data_as(_f64p), ev.ctypes.data_as(_u64p))
        self.labels[lo:hi] = lab
        c = self.counts[lo:hi]
        xi = self.X[lo:hi].astype(np.uint64)
        mom = np.zeros((5, k), np.uint64)
        for fld, v in enumerate([c * xi[:, 0], c * xi[:, 1], c * xi[:, 2], c,
                                 c * (xi[:, 0] ** 2 + xi[:, 1] ** 2 + xi[:, 2] ** 2)]):
            np.add.at(mom[fld], lab, v)
        return mom, int(ev[0])

    def finalize(self, mom, centers, total):
        N = mom[3].astype(np.float64)
        new = centers.copy()
        nz = mom[3] > 0
        for ch in range(3):
            new[nz, ch] = mom[ch][nz].astype(np.float64) / N[nz]
        Cc = centers
        sse = 0.0
        for t in np.nonzero(nz)[0]:
            S = mom[:3, t].astype(np.float64)
            sse += float(mom[4, t]) - 2 * float(np.dot(Cc[t], S)) + float(np.dot(Cc[t], Cc[t])) * N[t]
        return new, max(sse / total, 0.0), [int(t) for t in np.nonzero(~nz)[0]]

    def reseed_candidate(self, lo, hi, centers, taken):
        X = self.X[lo:hi]
        lab = self.labels[lo:hi]
        d = ((X - centers[lab]) ** 2).sum(1)
        best = (-1.0, 0xFFFFFFFF, 0)
        for j in range(hi - lo):
            r = int(self.rank[lo + j])
            if r in taken:
                continue
            if d[j] > best[0] or (d[j] == best[0] and r < best[1]):
                best = (float(d[j]), r, int(self.keys[lo + j]))
        return best


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, img, k, mode, iters, init_override, out_q):
    import torch.distributed as dist

    from paper_1011_0093_b200.distributed import TorchCollective

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_wsm_sharded(FakeShardBackend(init_override), img, k, mode=mode, max_iters=iters, coll=TorchCollective())
        out_q.put((rank, res.centers, res.iterations, res.dist_evals, res.sse_history))
    finally:
        dist.destroy_process_group()


def _run_gloo(world, img, k, mode=1, iters=10, init_override=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, img, k, mode, iters, init_override, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(outs, key=lambda o: o[0])


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 1000, 366922):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_pair_evals_rule():
    C0 = np.arange(12.0).reshape(4, 3)
    assert pair_evals(None, C0) == 6
    C1 = C0.copy()
    assert pair_evals(C0, C1) == 0
    C1[2, 0] += 1
    assert pair_evals(C0, C1) == 6 - 3  # three unmoved centers keep 3 pairs


@pytest.mark.parametrize("shards", [1, 2, 3, 5])
def test_local_shards_match_oracle(shards, port):
    img = gmm_image(64, 32, 10, 11)  # P = 2048
    h = port.build_histogram(img)
    ref = port.run_wsm(h.keys, h.counts, 2048, 8, mode=1, seed=1, trajectory=True)
    res = run_wsm_sharded(FakeShardBackend(), img, 8, shards=shards)
    assert res.iterations == ref.iterations
    np.testing.assert_array_equal(res.centers, ref.centers)
    assert res.dist_evals == ref.dist_evals
    np.testing.assert_allclose(res.sse_history, ref.sse_history, rtol=1e-9)


def test_gloo_world2_matches_oracle(port):
    img = gmm_image(64, 64, 12, 5)  # P = 4096
    h = port.build_histogram(img)
    ref = port.run_wsm(h.keys, h.counts, 4096, 12, mode=1, seed=1)
    outs = _run_gloo(2, img, 12)
    for rank, centers, iters, evals, hist in outs:
        assert iters == ref.iterations
        np.testing.assert_array_equal(centers, ref.centers)
        assert evals == ref.dist_evals
        np.testing.assert_allclose(hist, ref.sse_history, rtol=1e-9)


def test_gloo_world2_empty_cluster_reseed(port):
    """A center that owns nothing is re-seeded at the global farthest point
    (kmeans.hpp:272-294), the candidates exchanged by allgather."""
    img = gmm_image(32, 32, 6, 9)  # P = 1024
    h = port.build_histogram(img)
    init = port.init_centers(h.keys, 6, 3)
    init[4] = (999.0, 999.0, 999.0)
    # reference trajectory with the same init from the oracle primitives
    X = h.colors
    W = h.counts.astype(np.float64) / 1024.0
    lab = np.zeros(len(X), np.int32)
    Cc = init.copy()
    traj = []
    for it in range(4):
        D = np.zeros(36)
        order = np.zeros(36, np.int32)
        port._f("center_tables")(Cc.ctypes.data_as(_f64p), 6, D.ctypes.data_as(_f64p), order.ctypes.data_as(_i32p))
        sse = np.zeros(1)
        ev = np.zeros(1, np.uint64)
        port._f("assign_sort_means")(X.ctypes.data_as(_f64p), W.ctypes.data_as(_f64p), len(X),
                                     Cc.ctypes.data_as(_f64p), 6, D.ctypes.data_as(_f64p),
                                     order.ctypes.data_as(_i32p), lab.ctypes.data_as(_i32p), sse.ctypes.data_as(_f64p),
                                     ev.ctypes.data_as(_u64p))
        nxt = np.zeros(18)
        port._f("update_centers")(X.ctypes.data_as(_f64p), W.ctypes.data_as(_f64p), len(X), lab.ctypes.data_as(_i32p),
                                  Cc.ctypes.data_as(_f64p), 6, nxt.ctypes.data_as(_f64p))
        Cc = nxt.reshape(6, 3)
        traj.append(Cc.copy())
    outs = _run_gloo(2, img, 6, mode=0, iters=4, init_override=init)
    for rank, centers, iters, evals, hist in outs:
        assert iters == 4
        np.testing.assert_array_equal(centers, traj[-1])
    # the far center was re-seeded onto a sample color in iteration 1
    assert tuple(traj[0][4]) != (999.0, 999.0, 999.0)


# --------------------------------------------------------------------------- in-kernel exchange (host side)
def _handle_worker(rank, world, port, out_q):
    import torch.distributed as dist

    from paper_1011_0093_b200.distributed import exchange_handles

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes([rank]) * 64  # stands in for this rank's cudaIpcMemHandle_t
        out_q.put((rank, exchange_handles(mine)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_ipc_handles_in_rank_order():
    """PeerShardedQuantizer's setup: every rank receives all windows' IPC
    handles in rank order (cqb_xch_open indexes them by rank)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handle_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, hs in outs:
        assert hs == [bytes([0]) * 64, bytes([1]) * 64]


class _FakeXchLib:
    """Records PeerShardedQuantizer's C-ABI calls (test infrastructure): the
    window call writes a rank-tagged handle, the open call keeps what it was
    given, the sharded quantize returns the rank's pixel range."""

    def __init__(self):
        self.calls = []

    def cqb_xch_window(self, h, world, rank, buf):
        for i in range(len(buf)):
            buf[i] = 0x40 + rank
        self.calls.append(("window", world, rank))
        return 0

    def cqb_xch_open(self, h, buf):
        self.calls.append(("open", bytes(buf.raw)))
        return 0

    def cqb_quantize_sharded(self, h, d_rgb, n, k, term, seed, d_index, d_rgb_out, rng):
        from paper_1011_0093_b200.distributed import pixel_range

        world, rank = self.calls[0][1], self.calls[0][2]
        lo, hi = pixel_range(n, world, rank)
        rng[0], rng[1] = lo, hi
        t = term._obj
        self.calls.append(("quantize", d_rgb, n, k, (t.mode, t.max_iters, t.epsilon, t.hard_cap), seed, d_index, d_rgb_out))
        return 0

    def cqb_fetch_results(self, h, centers, hist, cap, rep):
        k = self._k
        for i in range(3 * k):
            centers[i] = float(i)
        for i in range(cap):
            hist[i] = 1.0 / (i + 1)
        rep._obj.iterations = 3
        rep._obj.dist_evals = 1000
        self.calls.append(("fetch", cap))
        return 0


class _FakeCtx:
    def __init__(self):
        self.h = 1234
        self.lib = _FakeXchLib()

    def check(self, rc):
        assert rc == 0


def _peer_worker(rank, world, port, out_q):
    import torch.distributed as dist

    from paper_1011_0093_b200 import api
    from paper_1011_0093_b200.distributed import PeerShardedQuantizer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = _FakeCtx()
        q = PeerShardedQuantizer(ctx=ctx)
        term = api.Termination.convergent(1e-4, 100)
        rng = q.enqueue(0xD000 + rank, 1000003, 256, term, seed=7, d_index=0xE000, d_rgb_out=0xF000)
        ctx.lib._k = 256
        centers, rep, hist = q.fetch()
        out_q.put((rank, q.world, q.rank, rng, ctx.lib.calls, centers.shape, rep.iterations, list(hist)))
    except Exception as e:  # surface the failure instead of a queue timeout
        out_q.put((rank, "error", repr(e), None, None, None, None, None))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_peer_quantizer_setup_path():
    """The production setup path of the in-kernel sharded loop on CPU:
    PeerShardedQuantizer over a world-2 gloo group opens its window with the
    group's world/rank, all-gathers the IPC handles and passes them to
    cqb_xch_open in rank order, forwards the launch arguments unchanged, and
    the ranks' pixel ranges tile the raster (16-pixel aligned starts)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in procs], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 1000003
    handles = bytes([0x40]) * 64 + bytes([0x41]) * 64
    ranges = []
    for r, (rank, world, qrank, rng, calls, cshape, iters, hist) in enumerate(outs):
        assert world != "error", qrank
        assert (rank, world, qrank) == (r, 2, r)
        assert calls[0] == ("window", 2, r)
        assert calls[1] == ("open", handles)  # every rank: all handles, rank order
        name, d_rgb, n_px, k, term, seed, d_index, d_out = calls[2]
        assert (name, d_rgb, n_px, k, seed, d_index, d_out) == ("quantize", 0xD000 + r, n, 256, 7, 0xE000, 0xF000)
        assert term[0] == 1 and term[3] == 100 and abs(term[2] - 1e-4) < 1e-12
        assert calls[3] == ("fetch", 100)
        assert cshape == (256, 3) and iters == 3 and len(hist) == 3
        ranges.append(rng)
    assert ranges[0][0] == 0 and ranges[0][1] == ranges[1][0] and ranges[1][1] == n
    assert all(lo % 16 == 0 for lo, _ in ranges)


def test_pixel_ranges_tile_the_raster():
    from paper_1011_0093_b200.distributed import pixel_range

    for n in (1, 15, 16, 17, 1000003, 4096 * 4096):
        for w in (1, 2, 3, 8):
            rs = [pixel_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(lo % 16 == 0 and lo <= hi for lo, hi in rs)


def test_exchange_protocol_two_slots_suffice():
    """Model of the in-kernel exchange (wsm.cuh, XB_* windows): each rank
    writes exchange s into slot s&1 of every window, publishes flag = s, waits
    for all flags >= s, then reads and sums. With ranks running at arbitrary
    relative speeds no slot is overwritten before its reader is done, so every
    rank sums exactly the values of exchange s."""
    import random
    import threading

    W, N = 4, 300
    flags = [[0] * W for _ in range(W)]
    pay = [[[None] * W for _ in range(2)] for _ in range(W)]
    errors = []

    def rank(r):
        rnd = random.Random(r)
        for s in range(1, N + 1):
            for dst in range(W):  # payload, then flag (release order)
                pay[dst][s & 1][r] = (s, r)
                flags[dst][r] = s
                if rnd.random() < 0.3:
                    time.sleep(0)
            while min(flags[r]) < s:
                time.sleep(0)
            got = [pay[r][s & 1][src] for src in range(W)]
            if got != [(s, src) for src in range(W)]:
                errors.append((r, s, got))
            if rnd.random() < 0.2:
                time.sleep(0.0005)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:3]


# --------------------------------------------------------------------------- sharded histogram
class FakeHistBackend:
    """CPU stand-in for DeviceHistBackend (cqb_hist_rows / cqb_hist_merge
    semantics, test infrastructure): CPU int32 tensors of {key, count, first}."""

    @staticmethod
    def _emit(keys, counts, first):
        import torch

        o = np.argsort(_morton(keys), kind="stable")
        t = np.stack([keys[o], counts[o], first[o]], 1).astype(np.int64)
        return torch.from_numpy(t.astype(np.uint32).view(np.int32).reshape(-1, 3).copy())

    def rows(self, img, n_pixels, world, rank):
        from paper_1011_0093_b200.distributed import pixel_range

        lo, hi = pixel_range(n_pixels, world, rank)
        px = img.numpy().reshape(-1, 3)[lo:hi].astype(np.uint32)
        keys = (px[:, 0] << 16) | (px[:, 1] << 8) | px[:, 2]
        u, first, counts = np.unique(keys, return_index=True, return_counts=True)
        t = self._emit(u, counts, first + lo)
        m = _morton(t.numpy().view(np.uint32)[:, 0])
        bounds = [int(np.searchsorted(m, ((o << 24) // world))) for o in range(world)] + [len(m)]
        return t, [bounds[o + 1] - bounds[o] for o in range(world)]

    def range(self, img, n_pixels, world, rank):
        t0, t1 = 2048 * rank // world, 2048 * (rank + 1) // world
        px = img.numpy().reshape(-1, 3).astype(np.uint32)
        keys = (px[:, 0] << 16) | (px[:, 1] << 8) | px[:, 2]
        u, first, counts = np.unique(keys, return_index=True, return_counts=True)
        m = _morton(u)
        sel = (m >= t0 * 8192) & (m < t1 * 8192)
        return self._emit(u[sel], counts[sel], first[sel])

    def merge(self, recv, world):
        a = recv.numpy().view(np.uint32).astype(np.int64)
        if len(a) == 0:
            return self._emit(np.zeros(0, np.uint32), np.zeros(0, np.int64), np.zeros(0, np.int64))
        u, inv = np.unique(a[:, 0], return_inverse=True)
        counts = np.bincount(inv, weights=a[:, 1], minlength=len(u)).astype(np.int64)
        first = np.full(len(u), np.iinfo(np.int64).max)
        np.minimum.at(first, inv, a[:, 2])
        return self._emit(u.astype(np.uint32), counts, first)


def _full_histogram(img):
    px = img.reshape(-1, 3).astype(np.uint32)
    keys = (px[:, 0] << 16) | (px[:, 1] << 8) | px[:, 2]
    u, first, counts = np.unique(keys, return_index=True, return_counts=True)
    return FakeHistBackend._emit(u, counts, first).numpy()


def _hist_worker(rank, world, port, img, out_q, split="rows"):
    import torch
    import torch.distributed as dist

    from paper_1011_0093_b200.distributed import TensorExchange, sharded_histogram, sharded_histogram_morton

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = torch.from_numpy(img.reshape(-1).copy())
        fn = sharded_histogram if split == "rows" else sharded_histogram_morton
        out = fn(FakeHistBackend(), t, img.shape[0] * img.shape[1], TensorExchange())
        out_q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,split", [(2, "rows"), (3, "rows"), (2, "morton"), (3, "morton")])
def test_gloo_sharded_histogram_matches_full(world, split):
    """Pixel-row sharded histogram through the real exchange code
    (TensorExchange: all-to-all of the owners' runs, all-gather of the owner
    lists) over gloo: every rank ends with the whole image's Morton-ordered
    histogram, entry for entry (counts summed across row shards, first pixel =
    global minimum), although no rank counted every pixel."""
    img = gmm_image(97, 61, 12, 5)
    img[::7, ::3] = img[0, 0]  # a color repeated across every row shard
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hist_worker, args=(r, world, port, img, q, split)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in procs], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _full_histogram(img)
    for _, got in outs:
        np.testing.assert_array_equal(got, ref)


def test_sharded_histogram_emulated_matches_full():
    """The one-process emulation (the single-GPU check's data path) with the
    CPU stand-in: W = 1..5 row shards give the full histogram."""
    import torch

    from paper_1011_0093_b200.distributed import sharded_histogram_emulated

    img = gmm_image(64, 50, 9, 8)
    ref = _full_histogram(img)
    t = torch.from_numpy(img.reshape(-1).copy())
    for w in (1, 2, 3, 5):
        got = sharded_histogram_emulated(FakeHistBackend(), t, img.shape[0] * img.shape[1], w).numpy()
        np.testing.assert_array_equal(got, ref)
