"""Sharded WSM across GPUs (one process per GPU, torch.distributed plumbing).

Config 4 of BASELINE.json: the unique samples are split into contiguous
ranges of the Morton-ordered sample array, one per rank. Every iteration of
run_weighted_kmeans (kmeans.hpp:336-376) becomes:

  1. ``backend.step(lo, hi, C, first)`` -> this shard's EXACT integer cluster
     moments [5][K] (Σc·r, Σc·g, Σc·b, Σc, Σc·|x|²) + its point evaluations
     (the sharded launch of the same persistent CUDA loop, moments only);
  2. ``allreduce(sum)`` of the moments and evaluation counts (int64, exact);
  3. ``backend.finalize(moments, C)`` on every rank -> identical new centers,
     moment-form SSE and empty-cluster list (device kernel);
  4. empty clusters (rare): per-rank reseed candidate (distance desc, rank
     asc), ``allgather``, pick the global best — update_centers'
     kmeans.hpp:272-294 rule;
  5. termination (kmeans.hpp:359-369) evaluated identically on every rank.

Integer sums make the trajectory independent of the number of ranks and of
the summation order, so N ranks reproduce the single-GPU run bit for bit.

The backend is pluggable: ``DeviceShardBackend`` drives the CUDA library
through the C ABI; the CPU tests plug in a numpy stand-in. The collective is
pluggable too: ``TorchCollective`` (gloo on CPU, NCCL on GPUs) or
``LocalCollective`` (several shards in one process: the single-GPU check).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced range of n samples for `rank` of `world`."""
    return n * rank // world, n * (rank + 1) // world


def pair_evals(prev: np.ndarray | None, cur: np.ndarray) -> int:
    """Center-pair distance evaluations of update_center_tables
    (kmeans.hpp:137-155): all K(K-1)/2 on the first build, then only pairs
    with at least one center that changed bitwise."""
    k = cur.shape[0]
    total = k * (k - 1) // 2
    if prev is None:
        return total
    still = int(np.sum(np.all(prev == cur, axis=1)))
    return total - still * (still - 1) // 2


# --------------------------------------------------------------------------- collectives
class LocalCollective:
    """Single process; all shards are local (allreduce = identity)."""

    world = 1
    rank = 0

    def allreduce_sum(self, a: np.ndarray) -> np.ndarray:
        return a

    def allgather(self, obj):
        return [obj]


class TorchCollective:
    """torch.distributed collectives on host int64/float64 arrays. With the
    NCCL backend the tensors go through the current CUDA device."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    def allreduce_sum(self, a: np.ndarray) -> np.ndarray:
        t = self.torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy()).to(self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy().view(a.dtype).reshape(a.shape)

    def allgather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


# --------------------------------------------------------------------------- device backend
class DeviceShardBackend:
    """The CUDA library through the sharded C-ABI entry points."""

    def __init__(self, device: int = 0):
        from . import _native

        self.ctx = _native.context(device)
        self.lib = self.ctx.lib
        self.k = 0

    def prepare(self, img: np.ndarray, k: int, seed: int):
        a = np.ascontiguousarray(img, np.uint8)
        P = a.size // 3
        n = C.c_uint64()
        C0 = np.zeros((k, 3))
        self.ctx.check(self.lib.cqb_shard_prepare(self.ctx.h, a.ctypes.data_as(_u8p), P, k, seed, C.byref(n),
                                                  C0.ctypes.data_as(_f64p)))
        self.k, self.total = k, P
        return int(n.value), P, C0

    def step(self, lo: int, hi: int, centers: np.ndarray, first: bool):
        Cin = np.ascontiguousarray(centers, np.float64)
        mom = np.zeros((5, self.k), np.uint64)
        ev = C.c_uint64()
        self.ctx.check(self.lib.cqb_shard_step(self.ctx.h, lo, hi, Cin.ctypes.data_as(_f64p), int(first),
                                               mom.ctypes.data_as(_u64p), C.byref(ev)))
        return mom, int(ev.value)

    def finalize(self, moments: np.ndarray, centers: np.ndarray, total: int):
        k = centers.shape[0]
        mom = np.ascontiguousarray(moments, np.uint64)
        Cin = np.ascontiguousarray(centers, np.float64)
        out = np.zeros((k, 3))
        sse = C.c_double()
        ne = C.c_int()
        el = (C.c_int * max(k, 1))()
        self.ctx.check(self.lib.cqb_finalize_moments(self.ctx.h, mom.ctypes.data_as(_u64p), Cin.ctypes.data_as(_f64p),
                                                     k, total, out.ctypes.data_as(_f64p), C.byref(sse), C.byref(ne),
                                                     el))
        return out, float(sse.value), [int(el[i]) for i in range(ne.value)]

    def reseed_candidate(self, lo: int, hi: int, centers: np.ndarray, taken: list):
        Cin = np.ascontiguousarray(centers, np.float64)
        tk = np.array(taken if taken else [0], np.uint32)
        d = C.c_double()
        r = C.c_uint32()
        key = C.c_uint32()
        self.ctx.check(self.lib.cqb_shard_reseed_candidate(self.ctx.h, lo, hi, Cin.ctypes.data_as(_f64p),
                                                           tk.ctypes.data_as(_u32p), len(taken), C.byref(d),
                                                           C.byref(r), C.byref(key)))
        return float(d.value), int(r.value), int(key.value)


# --------------------------------------------------------------------------- driver
@dataclass
class ShardedResult:
    centers: np.ndarray
    iterations: int
    sse: float
    dist_evals: int
    sse_history: list = field(default_factory=list)
    trajectory: list = field(default_factory=list)
    n_unique: int = 0


def _better(a, b) -> bool:
    """Reseed order: distance desc, then first-occurrence rank asc."""
    return a[0] > b[0] or (a[0] == b[0] and a[1] < b[1])


def run_wsm_sharded(backend, img: np.ndarray, k: int, mode: int = 1, max_iters: int = 10, eps: float = 1e-4,
                    cap: int = 100, seed: int = 1, coll=None, shards: int | None = None) -> ShardedResult:
    """WSM (mode 0) / WSM-C (mode 1) with the samples sharded over the ranks
    of `coll` (each rank owns one contiguous range). With LocalCollective and
    `shards` = W, one process runs W shards sequentially — the single-GPU
    check that sharding is exact."""
    coll = coll or LocalCollective()
    n, total, Cur = backend.prepare(img, k, seed)
    if shards is None:
        my = [shard_range(n, coll.world, coll.rank)]
    else:
        my = [shard_range(n, shards, r) for r in range(shards)]
    prev_sse = math.inf
    evals = 0
    res = ShardedResult(Cur, 0, 0.0, 0, n_unique=n)
    Cprev = None
    it = 0
    while True:
        it += 1
        evals += pair_evals(Cprev, Cur) if coll.rank == 0 else 0
        mom = np.zeros((5, k), np.uint64)
        ev = 0
        for lo, hi in my:
            m, e = backend.step(lo, hi, Cur, it == 1)
            mom += m
            ev += e
        mom = coll.allreduce_sum(mom)
        evals += ev
        Cnew, sse, empties = backend.finalize(mom, Cur, total)
        taken: list = []
        for e_cl in empties:
            best = (-1.0, 0xFFFFFFFF, 0)
            for lo, hi in my:
                cand = backend.reseed_candidate(lo, hi, Cur, taken)
                if _better(cand, best):
                    best = cand
            for cand in coll.allgather(best):
                if _better(cand, best):
                    best = cand
            taken.append(best[1])
            key = best[2]
            Cnew[e_cl] = ((key >> 16) & 255, (key >> 8) & 255, key & 255)
        res.sse_history.append(sse)
        res.trajectory.append(Cnew.copy())
        Cprev, Cur = Cur, Cnew
        if mode == 0:
            stop = it >= max_iters
        else:
            stop = sse == 0.0 or (prev_sse - sse) / sse <= eps or it >= cap
        prev_sse = sse
        if stop:
            break
    total_evals = coll.allreduce_sum(np.array([evals], np.uint64))[0]
    res.centers, res.iterations, res.sse, res.dist_evals = Cur, it, res.sse_history[-1], int(total_evals)
    return res


# --------------------------------------------------------------------------- in-kernel exchange
class PeerShardedQuantizer:
    """Config 4 across GPUs with the moment exchange INSIDE the persistent
    loop kernel (cqb_quantize_sharded): one process per GPU, each rank's loop
    writes its K x 5 exact moment sums into every peer's exchange window over
    NVLink once per iteration and sums the world's contributions itself — no
    host round trip and no collective call per iteration. The windows are
    cudaIpc-shared; torch.distributed only all-gathers the handles once.

    ``emulate=W`` (single GPU, tests): W block groups of the one cooperative
    launch act as the W ranks, with the same windows, flags and exchange code.
    """

    def __init__(self, ctx=None, group=None, emulate: int = 0, device: int = 0):
        from . import _native

        self.ctx = ctx or _native.context(device)
        self.lib = self.ctx.lib
        if emulate:
            self.world, self.rank, self.emulated = emulate, 0, True
            self.ctx.check(self.lib.cqb_xch_emulate(self.ctx.h, emulate))
            return
        import torch.distributed as dist

        single = not (dist.is_available() and dist.is_initialized())  # one rank: the X = 1 kernel alone
        self.world = 1 if single else dist.get_world_size(group)
        self.rank = 0 if single else dist.get_rank(group)
        self.emulated = False
        h = (C.c_ubyte * _native.IPC_HANDLE_BYTES)()
        self.ctx.check(self.lib.cqb_xch_window(self.ctx.h, self.world, self.rank, h))
        handles = [bytes(h)] if single else exchange_handles(bytes(h), group)
        buf = C.create_string_buffer(b"".join(handles), len(handles) * _native.IPC_HANDLE_BYTES)
        self.ctx.check(self.lib.cqb_xch_open(self.ctx.h, buf))

    def enqueue(self, d_rgb: int, n_pixels: int, k: int, term, seed: int = 1, d_index: int | None = None,
                d_rgb_out: int | None = None) -> tuple[int, int]:
        """Enqueue one sharded quantize on the context stream (device
        pointers); returns the pixel range this rank maps."""
        rng = np.zeros(2, np.uint64)
        t = term.native()
        self.ctx.check(self.lib.cqb_quantize_sharded(self.ctx.h, d_rgb, n_pixels, k, C.byref(t), seed, d_index,
                                                     d_rgb_out, rng.ctypes.data_as(_u64p)))
        self._k, self._cap = k, term.iteration_budget
        return int(rng[0]), int(rng[1])

    def enqueue_rows(self, img, n_pixels: int, k: int, term, seed: int = 1, d_index: int | None = None,
                     d_rgb_out: int | None = None, group=None, split: str = "rows") -> tuple[int, int]:
        """cqb_quantize_sharded with the histogram sharded too (``img``: the
        raster as a CUDA uint8 tensor on every rank). split="rows": this rank
        counts only its pixel rows, the owners merge (all-to-all);
        split="morton": this rank counts every pixel into its own Morton range
        of bins. Either way the whole histogram is then all-gathered (NCCL)
        and the loop and the map run as in enqueue."""
        backend = DeviceHistBackend(self.ctx)
        emu = sharded_histogram_emulated if split == "rows" else sharded_histogram_morton_emulated
        real = sharded_histogram if split == "rows" else sharded_histogram_morton
        if self.emulated:
            samples = emu(backend, img, n_pixels, self.world)
        else:
            import torch.distributed as dist

            if dist.is_available() and dist.is_initialized():
                samples = real(backend, img, n_pixels, TensorExchange(group))
            else:
                samples = emu(backend, img, n_pixels, 1)
        self._samples = samples  # alive until the enqueued work has read it (fetch)
        rng = np.zeros(2, np.uint64)
        t = term.native()
        self.ctx.check(self.lib.cqb_quantize_sharded_samples(self.ctx.h, img.data_ptr(), n_pixels, samples.data_ptr(),
                                                             samples.shape[0], k, C.byref(t), seed, d_index,
                                                             d_rgb_out, rng.ctypes.data_as(_u64p)))
        self._k, self._cap = k, term.iteration_budget
        return int(rng[0]), int(rng[1])

    def fetch(self):
        """Wait; return (centers [k,3], report, sse_history). report.dist_evals
        is this rank's share (sum over ranks for the reference's count)."""
        from . import _native as N

        k, cap = self._k, self._cap
        centers = np.zeros(3 * k)
        hist = np.zeros(cap)
        rep = N.Report()
        self.ctx.check(self.lib.cqb_fetch_results(self.ctx.h, centers.ctypes.data_as(_f64p),
                                                  hist.ctypes.data_as(_f64p), cap, C.byref(rep)))
        return centers.reshape(k, 3), rep, hist[: rep.iterations].copy()


def pixel_range(n_pixels: int, world: int, rank: int) -> tuple[int, int]:
    """The raster slice rank ``rank`` maps in cqb_quantize_sharded (capi.cu):
    contiguous, 16-pixel aligned starts (16-B vector stores), the last rank
    takes the tail."""
    q = (n_pixels + 15) // 16
    lo = min(n_pixels, q * rank // world * 16)
    hi = n_pixels if rank == world - 1 else min(n_pixels, q * (rank + 1) // world * 16)
    return lo, hi


def exchange_handles(handle: bytes, group=None) -> list[bytes]:
    """All-gather of the ranks' IPC handles, in rank order (host plumbing)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    assert all(isinstance(h, bytes) and len(h) == len(handle) for h in out)
    return out


# --------------------------------------------------------------------------- sharded histogram
# build_histogram (histogram.hpp:65-99) split over the ranks by pixel rows,
# with bin ownership by Morton range (include/colorq_b200.h, cqb_hist_rows):
# rank r counts the rows it maps, sends each owner its run of touched bins,
# owners merge and compact, and the owners' lists are all-gathered — the
# whole image's Morton-ordered histogram, identical to the unsharded one,
# without any rank counting every pixel.
class DeviceHistBackend:
    """cqb_hist_rows / cqb_hist_merge on one context (tensors on its GPU)."""

    def __init__(self, ctx):
        self.ctx, self.lib = ctx, ctx.lib

    def rows(self, img, n_pixels: int, world: int, rank: int):
        import torch

        lo, hi = pixel_range(n_pixels, world, rank)
        out = torch.empty((max(hi - lo, 1), 3), dtype=torch.int32, device=img.device)
        n = C.c_uint64()
        counts = np.zeros(world, np.uint64)
        self.ctx.check(self.lib.cqb_hist_rows(self.ctx.h, img.data_ptr(), n_pixels, world, rank, out.data_ptr(),
                                              out.shape[0], C.byref(n), counts.ctypes.data_as(_u64p)))
        return out[: n.value], [int(c) for c in counts]

    def range(self, img, n_pixels: int, world: int, rank: int):
        """cqb_hist_range: every pixel counted into this rank's Morton range
        only; returns its owner list (Morton-ordered triplets)."""
        import torch

        # the range is whole compaction tiles (<= 16384 bins each) around 2^24 / world bins
        cap = max(1, min(n_pixels, (1 << 24) // world + (1 << 14)))
        out = torch.empty((cap, 3), dtype=torch.int32, device=img.device)
        n = C.c_uint64()
        self.ctx.check(self.lib.cqb_hist_range(self.ctx.h, img.data_ptr(), n_pixels, world, rank, out.data_ptr(),
                                               cap, C.byref(n)))
        return out[: n.value]

    def merge(self, recv, world: int):
        import torch

        cap = max(1, min(recv.shape[0], ((1 << 24) + world - 1) // world + 1))
        out = torch.empty((cap, 3), dtype=torch.int32, device=recv.device)
        n = C.c_uint64()
        self.ctx.check(self.lib.cqb_hist_merge(self.ctx.h, recv.data_ptr() if recv.shape[0] else None,
                                               recv.shape[0], out.data_ptr(), cap, C.byref(n)))
        return out[: n.value]


class TensorExchange:
    """All-to-all and all-gather of [n, 3] int32 sample triplets over a
    torch.distributed group (NCCL for CUDA tensors, gloo for CPU ones)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def alltoallv(self, send, send_counts: list):
        import torch
        import torch.distributed as dist

        sc = torch.tensor(send_counts, dtype=torch.int64, device=send.device)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = [int(v) for v in rc.tolist()]
        recv = torch.empty((sum(recv_counts), 3), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=recv_counts,
                               input_split_sizes=list(send_counts), group=self.group)
        return recv

    def allgatherv(self, t):
        import torch
        import torch.distributed as dist

        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ns = torch.empty(self.world, dtype=torch.int64, device=t.device)
        dist.all_gather_into_tensor(ns, n, group=self.group)
        sizes = [int(v) for v in ns.tolist()]
        m = max(sizes)
        pad = torch.zeros((m, 3), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        out = torch.empty((self.world * m, 3), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, pad, group=self.group)
        return torch.cat([out[r * m: r * m + sizes[r]] for r in range(self.world)])


def sharded_histogram(backend, img, n_pixels: int, exchange):
    """This rank's share of the pixel-row sharded histogram; returns the whole
    image's Morton-ordered {key, count, first pixel} triplets (every rank)."""
    _sync(img)
    local, counts = backend.rows(img, n_pixels, exchange.world, exchange.rank)
    recv = exchange.alltoallv(local, counts)
    _sync(recv)
    own = backend.merge(recv, exchange.world)
    out = exchange.allgatherv(own)
    _sync(out)
    return out


def sharded_histogram_morton(backend, img, n_pixels: int, exchange):
    """Morton-range split: every rank holds the raster and counts all its
    pixels, but only into the bins of its own Morton range (no all-to-all:
    each owner list is complete); the lists are all-gathered (NCCL)."""
    _sync(img)
    own = backend.range(img, n_pixels, exchange.world, exchange.rank)
    out = exchange.allgatherv(own)
    _sync(out)
    return out


def sharded_histogram_morton_emulated(backend, img, n_pixels: int, world: int):
    """The Morton-range split in one process (single-GPU check)."""
    import torch

    _sync(img)
    out = torch.cat([backend.range(img, n_pixels, world, r) for r in range(world)])
    _sync(out)
    return out


def _sync(t):
    """The library's stream reads what torch's stream produced (and back)."""
    if getattr(t, "is_cuda", False):
        import torch

        torch.cuda.current_stream(t.device).synchronize()


def sharded_histogram_emulated(backend, img, n_pixels: int, world: int):
    """The same data path in one process: the W ranks' row counts in
    sequence, the all-to-all and all-gather as slicing (single-GPU check)."""
    import torch

    _sync(img)
    runs = [backend.rows(img, n_pixels, world, r) for r in range(world)]
    owners = []
    for o in range(world):
        parts = [loc[sum(c[:o]): sum(c[: o + 1])] for loc, c in runs]
        recv = torch.cat(parts)
        _sync(recv)
        owners.append(backend.merge(recv, world))
    out = torch.cat(owners)
    _sync(out)
    return out
