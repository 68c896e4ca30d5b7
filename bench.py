#!/usr/bin/env python
"""Benchmark of the B200 WSM quantize path (BASELINE.json metric
"WSM quantize Mpixel/s at K=256").

Workload (default): BASELINE config 2 (768x512 GMM-256 image, K=256,
convergent(1e-4, cap 100), init seed 1) — configs[1], the config the metric is
quoted on. One step = one full quantize (histogram + WSM-C + map + MSE) of one
image per rank. N > 1 (torchrun): every rank quantizes its own image (replica
/ weak scaling, no data-path collective). `--config cfg4` selects the
4096x4096 uniform config instead.

  value : P * ranks / (max over ranks of the per-step device time), image
          resident in HBM, CUDA events on the library stream, L2 flushed
          (256 MiB write) between timed steps.
  e2e   : the same metric through the public C-ABI call (cqb_quantize) with
          pinned HOST buffers: H2D of the image and D2H of the index map,
          mapped raster, palette and report inside the timed region.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified colorq headers compiled here) on all host cores,
one image per worker thread (the bench.hpp:187-223 pool pattern).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1011_0093_b200.configs import CONFIGS, EPSILON, HARD_CAP, INIT_SEED  # noqa: E402

METRIC = "WSM quantize Mpixel/s at K=256"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--k", type=int, default=None, help="default: 256 if the config lists it, else its K")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="shard the unique samples over the ranks (in-kernel NVLink exchange); default for cfg4 at N>1")
    ap.add_argument("--hist", choices=["replicated", "rows", "morton"], default=None,
                    help="sharded path: histogram replicated on every rank (default at N=1), sharded by pixel rows "
                         "with a Morton-range bin ownership exchange (cqb_hist_rows / cqb_hist_merge + NCCL), or "
                         "by Morton range over every pixel (cqb_hist_range + NCCL all-gather; default at N>1)")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="single GPU: W block groups of the loop act as W sharded ranks (exchange overhead)")
    return ap.parse_args()


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


E2E_INFLIGHT = 3  # concurrent host callers of the e2e measurement
RED_PAIRS_PEAK = 106.3e9  # random RED pairs/s on a 32 MiB bin slice (profiles/r02/microbench_mem.txt)


def _workload(cfg, k):
    return (f"{cfg.name}: {cfg.width}x{cfg.height} {cfg.description}; K={k}; "
            f"convergent(eps={EPSILON}, cap={HARD_CAP}); init seed {INIT_SEED}")


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x0000000000000008: "hw_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000004: "sw_power_cap",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


# --------------------------------------------------------------------------- reference arm
def run_reference(a, cfg, world, rank):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    colorq headers compiled here) on the same config. One step = one full
    quantize of one image (histogram + WSM-C + map + mse) on one host thread;
    the steps run `cores` at a time on a native thread pool (the
    bench.hpp:187-223 pattern), because the reference has no intra-image
    parallelism. The timed count is rounded up to whole waves of `cores`
    images so every thread stays busy: value = images * P / wall."""
    if rank != 0:
        return None
    from oracle.oracle import Oracle, available

    if not available("reference"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libcolorq_ref.so not built"}))
        return None
    ref = Oracle("reference")
    cores = _host_cores()
    P = cfg.pixels
    n_timed = max(1, math.ceil(a.steps / cores)) * cores
    distinct = cfg.images > 1  # config 5: every image its own seed
    imgs = [cfg.image(i) for i in range(min(n_timed, cfg.images))] if distinct else [cfg.image()]
    if a.warmup > 0:
        w = [imgs[i % len(imgs)] for i in range(min(a.warmup, cores))]
        ref.quantize_many(w, a.k, cores, mode=1, eps=EPSILON, cap=HARD_CAP, seed=INIT_SEED)
    timed = [imgs[i % len(imgs)] for i in range(n_timed)]
    ms, mses, its = ref.quantize_many(timed, a.k, cores, mode=1, eps=EPSILON, cap=HARD_CAP, seed=INIT_SEED)
    value = P * n_timed / (ms * 1e-3) / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": "Mpixel/s", "impl": "reference", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / n_timed,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": _workload(cfg, a.k), "pixels": P, "images_timed": n_timed, "threads": cores,
                   "timed": "wall clock of the whole timed pool (images_timed full quantizes, `threads` at a time)"},
        "cpu_baseline": {"value": value, "unit": "Mpixel/s", "cores": cores, "kind": "reference",
                         "sample": f"{n_timed} full quantizes of the {cfg.name} image ({P} px, K={a.k}) on "
                                   f"{cores} threads, one image per thread (oracle/_ref, g++ -O2), "
                                   f"iterations={int(its[0])}, wall {ms / 1e3:.1f} s"},
        "e2e": {"value": value, "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return line


def cpu_baseline_sample(cfg, k, img):
    """oracle/_ref on all host cores, one image per thread, bounded to ~10-30 s:
    the 4096^2 configs use their top-left 2048x2048 quarter (the reference
    needs ~50 s per full cfg4 image on one core)."""
    from oracle.oracle import Oracle, available

    if not available("reference"):
        return None
    ref = Oracle("reference")
    cores = _host_cores()
    if cfg.pixels > (8 << 20):
        sub = np.ascontiguousarray(img[:2048, :2048])
        what = f"the top-left 2048x2048 quarter of the {cfg.name} image"
    else:
        sub = img
        what = f"the {cfg.name} image"
    px = sub.shape[0] * sub.shape[1]
    ms, _, its = ref.quantize_many([sub] * cores, k, cores, mode=1, eps=EPSILON, cap=HARD_CAP, seed=INIT_SEED)
    return {"value": px * cores / (ms * 1e-3) / 1e6, "unit": "Mpixel/s", "cores": cores, "kind": "reference",
            "sample": f"{cores} concurrent copies of {what} (one per thread), full quantize "
                      f"(histogram+WSM-C K={k}+map+mse), {int(its[0])} iterations, wall {ms:.0f} ms"}


# --------------------------------------------------------------------------- our arm
def measure_device(lib, ctx, torch, d_img, P, k, steps, warmup, stream, flush, profile=False):
    """Per-step device time (ms) with CUDA events on the library stream."""
    from paper_1011_0093_b200 import _native as N

    term = N.Termination(1, 10, EPSILON, HARD_CAP)
    d_idx = torch.empty(P, dtype=torch.uint8, device=d_img.device)
    d_out = torch.empty(3 * P, dtype=torch.uint8, device=d_img.device)
    rep = N.Report()
    hist = np.zeros(HARD_CAP)
    cent = np.zeros(3 * k)

    def one(sync):
        rc = lib.cqb_quantize_device(ctx.h, C.c_void_p(d_img.data_ptr()), P, k, C.byref(term), INIT_SEED,
                                     C.c_void_p(d_idx.data_ptr()), C.c_void_p(d_out.data_ptr()), sync,
                                     cent.ctypes.data_as(C.POINTER(C.c_double)),
                                     hist.ctypes.data_as(C.POINTER(C.c_double)), HARD_CAP, C.byref(rep))
        ctx.check(rc)

    times, stage = [], []
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches = 0
    with torch.cuda.stream(stream):  # flush, events and the library share one stream
        for _ in range(warmup):
            flush()
            one(1)
        for i in range(steps):
            flush()
            evs[i][0].record(stream)
            one(0)
            evs[i][1].record(stream)
            if profile:
                ms = (C.c_float * 7)()
                ctx.check(lib.cqb_stage_times(ctx.h, ms, 7))
                tl = np.zeros(8 * HARD_CAP, np.uint64)
                ctx.check(lib.cqb_loop_timeline(ctx.h, tl.ctypes.data_as(C.POINTER(C.c_uint64)), HARD_CAP))
                stage.append((list(ms), tl.reshape(HARD_CAP, 8).astype(np.int64)))
    torch.cuda.synchronize()
    for a, b in evs:
        times.append(a.elapsed_time(b))
    ctx.check(lib.cqb_fetch_results(ctx.h, cent.ctypes.data_as(C.POINTER(C.c_double)),
                                    hist.ctypes.data_as(C.POINTER(C.c_double)), HARD_CAP, C.byref(rep)))
    launches = steps * int(rep.gpu_launches)  # kernels of the library per quantize (counted by the C ABI)
    return times, stage, rep, cent.reshape(k, 3).copy(), launches


def run_ours(a, cfg, world, rank, local):
    import torch
    import torch.distributed as dist

    from paper_1011_0093_b200 import _native as N
    from paper_1011_0093_b200 import api

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    ctx = N.context(local)
    lib = ctx.lib
    stream = torch.cuda.Stream(device=dev)
    ctx.check(lib.cqb_set_stream(ctx.h, C.c_void_p(stream.cuda_stream)))
    img = cfg.image()  # every rank: its own replica of the config image
    P = cfg.pixels
    k = a.k
    d_img = torch.from_numpy(img.reshape(-1)).to(dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.fill_(1)  # > L2 (126 MB): evicts the previous step's working set

    # ---- device-resident timing (value) ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t_wall0 = time.perf_counter()
    times, _, rep, centers, launches = measure_device(lib, ctx, torch, d_img, P, k, a.steps, a.warmup, stream, flush)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = P * world * a.steps / (total_ms * 1e-3) / 1e6

    # ---- per-stage attribution + roofline of the dominant kernel ----
    ctx.check(lib.cqb_set_profiling(ctx.h, 1))
    _, stage, rep_p, _, _ = measure_device(lib, ctx, torch, d_img, P, k, max(3, min(a.steps, 5)), 1, stream, flush,
                                           profile=True)
    ctx.check(lib.cqb_set_profiling(ctx.h, 0))
    st = np.median(np.array([x[0] for x in stage]), axis=0)
    names = N.STAGES
    stage_ms = {n: float(v) for n, v in zip(names, st)}
    n_unique = int(rep.n_unique)
    iters = int(rep.iterations)
    phases = _loop_phases(stage[-1][1], iters)
    peaks = _peaks()
    dom = max(stage_ms, key=stage_ms.get)
    if dom == "wsm_loop":
        evals1 = first_iteration_evals(lib, ctx, torch, d_img, P, k, stream)
        roof = _loop_roofline(stage_ms[dom], P, n_unique, iters, k, peaks, int(rep.dist_evals), evals1, phases)
    else:
        roof = _roofline(dom, stage_ms[dom], P, n_unique, iters, k, peaks, int(rep.dist_evals))

    # ---- e2e through the public C-ABI call with pinned host buffers ----
    # outputs as the reference's pipeline (methods.hpp generate_palette ->
    # image_ops.hpp map_pixels -> metrics.hpp mse): palette, mapped raster,
    # MSE and the run report; no index map
    # E2E_INFLIGHT host threads, each with its own context, stream and pinned
    # buffers, call the API concurrently (a host-side image stream): one
    # call's H2D / D2H copies overlap another call's kernels. Every step is
    # one complete host-to-host quantize; the timed region is the wall clock
    # from the first call's start to the last call's return.
    term = api.Termination.convergent(EPSILON, HARD_CAP)
    ctx.check(lib.cqb_set_stream(ctx.h, None))
    bufs = []
    for _ in range(E2E_INFLIGHT):
        pin_img = torch.from_numpy(img.reshape(-1)).pin_memory()
        pin_out = torch.empty(3 * P, dtype=torch.uint8).pin_memory()
        bufs.append((pin_img, pin_out, pin_img.numpy().reshape(img.shape), pin_out.numpy().reshape(img.shape)))

    def e2e_worker(j, n):
        torch.cuda.set_device(local)
        h_img, h_out = bufs[j][2], bufs[j][3]
        q = None
        for _ in range(n):
            q = api.quantize(h_img, k, term, INIT_SEED, index_map=False, out_mapped=h_out, device=local)
        return q

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(E2E_INFLIGHT) as ex:
        list(ex.map(lambda j: e2e_worker(j, max(1, a.warmup)), range(E2E_INFLIGHT)))
        flush()
        torch.cuda.synchronize()
        shares = [a.steps // E2E_INFLIGHT + (1 if j < a.steps % E2E_INFLIGHT else 0) for j in range(E2E_INFLIGHT)]
        t0 = time.perf_counter()
        outs = list(ex.map(lambda j: e2e_worker(j, shares[j]), range(E2E_INFLIGHT)))
        e2e_s = time.perf_counter() - t0
    q = outs[0]
    for j in range(E2E_INFLIGHT):
        assert shares[j] == 0 or np.array_equal(bufs[j][3], bufs[0][3]), "e2e lanes disagree"
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = P * world * a.steps / e2e_s / 1e6
    assert np.array_equal(q.palette, centers), "e2e and device-resident paths disagree"

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload(cfg, k), "pixels": P, "n_unique": n_unique, "iterations": iters,
                       "k": k, "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "timed": "per-step CUDA events on the library stream; value = P*ranks*steps / max-rank sum",
                       "wall_bracket_s": round(t_wall, 4)},
            "e2e": {"value": e2e_value, "unit": "Mpixel/s", "h2d_bytes_per_step": 3 * P,
                    "d2h_bytes_per_step": 3 * P + 8 * 3 * k + 8 * HARD_CAP + 64,
                    "inflight": E2E_INFLIGHT,
                    "path": f"cqb_quantize_ex (C ABI) with pinned host buffers, wall clock over all steps, "
                            f"{E2E_INFLIGHT} host threads calling concurrently (own context + stream each, so "
                            f"one call's copies overlap another's kernels); outputs as the reference pipeline: "
                            f"palette, mapped raster, MSE, report; H2D / D2H in 8 slices overlapped with the "
                            f"histogram count and the map"},
            "gpu_launches": launches,
            "roofline": roof,
            "hbm_stages": _hbm_stages(stage_ms, P, n_unique, peaks),
            "stages_ms": {kk: round(v, 5) for kk, v in stage_ms.items()},
            "loop_phases_us": phases,
            "dist_evals": int(rep.dist_evals),
            "clocks": clk,
        }
        if world == 1 and not a.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample(cfg, k, img)
        if world == 1 and not a.no_secondary:
            line["other_configs"] = other_configs(lib, ctx, torch, dev, stream, flush, skip=(cfg.name, k))
            line["secondary_cfg5"] = batch_cfg5(ctx, torch, dev, stream, flush, n_images=16, steps=2, warmup=1)
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return line


def other_configs(lib, ctx, torch, dev, stream, flush, skip=None):
    """The other single-image BASELINE configs at each of their K,
    device-resident (same protocol as `value`, 5 timed steps, L2 flushed)."""
    out = {}
    for name, k in (("cfg1", 32), ("cfg2", 64), ("cfg2", 256), ("cfg3", 256), ("cfg4", 256)):
        if (name, k) == skip:
            continue
        cfg = CONFIGS[name]
        d = torch.from_numpy(cfg.image().reshape(-1)).to(dev)
        ctx.check(lib.cqb_set_stream(ctx.h, C.c_void_p(stream.cuda_stream)))
        times, _, rep, _, _ = measure_device(lib, ctx, torch, d, cfg.pixels, k, 5, 2, stream, flush)
        ms = sum(times) / len(times)
        out[f"{name}_k{k}"] = {"value": cfg.pixels / (ms * 1e-3) / 1e6, "unit": "Mpixel/s", "ms_per_step": ms,
                               "n_unique": int(rep.n_unique), "iterations": int(rep.iterations),
                               "dist_evals": int(rep.dist_evals)}
    return out


def batch_cfg5(ctx, torch, dev, stream, flush, n_images=16, steps=2, warmup=1, lanes_list=(1, 4)):
    """Config 5: independent 1024x1024 GMM-256 images (seeds 1000+i), K=256,
    device-resident, `lanes` images in flight on this GPU (cqb_quantize_batch).
    Aggregate Mpixel/s from CUDA events on the caller's stream (the batch call
    joins its lane streams back into it)."""
    from paper_1011_0093_b200 import api

    cfg = CONFIGS["cfg5"]
    imgs = [torch.from_numpy(cfg.image(i).reshape(-1)).to(dev) for i in range(n_images)]
    term = api.Termination.convergent(EPSILON, HARD_CAP)
    out = {"workload": f"cfg5: {n_images} x {cfg.width}x{cfg.height} GMM-256 images (seeds 1000+i), K=256, "
                       f"convergent(eps={EPSILON}, cap={HARD_CAP})", "unit": "Mpixel/s"}
    ctx.check(ctx.lib.cqb_set_stream(ctx.h, C.c_void_p(stream.cuda_stream)))
    with torch.cuda.stream(stream):
        for lanes in lanes_list:
            for _ in range(warmup):
                api.quantize_batch_device(imgs, 256, term, INIT_SEED, lanes=lanes)
            tot = 0.0
            for _ in range(steps):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _, reps = api.quantize_batch_device(imgs, 256, term, INIT_SEED, lanes=lanes)
                e1.record(stream)
                e1.synchronize()
                tot += e0.elapsed_time(e1)
            out[f"lanes{lanes}"] = {"value": cfg.pixels * n_images * steps / (tot * 1e-3) / 1e6,
                                    "ms_per_batch": tot / steps,
                                    "iterations": [r.iterations for r in reps[:8]]}
    return out


def _loop_phases(tl, iters):
    """Mean per-iteration phase durations (us) of block 0 from the loop's
    globaltimer stamps (iterations >= 2; iteration 1 reported separately)."""
    tl = tl[:iters]
    if iters < 3 or not tl[:, 0].all():
        return None
    a = tl[1:-1]
    nxt = tl[2:, 0]
    d = lambda x, y: float(np.mean(y - x)) / 1e3  # noqa: E731
    return {
        "iter1_assign_us": float(tl[0, 3] - tl[0, 0]) / 1e3,
        "points_us": d(a[:, 0], a[:, 2]),
        "flush_us": d(a[:, 2], a[:, 3]),
        "barrier1_us": d(a[:, 3], a[:, 4]),
        "finalize_us": d(a[:, 4], a[:, 5]),
        "tables_us": d(a[:, 5], a[:, 6]),
        "barrier2_us": d(a[:, 6], nxt),
        "iteration_us": float(np.mean(np.diff(tl[1:, 0]))) / 1e3,
        "changed_per_iter": [int(v) & 0xFFFFFFFF for v in tl[1:8, 7]],
        "active_per_iter": [int(v) >> 32 for v in tl[1:8, 7]],
        "changed_mean": float(np.mean(tl[1:, 7] & 0xFFFFFFFF)),
        "active_mean": float(np.mean(tl[1:, 7] >> 32)),
    }


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def _roofline(stage, ms, P, n_unique, iters, k, peaks, evals):
    """Algorithmic bytes per launch of the dominant kernel."""
    if stage == "wsm_loop":
        # per iteration per sample: u32 key + u32 count + u8 label read + u8 label write
        traffic_alg = 10.0 * n_unique * iters
        note = (f"10 B/sample/iteration x N'={n_unique} x {iters} iterations; "
                f"{evals / (ms * 1e-3) / 1e9:.2f} G dist evals/s")
    elif stage in ("hist_count",):
        traffic_alg = 3.0 * P
        note = "3P bytes (u8x3 raster read); bin atomics not counted"
    elif stage == "bins_compact":
        traffic_alg = 8.0 * (1 << 24) + 12.0 * n_unique
        note = "128 MiB bin-table scan + 12 B per unique color written (Morton samples)"
    elif stage == "prep_small":
        traffic_alg = 3.0 * P + 2.0 * (1 << 21) + 12.0 * n_unique
        note = "3P raster read + 2 MiB occupancy bitmap written and read + 12 B per unique color written"
    elif stage == "map_pixels":
        traffic_alg = 7.0 * P
        note = "3P read + P index + 3P RGB written"
    else:
        traffic_alg = 8.0 * n_unique
        note = "8 B per unique color"
    achieved = traffic_alg / (ms * 1e-3) / 1e9
    out = {"kernel": stage, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
           "frac": achieved / peaks["hbm_gbs"], "traffic": _ncu_traffic(stage, P), "kernel_ms": ms,
           "algorithmic_bytes": traffic_alg, "peak_source": peaks["source"], "note": note}
    if stage == "wsm_loop" and evals:
        # BASELINE's second metric: point-center evaluations/s against the FP64
        # issue roofline (8 FP64 ops per evaluation, no FMA; DADD/DMUL peak
        # measured by tools/microbench.cu: 62.4 ops/SM/clk -> profiles/r01/microbench_primitives.txt)
        fp64_ops = 18.16e12
        out["evals_roofline"] = {"achieved_evals_per_s": evals / (ms * 1e-3), "peak_evals_per_s": fp64_ops / 8,
                                 "frac": evals / (ms * 1e-3) / (fp64_ops / 8),
                                 "peak_source": "measured DADD/DMUL throughput / 8 ops per evaluation"}
    return out


# Measured CUDA-core issue rate (tools/microbench.cu on this B200 pool,
# profiles/r01/microbench_primitives.txt): 111.4 FADD per SM per clock.
F32_ISSUE_PER_S = 32.41e12
FLOP_PER_EVAL = 8    # 3 sub, 3 mul, 2 add per distance evaluation
SLOTS_PER_EVAL = 6   # SURVEY.md §8(d)'s model: 3 FSUB + FMUL + 2 FFMA issue slots per evaluation (the kernel's own
                     # candidate evaluations are 3 FFMA each in difference form, scan_f32e; its own-center ones are 6)


def first_iteration_evals(lib, ctx, torch, d_img, P, k, stream):
    """dist_evals of a one-iteration run (fixed(1)) = iteration 1's point
    evaluations + the k(k-1)/2 pairs of the initial center tables."""
    from paper_1011_0093_b200 import _native as N

    term = N.Termination(0, 1, EPSILON, HARD_CAP)
    rep = N.Report()
    cent = np.zeros(3 * k)
    with torch.cuda.stream(stream):
        ctx.check(lib.cqb_quantize_device(ctx.h, C.c_void_p(d_img.data_ptr()), P, k, C.byref(term), INIT_SEED,
                                          None, None, 1, cent.ctypes.data_as(C.POINTER(C.c_double)), None, 0,
                                          C.byref(rep)))
    return int(rep.dist_evals)


def _loop_roofline(ms, P, n_unique, iters, k, peaks, evals, evals1, phases):
    """Roofline of the persistent WSM loop (k_wsm_loop), SURVEY.md §8(d).

    Algorithmic work = the reference's own dist_evals (exact, kmeans.hpp:214,
    228, 237) at 8 FLOP each. Iterations >= 2 (FP32-screened sort-means
    scans, the bulk of the launch) are reported as the headline: achieved =
    8 * E(>=2) / their time, peak = 8/6 * the measured FP32 issue rate (6
    issue slots per evaluation). Iteration 1 (integer dp4a over per-cell
    candidate lists, which skip most of the reference's evaluations) is
    reported separately. `model` is §8(d)'s per-launch floor
    max(E1*6/F32, 10 N'/BW) + max(E(>=2)*6/F32, (I-1)*10 N'/BW) against the
    measured loop time."""
    pairs0 = k * (k - 1) // 2
    e1 = max(evals1 - pairs0, 0)
    e_rest = max(evals - evals1, 0)  # includes the later tables' pair evaluations (< 0.1%)
    t = ms * 1e-3
    t1 = (phases or {}).get("iter1_assign_us", 0.0) * 1e-6
    t_rest = max(t - t1, 1e-12)
    peak = FLOP_PER_EVAL / SLOTS_PER_EVAL * F32_ISSUE_PER_S / 1e12
    achieved = FLOP_PER_EVAL * e_rest / t_rest / 1e12
    bw = peaks["hbm_gbs"] * 1e9
    mem_iter = 10.0 * n_unique / bw
    t_roof = max(e1 * SLOTS_PER_EVAL / F32_ISSUE_PER_S, mem_iter) + max(
        e_rest * SLOTS_PER_EVAL / F32_ISSUE_PER_S, (iters - 1) * mem_iter)
    return {
        "kernel": "k_wsm_loop", "bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved / peak, "traffic": _ncu_traffic("wsm_loop", P), "kernel_ms": ms,
        "peak_source": "measured FADD issue rate 32.41e12/s (tools/microbench.cu) x 8 FLOP / 6 slots",
        "note": (f"iterations 2..{iters}: {e_rest} reference distance evaluations (8 FLOP each) in "
                 f"{t_rest * 1e3:.3f} ms; candidates are evaluated in difference form (one 16-B shared load + 3 FFMA), "
                 f"the loop is issue/latency-bound (ncu: 70% of the SM issue rate, 24 of 32 threads active), "
                 f"its working set ({10 * n_unique / 1e6:.0f} MB per iteration) stays in L2"),
        "iteration1": {"evals": e1, "us": t1 * 1e6,
                       "reference_evals_per_s": e1 / t1 if t1 > 0 else None,
                       "note": "integer dp4a argmin over per-16^3-cell candidate lists: most of the "
                               "reference's evaluations are never performed"},
        "model": {"t_roof_us": t_roof * 1e6, "t_meas_us": t * 1e6, "frac": t_roof / t,
                  "compute_us": (e1 + e_rest) * SLOTS_PER_EVAL / F32_ISSUE_PER_S * 1e6,
                  "memory_us": iters * mem_iter * 1e6,
                  "def": "max(E1*6/F32, 10N'/HBM) + max(E>=2*6/F32, (I-1)*10N'/HBM), SURVEY.md 8(d)"},
    }


def _ncu_traffic(stage, P):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed
    ncu --set full capture (profiles/*/traffic.json), for the same image size."""
    for rnd in ("r02", "r01"):  # newest first
        f = os.path.join(ROOT, "profiles", rnd, "traffic.json")
        try:
            with open(f) as fh:
                d = json.load(fh)
        except Exception:
            continue
        e = d.get(stage, {}).get(str(P))
        if e is not None:
            return e
    return None


SMALL_PATH_PIXELS = 2 << 20  # capi.cu OCC_MAX_PIXELS: below it the histogram is K1 + the fused k_prep_small


def _hbm_stages(stage_ms, P, n_unique, peaks):
    """Achieved algorithmic GB/s of the HBM-bound stages."""
    out = {}
    if P < SMALL_PATH_PIXELS:
        # the small-image histogram (K1 + k_prep_small) spans the reset .. init_rank events
        ms = sum(stage_ms.get(st, 0.0) for st in ("reset", "hist_count", "bins_compact", "init_rank"))
        if ms > 0:
            r = _roofline("prep_small", ms, P, n_unique, 1, 0, peaks, 0)
            out["prep_small"] = {"achieved_gbs": round(r["achieved"], 1), "frac": round(r["frac"], 4),
                                 "algorithmic_bytes": r["algorithmic_bytes"], "ms": round(ms, 4), "note": r["note"]}
    for st in (("map_pixels",) if P < SMALL_PATH_PIXELS else ("hist_count", "bins_compact", "map_pixels")):
        if st in stage_ms and stage_ms[st] > 0:
            r = _roofline(st, stage_ms[st], P, n_unique, 1, 0, peaks, 0)
            out[st] = {"achieved_gbs": round(r["achieved"], 1), "frac": round(r["frac"], 4),
                       "algorithmic_bytes": r["algorithmic_bytes"], "ms": round(stage_ms[st], 4)}
    if "hist_count" in out:
        # K1's bound is the L2 atomic unit, not HBM: one RED pair (count add +
        # first-pixel max on one 8-B bin) per pixel run, counted here as one
        # per pixel (exact for uniform data), against the measured ceiling of
        # random RED pairs on a 32 MiB table slice (tools/microbench_mem.cu)
        ach = P / (stage_ms["hist_count"] * 1e-3)
        out["hist_count"]["l2_atomic_roofline"] = {
            "achieved_gpairs_s": round(ach / 1e9, 1), "peak_gpairs_s": RED_PAIRS_PEAK / 1e9,
            "frac": round(ach / RED_PAIRS_PEAK, 4),
            "peak_source": "measured: random RED.ADD+RED.MAX pairs over a 32 MiB slice, "
                           "profiles/r02/microbench_mem.txt"}
    return out


def run_batch(a, cfg, world, rank, local):
    """--config cfg5: one step = the batch of cfg.images independent images
    per rank (replicas), `lanes` images in flight per GPU (cqb_quantize_batch).
    value = aggregate Mpixel/s over all ranks; e2e adds the H2D copies of the
    batch (pinned) and the D2H of the index maps."""
    import torch
    import torch.distributed as dist

    from paper_1011_0093_b200 import _native as N
    from paper_1011_0093_b200 import api

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    ctx = N.context(local)
    stream = torch.cuda.Stream(device=dev)
    ctx.check(ctx.lib.cqb_set_stream(ctx.h, C.c_void_p(stream.cuda_stream)))
    n = cfg.images
    host = [torch.from_numpy(cfg.image(i + rank * n).reshape(-1)).pin_memory() for i in range(n)]
    imgs = [h.to(dev) for h in host]
    idx = [torch.empty(cfg.pixels, dtype=torch.uint8, device=dev) for _ in range(n)]
    idx_h = [torch.empty(cfg.pixels, dtype=torch.uint8).pin_memory() for _ in range(n)]
    term = api.Termination.convergent(EPSILON, HARD_CAP)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lanes = 4
    with torch.cuda.stream(stream):
        for _ in range(a.warmup):
            api.quantize_batch_device(imgs, a.k, term, INIT_SEED, lanes=lanes, index_out=idx)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = ClockSampler(local)
        clocks.start()
        tot = 0.0
        for _ in range(a.steps):
            flush_buf.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, reps = api.quantize_batch_device(imgs, a.k, term, INIT_SEED, lanes=lanes, index_out=idx)
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        clk = clocks.stop()
        # e2e: pinned host images -> device, batch, index maps -> host, all timed
        e2e = 0.0
        for _ in range(a.steps):
            flush_buf.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for h, d in zip(host, imgs):
                d.copy_(h, non_blocking=True)
            _, reps = api.quantize_batch_device(imgs, a.k, term, INIT_SEED, lanes=lanes, index_out=idx)
            for h, d in zip(idx_h, idx):
                h.copy_(d, non_blocking=True)
            torch.cuda.synchronize()
            e2e += time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([tot, e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot, e2e = float(t[0].item()), float(t[1].item())
    px = cfg.pixels * n * world * a.steps
    if rank == 0:
        line = {
            "metric": METRIC, "value": px / (tot * 1e-3) / 1e6, "unit": "Mpixel/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": tot / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {n} x {cfg.width}x{cfg.height} GMM-256 images per rank "
                                   f"(seeds 1000+i), K={a.k}, convergent(eps={EPSILON}, cap={HARD_CAP})",
                       "images_per_step_per_rank": n, "lanes": lanes, "parallelism": f"replicas x{world}",
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "iterations_first8": [r.iterations for r in reps[:8]]},
            "e2e": {"value": px / e2e / 1e6, "unit": "Mpixel/s", "h2d_bytes_per_step": 3 * cfg.pixels * n,
                    "d2h_bytes_per_step": cfg.pixels * n + n * (8 * 3 * a.k + 64),
                    "path": "pinned H2D of the batch + cqb_quantize_batch + D2H of the index maps, wall clock"},
            "gpu_launches": a.steps * n * int(reps[0].gpu_launches),
            "clocks": clk,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_sharded(a, cfg, world, rank, local):
    """BASELINE config 4 as the north star shards it: every rank holds the
    image and builds the histogram, the unique samples are split into `world`
    contiguous Morton ranges, and the per-iteration all-reduce of the K x 5
    exact moment sums runs INSIDE the persistent loop kernel over NVLink
    (cqb_quantize_sharded; no host round trip, no NCCL call per iteration).
    Each rank maps its own pixel range. Strong scaling: one image per step for
    the whole job. `--emulate-ranks W` (one GPU): the W ranks are block groups
    of the single launch — the same exchange code, to measure its overhead."""
    import torch
    import torch.distributed as dist

    from paper_1011_0093_b200 import _native as N
    from paper_1011_0093_b200 import api
    from paper_1011_0093_b200.distributed import PeerShardedQuantizer

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = N.context(local)
    lib = ctx.lib
    stream = torch.cuda.Stream(device=dev)
    ctx.check(lib.cqb_set_stream(ctx.h, C.c_void_p(stream.cuda_stream)))
    q = PeerShardedQuantizer(ctx=ctx, emulate=a.emulate_ranks if world == 1 else 0)
    img = cfg.image()
    P, k = cfg.pixels, a.k
    term = api.Termination.convergent(EPSILON, HARD_CAP)
    d_img = torch.from_numpy(img.reshape(-1)).to(dev)
    d_idx = torch.empty(P, dtype=torch.uint8, device=dev)
    d_out = torch.empty(3 * P, dtype=torch.uint8, device=dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    hist = a.hist or ("morton" if world > 1 else "replicated")
    rows = hist in ("rows", "morton")

    def one():
        if rows:  # histogram sharded too (pixel rows + all-to-all, or Morton ranges), then all-gathered
            return q.enqueue_rows(d_img, P, k, term, INIT_SEED, d_idx.data_ptr(), d_out.data_ptr(), split=hist)
        return q.enqueue(d_img.data_ptr(), P, k, term, INIT_SEED, d_idx.data_ptr(), d_out.data_ptr())

    def tmax(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with torch.cuda.stream(stream):
        for _ in range(a.warmup):
            flush_buf.fill_(1)
            one()
            q.fetch()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    with torch.cuda.stream(stream):
        for i in range(a.steps):
            flush_buf.fill_(1)
            evs[i][0].record(stream)
            one()
            evs[i][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = tmax(sum(x.elapsed_time(y) for x, y in evs))
    centers, rep, _ = q.fetch()
    launches = a.steps * int(rep.gpu_launches)
    evals = int(rep.dist_evals)
    if world > 1:
        t = torch.tensor([evals], device=dev, dtype=torch.int64)
        dist.all_reduce(t)
        evals = int(t.item())
    # stage attribution (loop kernel time) on a few profiled steps
    ctx.check(lib.cqb_set_profiling(ctx.h, 1))
    st = []
    with torch.cuda.stream(stream):
        for _ in range(3):
            flush_buf.fill_(1)
            one()
            q.fetch()
            ms = (C.c_float * 7)()
            ctx.check(lib.cqb_stage_times(ctx.h, ms, 7))
            st.append(list(ms))
            tl = np.zeros(8 * HARD_CAP, np.uint64)
            ctx.check(lib.cqb_loop_timeline(ctx.h, tl.ctypes.data_as(C.POINTER(C.c_uint64)), HARD_CAP))
    ctx.check(lib.cqb_set_profiling(ctx.h, 0))
    stage_ms = {n: float(v) for n, v in zip(N.STAGES, np.median(np.array(st), axis=0))}
    phases = _loop_phases(tl.reshape(HARD_CAP, 8).astype(np.int64), int(rep.iterations))
    # e2e: pinned host image in, this rank's slice of the index map + mapped raster out
    pin_img = torch.from_numpy(img.reshape(-1)).pin_memory()
    pin_idx = torch.empty(P, dtype=torch.uint8).pin_memory()
    pin_out = torch.empty(3 * P, dtype=torch.uint8).pin_memory()
    e2e = []
    bo = 0
    for i in range(a.warmup + a.steps):
        flush_buf.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            d_img.copy_(pin_img, non_blocking=True)
            lo, hi = one()
            pin_idx[lo:hi].copy_(d_idx[lo:hi], non_blocking=True)
            pin_out[3 * lo:3 * hi].copy_(d_out[3 * lo:3 * hi], non_blocking=True)
            c2, _, _ = q.fetch()
        stream.synchronize()
        if i >= a.warmup:
            e2e.append(time.perf_counter() - t0)
        bo = 4 * (hi - lo)
    e2e_s = tmax(sum(e2e))
    assert np.array_equal(c2, centers)
    ok = None
    if rank == 0 and world == 1 and a.emulate_ranks:  # the emulated ranks equal the one-rank path
        single = api.quantize(img, k, term, INIT_SEED, index_map=False, mapped=False, device=local)
        ok = bool(np.array_equal(single.palette, centers) and single.report.dist_evals == evals)
    if world > 1:
        dist.barrier()
    if rank == 0:
        peaks = _peaks()
        n_unique, iters = int(rep.n_unique), int(rep.iterations)
        value = P * a.steps / (total_ms * 1e-3) / 1e6
        ranks = world if world > 1 else max(a.emulate_ranks, 1)
        line = {
            "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload(cfg, k), "pixels": P, "n_unique": n_unique, "iterations": iters,
                       "k": k, "parallelism": (f"sample shards x{world}, in-kernel NVLink exchange" if world > 1 else
                                               f"sample shards x{ranks} emulated as block groups on one GPU"),
                       "histogram": {"rows": "pixel-row shards, Morton-range bin owners, NCCL all-to-all + all-gather",
                                     "morton": "Morton-range shards over every pixel, NCCL all-gather"}.get(
                                         hist, "replicated on every rank"),
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "timed": "per-step CUDA events on the library stream; value = P*steps / max-rank sum"},
            "e2e": {"value": P * a.steps / e2e_s / 1e6, "unit": "Mpixel/s", "h2d_bytes_per_step": 3 * P,
                    "d2h_bytes_per_step": bo, "path": "cqb_quantize_sharded, pinned host image in, own slice out"},
            "gpu_launches": launches,
            "roofline": _roofline("wsm_loop", stage_ms["wsm_loop"], P, n_unique, iters, k, peaks, evals),
            "stages_ms": {kk: round(v, 5) for kk, v in stage_ms.items()},
            "loop_phases_us": phases, "dist_evals": evals, "clocks": clk,
        }
        if ok is not None:
            line["matches_single_rank"] = ok
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    a = _args()
    world, rank, local = _dist()
    cfg = CONFIGS[a.config]
    if a.k is None:
        a.k = 256 if 256 in cfg.ks else cfg.ks[0]
    if a.impl == "reference":
        run_reference(a, cfg, world, rank)
        return
    if cfg.images > 1:
        run_batch(a, cfg, world, rank, local)
        return
    if a.shard or a.emulate_ranks > 0 or (cfg.name == "cfg4" and world > 1):
        run_sharded(a, cfg, world, rank, local)
        return
    run_ours(a, cfg, world, rank, local)


if __name__ == "__main__":
    main()
