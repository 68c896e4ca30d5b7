"""Python mirror of the reference colorq operator API for the WSM hot path.

Same names, argument meaning and error behaviour as the C++ functions in
/root/reference/proj/include/colorq (std::invalid_argument -> ValueError via
``CqbInvalidArgument``), each one a thin host call into the sm_100a CUDA
library through the C ABI (include/colorq_b200.h):

  build_histogram  histogram.hpp:65-108
  init/run_wsm     kmeans.hpp:394-404 (+ Termination :25-38)
  generate_palette methods.hpp:107-197, WSM / WSM-C branch :182-189
  map_pixels       image_ops.hpp:18-51 (+ an index-map variant)
  mse              metrics.hpp:18-29
  quantize         the CLI's quantize composition (tools/colorq.cpp:96-102)
                   fused into one device pass.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import CqbInvalidArgument, context

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Termination:
    """kmeans.hpp:25-38. mode 'fixed' (max_iters) or 'convergent' (epsilon, hard_cap)."""

    mode: str = "fixed"
    max_iters: int = 10
    epsilon: float = 1e-4
    hard_cap: int = 1000

    @staticmethod
    def fixed(iters: int) -> "Termination":
        return Termination("fixed", iters, 1e-4, 1000)

    @staticmethod
    def convergent(eps: float = 1e-4, cap: int = 1000) -> "Termination":
        if not eps > 0:
            raise ValueError("convergent termination requires epsilon > 0")
        return Termination("convergent", 10, eps, cap)

    def native(self) -> N.Termination:
        return N.Termination(1 if self.mode == "convergent" else 0, self.max_iters, self.epsilon, self.hard_cap)

    @property
    def iteration_budget(self) -> int:
        return self.hard_cap if self.mode == "convergent" else self.max_iters


@dataclass
class RunReport:
    """report.hpp:33-53 (+ device extras)."""

    method: str = ""
    k: int = 0
    seed: int = 0
    iterations: int = 0
    sse: float = math.nan
    mse: float = 0.0
    elapsed_ms: float = 0.0
    dist_evals: int = 0
    sse_history: list = field(default_factory=list)
    n_unique: int = 0
    map_ms: float = 0.0
    empty_events: int = 0
    gpu_launches: int = 0

    @staticmethod
    def csv_header() -> str:
        return "method,k,seed,iterations,sse,mse,elapsed_ms,dist_evals"

    def csv_row(self) -> str:
        g = lambda v: f"{v:.6g}"  # noqa: E731  fmt_g6, report.hpp:13-17
        return (f"{self.method},{self.k},{self.seed},{self.iterations},{g(self.sse)},{g(self.mse)},"
                f"{g(self.elapsed_ms)},{self.dist_evals}")


@dataclass
class ColorHistogram:
    """histogram.hpp:56-63, plus the packed keys and first-occurrence index."""

    keys: np.ndarray
    counts: np.ndarray
    weights: np.ndarray
    total_pixels: int
    first_index: np.ndarray | None = None

    @property
    def colors(self) -> np.ndarray:
        k = self.keys
        return np.stack([(k >> 16) & 255, (k >> 8) & 255, k & 255], axis=1).astype(np.float64)

    def size(self) -> int:
        return int(self.keys.shape[0])

    def __len__(self) -> int:
        return self.size()


@dataclass
class KmRunResult:
    palette: np.ndarray  # K x 3 float64
    report: RunReport
    trajectory: np.ndarray | None = None
    labels: np.ndarray | None = None


@dataclass
class QuantizeOutcome:
    palette: np.ndarray
    report: RunReport
    index_map: np.ndarray | None = None
    mapped: np.ndarray | None = None
    error: np.ndarray | None = None


@dataclass(frozen=True)
class MethodParams:
    """methods.hpp:71-85 (the WSM-relevant knobs)."""

    id: str = "wsm"  # "wsm" / "km" / "fkm" (fixed iters) or "wsm-c" / "km-c" / "fkm-c" (convergent)
    iters: int = 10
    epsilon: float = 1e-4
    hard_cap: int = 1000
    k_prime: int = 8  # fkm neighbour count (methods.hpp:75)

    def termination(self) -> Termination:
        if self.id in ("wsm-c", "km-c", "fkm-c"):
            return Termination.convergent(self.epsilon, self.hard_cap)
        return Termination.fixed(self.iters)


class UnknownMethodError(ValueError):
    """methods.hpp:25-27."""


def _rgb(img: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.uint8)
    if a.ndim < 2 or a.shape[-1] != 3:
        raise ValueError("expected an (..., 3) uint8 RGB array")
    return a


def _report_from(rep: N.Report, method: str, hist: np.ndarray) -> RunReport:
    return RunReport(method=method, k=rep.k, seed=int(rep.seed), iterations=rep.iterations, sse=rep.sse,
                     mse=rep.mse, elapsed_ms=rep.elapsed_ms, dist_evals=int(rep.dist_evals),
                     sse_history=list(hist[: rep.iterations]), n_unique=int(rep.n_unique), map_ms=rep.map_ms,
                     empty_events=rep.empty_events, gpu_launches=rep.gpu_launches)


# ---------------------------------------------------------------------------
def build_histogram(img: np.ndarray, device: int = 0) -> ColorHistogram:
    """Unique colors in first-occurrence order with counts and weights."""
    a = _rgb(img)
    n = a.size // 3
    if n == 0:
        raise CqbInvalidArgument(N.CQB_ERR_INVALID_ARGUMENT, "build_histogram: empty image")
    ctx = context(device)
    keys = np.empty(n, np.uint32)
    counts = np.empty(n, np.uint32)
    weights = np.empty(n, np.float64)
    first = np.empty(n, np.uint32)
    nu = C.c_uint64()
    ctx.check(ctx.lib.cqb_build_histogram(ctx.h, _p(a, _u8p), n, _p(keys, _u32p), _p(counts, _u32p),
                                          _p(weights, _f64p), _p(first, _u32p), n, C.byref(nu)))
    m = nu.value
    return ColorHistogram(keys[:m].copy(), counts[:m].copy(), weights[:m].copy(), n, first[:m].copy())


def _hist_arrays(hist: ColorHistogram):
    keys = np.ascontiguousarray(hist.keys, np.uint32)
    counts = np.ascontiguousarray(hist.counts, np.uint32)
    return keys, counts


def run_wsm(hist: ColorHistogram, k: int, term: Termination, seed: int, trajectory: bool = False,
            labels: bool = False, device: int = 0) -> KmRunResult:
    """init_centers + sort-means loop over a histogram (kmeans.hpp:394-404)."""
    ctx = context(device)
    keys, counts = _hist_arrays(hist)
    n = keys.shape[0]
    cap = term.iteration_budget
    centers = np.zeros(3 * max(k, 1))
    hist_out = np.zeros(cap)
    traj = np.zeros((cap, max(k, 1), 3)) if trajectory else None
    lab = np.zeros(n, np.uint8) if labels else None
    rep = N.Report()
    t = term.native()
    ctx.check(ctx.lib.cqb_run_wsm(ctx.h, _p(keys, _u32p), _p(counts, _u32p), n, hist.total_pixels, k, C.byref(t),
                                  seed, _p(centers, _f64p), _p(hist_out, _f64p), cap, _p(traj, _f64p),
                                  cap if trajectory else 0, _p(lab, _u8p), C.byref(rep)))
    r = _report_from(rep, "wsm-c" if term.mode == "convergent" else "wsm", hist_out)
    return KmRunResult(centers.reshape(-1, 3)[:k].copy(), r,
                       traj[: rep.iterations].copy() if traj is not None else None, lab)


def wsm_iterate(hist: ColorHistogram, centers: np.ndarray, labels: np.ndarray, term: Termination,
                dense_first: bool = False, device: int = 0):
    """Teacher-forced iterations of the device loop from given centers/labels.
    Returns (next_centers, labels, report)."""
    ctx = context(device)
    keys, counts = _hist_arrays(hist)
    n = keys.shape[0]
    Cin = np.ascontiguousarray(centers, np.float64).reshape(-1)
    k = Cin.shape[0] // 3
    lab = np.ascontiguousarray(labels, np.uint8).copy()
    cap = term.iteration_budget
    out = np.zeros(3 * k)
    h = np.zeros(cap)
    rep = N.Report()
    t = term.native()
    ctx.check(ctx.lib.cqb_wsm_iterate(ctx.h, _p(keys, _u32p), _p(counts, _u32p), n, hist.total_pixels, k,
                                      _p(Cin, _f64p), _p(lab, _u8p), int(dense_first), C.byref(t), _p(out, _f64p),
                                      _p(h, _f64p), cap, C.byref(rep)))
    return out.reshape(k, 3), lab, _report_from(rep, "wsm", h)


def quantize(img: np.ndarray, k: int, term: Termination | None = None, seed: int = 1, index_map: bool = True,
             mapped: bool = True, device: int = 0, out_index: np.ndarray | None = None,
             out_mapped: np.ndarray | None = None, error: bool = False) -> QuantizeOutcome:
    """Histogram + WSM + map + MSE in one device pass (host buffers).
    ``out_index`` / ``out_mapped`` may be caller-owned (e.g. pinned) arrays.
    ``error=True`` also returns error_image(img, mapped) (image_ops.hpp:55-71)
    in ``QuantizeOutcome.error``, fused into the map pass."""
    a = _rgb(img)
    if a.ndim == 3:
        h, w = a.shape[0], a.shape[1]
    else:
        h, w = a.size // 3, 1
    term = term or Termination.convergent()
    ctx = context(device)
    cap = term.iteration_budget
    centers = np.zeros(3 * max(k, 1))
    hist_out = np.zeros(cap)
    idx = out_index if out_index is not None else (np.empty(a.shape[:-1], np.uint8) if index_map else None)
    out = out_mapped if out_mapped is not None else (np.empty_like(a) if mapped else None)
    if idx is not None:
        assert idx.flags.c_contiguous and idx.dtype == np.uint8 and idx.size == a.size // 3
    if out is not None:
        assert out.flags.c_contiguous and out.dtype == np.uint8 and out.size == a.size
    err = np.empty_like(a) if error else None
    rep = N.Report()
    t = term.native()
    ctx.check(ctx.lib.cqb_quantize_ex(ctx.h, _p(a, _u8p), w, h, k, C.byref(t), seed, _p(centers, _f64p),
                                      _p(hist_out, _f64p), cap, _p(idx, _u8p), _p(out, _u8p), _p(err, _u8p),
                                      C.byref(rep)))
    r = _report_from(rep, "wsm-c" if term.mode == "convergent" else "wsm", hist_out)
    return QuantizeOutcome(centers.reshape(-1, 3)[:k].copy(), r, idx, out, err)


def quantize_batch_device(images, k: int, term: Termination | None = None, seed: int = 1, lanes: int = 4,
                          index_out=None, mapped_out=None, device: int = 0):
    """Config 5: quantize independent DEVICE-resident images (CUDA tensors
    of u8x3 pixels, or (device_pointer, n_pixels) pairs) with ``lanes``
    images in flight on one GPU (cqb_quantize_batch). ``index_out`` /
    ``mapped_out``: optional lists of device tensors (16-B aligned).
    Returns (palettes [n, k, 3] float64, [RunReport])."""
    n = len(images)
    term = term or Termination.convergent()
    ctx = context(device)

    def ptr(x):
        return int(x[0]) if isinstance(x, tuple) else int(x.data_ptr())

    def npx(x):
        return int(x[1]) if isinstance(x, tuple) else int(x.numel()) // 3

    ptrs = (C.c_void_p * max(n, 1))(*[ptr(x) for x in images])
    pix = np.array([npx(x) for x in images] or [0], np.uint64)
    outs = []
    for lst in (index_out, mapped_out):
        outs.append(None if lst is None else (C.c_void_p * max(n, 1))(*[None if o is None else int(o.data_ptr())
                                                                          for o in lst]))
    centers = np.zeros(max(n, 1) * 3 * max(k, 1))
    reps = (N.Report * max(n, 1))()
    t = term.native()
    ctx.check(ctx.lib.cqb_quantize_batch(ctx.h, n, ptrs, _p(pix, _u64p), k, C.byref(t), seed, outs[0], outs[1],
                                         lanes, _p(centers, _f64p), reps))
    name = "wsm-c" if term.mode == "convergent" else "wsm"
    return (centers[: n * 3 * k].reshape(n, k, 3).copy(),
            [_report_from(reps[i], name, np.zeros(0)) for i in range(n)])


# --------------------------------------------------------------------------- point sets
# kmeans.hpp's span<const Vec3> API (init_centers, assign_sort_means /
# assign_naive, update_centers, weighted_sse, run_wsm_points) on the device
# point-set kernels (points.cuh), k <= 1024.
_i32p = C.POINTER(C.c_int32)


def _pts(points, weights=None):
    X = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    W = None if weights is None else np.ascontiguousarray(weights, np.float64).reshape(-1)
    if W is not None and W.shape[0] != X.shape[0]:
        raise CqbInvalidArgument(N.CQB_ERR_INVALID_ARGUMENT, "points and weights differ in length")
    return X, W


def init_centers(points, k: int, seed: int, device: int = 0) -> np.ndarray:
    """kmeans.hpp:53-74: k distinct points by the seeded partial Fisher-Yates."""
    X, _ = _pts(points)
    ctx = context(device)
    chosen = np.zeros(max(k, 1), np.uint32)
    ctx.check(ctx.lib.cqb_init_centers(ctx.h, X.shape[0], k, seed, _p(chosen, _u32p)))
    return X[chosen[:k]].copy()


def assign_points(points, weights, centers, memberships=None, naive: bool = False, device: int = 0):
    """assign_sort_means from `memberships` (kmeans.hpp:201-239), or
    assign_naive (:83-106). Returns (memberships, weighted_sse, dist_evals)."""
    X, W = _pts(points, weights)
    Cc = np.ascontiguousarray(centers, np.float64).reshape(-1)
    m = np.zeros(X.shape[0], np.int32) if memberships is None else np.ascontiguousarray(memberships, np.int32).copy()
    sse, ev = np.zeros(1), np.zeros(1, np.uint64)
    ctx = context(device)
    ctx.check(ctx.lib.cqb_points_assign(ctx.h, _p(X, _f64p), _p(W, _f64p), X.shape[0], _p(Cc, _f64p), Cc.size // 3,
                                        None, None, int(naive), _p(m, _i32p), _p(sse, _f64p), _p(ev, _u64p), None,
                                        None))
    return m, float(sse[0]), int(ev[0])


def update_centers(points, weights, memberships, prev, device: int = 0) -> np.ndarray:
    """kmeans.hpp:245-302 (empty clusters re-seeded)."""
    X, W = _pts(points, weights)
    m = np.ascontiguousarray(memberships, np.int32)
    P = np.ascontiguousarray(prev, np.float64).reshape(-1)
    out = np.zeros_like(P)
    ctx = context(device)
    ctx.check(ctx.lib.cqb_points_update(ctx.h, _p(X, _f64p), _p(W, _f64p), X.shape[0], _p(m, _i32p), _p(P, _f64p),
                                        P.size // 3, _p(out, _f64p)))
    return out.reshape(-1, 3)


def weighted_sse(points, weights, centers, memberships, device: int = 0) -> float:
    """kmeans.hpp:306-317."""
    X, W = _pts(points, weights)
    Cc = np.ascontiguousarray(centers, np.float64).reshape(-1)
    m = np.ascontiguousarray(memberships, np.int32)
    out = np.zeros(1)
    ctx = context(device)
    ctx.check(ctx.lib.cqb_points_sse(ctx.h, _p(X, _f64p), _p(W, _f64p), X.shape[0], _p(Cc, _f64p), Cc.size // 3,
                                     _p(m, _i32p), _p(out, _f64p)))
    return float(out[0])


def run_wsm_points(points, weights, k: int, term: Termination | None = None, seed: int = 1, trajectory: bool = False,
                   device: int = 0) -> KmRunResult:
    """kmeans.hpp:379-390: Weighted Sort-Means over an arbitrary weighted point set."""
    X, W = _pts(points, weights)
    term = term or Termination.convergent()
    cap = term.iteration_budget
    centers = np.zeros(3 * max(k, 1))
    hist = np.zeros(cap)
    traj = np.zeros((cap, max(k, 1), 3)) if trajectory else None
    m = np.zeros(X.shape[0], np.int32)
    rep = N.Report()
    t = term.native()
    ctx = context(device)
    ctx.check(ctx.lib.cqb_run_wsm_points(ctx.h, _p(X, _f64p), _p(W, _f64p), X.shape[0], k, C.byref(t), seed,
                                         _p(centers, _f64p), _p(hist, _f64p), cap, _p(traj, _f64p),
                                         cap if trajectory else 0, _p(m, _i32p), C.byref(rep)))
    r = _report_from(rep, "wsm-c" if term.mode == "convergent" else "wsm", hist)
    return KmRunResult(centers.reshape(-1, 3)[:k].copy(), r, traj[: rep.iterations].copy() if trajectory else None, m)


def generate_palette(img: np.ndarray, mp: MethodParams, k: int, seed: int, device: int = 0) -> QuantizeOutcome:
    """methods.hpp:107-197 — the WSM / WSM-C branch only (the comparator
    quantizers are outside this framework's scope)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    if mp.id in ("km", "km-c"):  # methods.hpp:155-160
        q = run_km_full(img, k, mp.termination(), seed, device=device)
        q.report.method = mp.id
        return q
    if mp.id in ("fkm", "fkm-c"):  # methods.hpp:163-178 (row f4)
        q = run_fkm(img, k, mp.k_prime, mp.termination(), seed, device=device)
        q.report.method = mp.id
        return q
    if mp.id not in ("wsm", "wsm-c"):
        raise UnknownMethodError(f"method '{mp.id}' is not provided by the B200 WSM path")
    q = quantize(img, k, mp.termination(), seed, index_map=False, mapped=False, device=device)
    q.report.method = mp.id
    q.report.mse = 0.0  # the caller fills mse (methods.hpp:104-106)
    return q


def error_image(original: np.ndarray, quantized: np.ndarray, device: int = 0) -> np.ndarray:
    """image_ops.hpp:55-71: per channel 255 - min(255, 4|o - q|) (device kernel)."""
    a, b = _rgb(original), _rgb(quantized)
    if a.shape != b.shape:
        raise CqbInvalidArgument(N.CQB_ERR_INVALID_ARGUMENT, "error_image: dimension mismatch")
    out = np.empty_like(a)
    ctx = context(device)
    ctx.check(ctx.lib.cqb_error_image(ctx.h, _p(a, _u8p), _p(b, _u8p), a.size // 3, _p(out, _u8p)))
    return out


def run_km_full(img: np.ndarray, k: int, term: Termination | None = None, seed: int = 1,
                device: int = 0) -> QuantizeOutcome:
    """Conventional k-means over every pixel (kmeans.hpp:409-426): KM / KM-C."""
    a = _rgb(img)
    if a.ndim != 3:
        raise CqbInvalidArgument(N.CQB_ERR_INVALID_ARGUMENT, "run_km_full: expects an H x W x 3 image")
    h, w = a.shape[0], a.shape[1]
    term = term or Termination.convergent()
    ctx = context(device)
    cap = term.iteration_budget
    centers = np.zeros(3 * max(k, 1))
    hist_out = np.zeros(cap)
    rep = N.Report()
    t = term.native()
    ctx.check(ctx.lib.cqb_run_km_full(ctx.h, _p(a, _u8p), w, h, k, C.byref(t), seed, _p(centers, _f64p),
                                      _p(hist_out, _f64p), cap, C.byref(rep)))
    r = _report_from(rep, "km-c" if term.mode == "convergent" else "km", hist_out)
    return QuantizeOutcome(centers.reshape(-1, 3)[:k].copy(), r)


def run_fkm(img: np.ndarray, k: int, k_prime: int = 8, term: Termination | None = None, seed: int = 1,
            device: int = 0) -> QuantizeOutcome:
    """Finite-state k-means over every pixel (fast_variants.hpp:20-81): FKM / FKM-C."""
    a = _rgb(img)
    if a.ndim != 3:
        raise CqbInvalidArgument(N.CQB_ERR_INVALID_ARGUMENT, "run_fkm: expects an H x W x 3 image")
    h, w = a.shape[0], a.shape[1]
    term = term or Termination.convergent()
    ctx = context(device)
    cap = term.iteration_budget
    centers = np.zeros(3 * max(k, 1))
    hist_out = np.zeros(cap)
    rep = N.Report()
    t = term.native()
    ctx.check(ctx.lib.cqb_run_fkm(ctx.h, _p(a, _u8p), w, h, k, k_prime, C.byref(t), seed, _p(centers, _f64p),
                                  _p(hist_out, _f64p), cap, C.byref(rep)))
    r = _report_from(rep, "fkm-c" if term.mode == "convergent" else "fkm", hist_out)
    return QuantizeOutcome(centers.reshape(-1, 3)[:k].copy(), r)


def map_pixels_indexed(img: np.ndarray, palette: np.ndarray, device: int = 0):
    """map_pixels + the u8 index map + the squared-error sum."""
    a = _rgb(img)
    P = np.ascontiguousarray(palette, np.float64).reshape(-1)
    k = P.shape[0] // 3
    if k < 1:
        raise CqbInvalidArgument(N.CQB_ERR_INVALID_ARGUMENT, "map_pixels: empty palette")
    ctx = context(device)
    n = a.size // 3
    out = np.empty_like(a)
    idx = np.empty(a.shape[:-1], np.uint8)
    err = C.c_uint64()
    ctx.check(ctx.lib.cqb_map_pixels(ctx.h, _p(a, _u8p), n, _p(P, _f64p), k, _p(out, _u8p), _p(idx, _u8p),
                                     C.byref(err)))
    return out, idx, int(err.value)


def map_pixels(img: np.ndarray, palette: np.ndarray, device: int = 0) -> np.ndarray:
    """image_ops.hpp:18-51."""
    return map_pixels_indexed(img, palette, device)[0]


def mse(a: np.ndarray, b: np.ndarray, device: int = 0) -> float:
    """metrics.hpp:18-29."""
    x = _rgb(a)
    y = _rgb(b)
    if x.shape != y.shape:
        raise ValueError("mse: dimension mismatch")
    ctx = context(device)
    out = C.c_double()
    ctx.check(ctx.lib.cqb_mse(ctx.h, _p(x, _u8p), _p(y, _u8p), x.size // 3, C.byref(out)))
    return out.value


def psnr(mse_value: float) -> float:
    """metrics.hpp:32-36 (host scalar formula)."""
    if mse_value < 0:
        raise ValueError("psnr: negative MSE")
    if mse_value == 0:
        return math.inf
    return 20.0 * math.log10(255.0 / math.sqrt(mse_value))
