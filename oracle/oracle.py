"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the two CPU checkers.

* ``Oracle("port")``      -> oracle/build/liboracle.so, the plain-C restatement
  (oracle/wsm_oracle.c) of the reference algorithm, each function citing the
  reference file:line it follows.
* ``Oracle("reference")`` -> oracle/_ref/libcolorq_ref.so, the reference's own
  headers compiled unchanged (oracle/ref_capi.cpp + oracle/Makefile).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package
``paper_1011_0093_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libcolorq_ref.so")

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def build() -> None:
    """Compile the checkers (make -f oracle/Makefile)."""
    import subprocess

    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def available(kind: str) -> bool:
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)


@dataclass
class WsmResult:
    centers: np.ndarray
    iterations: int
    sse: float
    dist_evals: int
    sse_history: np.ndarray
    trajectory: np.ndarray | None = None
    labels: np.ndarray | None = None
    label_trajectory: np.ndarray | None = None


@dataclass
class Histogram:
    keys: np.ndarray
    counts: np.ndarray
    weights: np.ndarray
    total_pixels: int = 0

    @property
    def colors(self) -> np.ndarray:
        k = self.keys
        return np.stack([(k >> 16) & 255, (k >> 8) & 255, k & 255], axis=1).astype(np.float64)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -f oracle/Makefile)")
        self.lib = C.CDLL(path)
        L = self.lib
        pre = "orc_" if kind == "port" else "ref_"
        self._f = lambda name: getattr(L, pre + name)
        f = self._f
        f("mt64_stream").argtypes = [C.c_uint64, _u64p, C.c_int]
        if kind == "port":
            f("build_histogram").argtypes = [_u8p, C.c_uint64, _u32p, _u32p, _f64p]
            f("build_histogram").restype = C.c_int64
            f("run_wsm").argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.c_uint64, _f64p, _f64p, _u64p, _f64p, C.c_int,
                                     _f64p, C.c_int, _i32p, _i32p]
            f("map_pixels").argtypes = [_u8p, C.c_uint64, _f64p, C.c_int, _u8p, _u8p]
            f("center_tables").argtypes = [_f64p, C.c_int, _f64p, _i32p]
            f("assign_sort_means").argtypes = [_f64p, _f64p, C.c_uint64, _f64p, C.c_int, _f64p, _i32p, _i32p,
                                               _f64p, _u64p]
            f("assign_naive").argtypes = [_f64p, C.c_uint64, _f64p, C.c_int, _i32p]
            f("update_centers").argtypes = [_f64p, _f64p, C.c_uint64, _i32p, _f64p, C.c_int, _f64p]
            f("update_centers").restype = C.c_int
            f("init_centers").argtypes = [_f64p, C.c_uint64, C.c_int, C.c_uint64, _f64p, _u32p]
            f("pair_evals").argtypes = [_f64p, _f64p, C.c_int, C.c_int]
            f("pair_evals").restype = C.c_uint64
        else:
            f("build_histogram").argtypes = [_u8p, C.c_uint64, _u32p, _u32p, _f64p, C.c_uint64, C.c_uint64]
            f("build_histogram").restype = C.c_int64
            f("run_wsm").argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.c_uint64, _f64p, _f64p, _u64p, _f64p, C.c_int,
                                     _f64p, C.c_int]
            f("map_pixels").argtypes = [_u8p, C.c_uint64, _f64p, C.c_int, _u8p]
            f("sort_means_step").argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, _f64p, C.c_int, _i32p, _f64p,
                                             _u64p, _f64p, _i32p]
            f("update_centers").argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, _i32p, _f64p, C.c_int, _f64p]
            f("init_centers").argtypes = [_u32p, C.c_uint64, C.c_int, C.c_uint64, _f64p]
            f("next_prime").argtypes = [C.c_uint64]
            f("next_prime").restype = C.c_uint64
            f("universal_hash").argtypes = [C.c_uint8] * 3 + [C.c_uint64] * 4
            f("universal_hash").restype = C.c_uint64
            f("quantize").argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                      C.c_uint64, _f64p, _i32p, _f64p, _u64p, _u8p, _f64p, _f64p, _f64p]
            f("quantize_many").argtypes = [C.POINTER(_u8p), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_double, C.c_int, C.c_uint64, C.c_int, _f64p, _i32p]
            f("quantize_many").restype = C.c_double
            f("init_centers_points").argtypes = [_f64p, C.c_uint64, C.c_int, C.c_uint64, _f64p]
            f("points_assign").argtypes = [_f64p, _f64p, C.c_uint64, _f64p, C.c_int, C.c_int, _i32p, _f64p, _u64p,
                                           _u64p]
            f("points_update").argtypes = [_f64p, _f64p, C.c_uint64, _i32p, _f64p, C.c_int, _f64p]
            f("points_sse").argtypes = [_f64p, _f64p, C.c_uint64, _f64p, C.c_int, _i32p]
            f("points_sse").restype = C.c_double
            f("run_wsm_points").argtypes = [_f64p, _f64p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                            C.c_uint64, _f64p, _f64p, _u64p, _f64p, C.c_int]
            f("write_ppm").argtypes = [_u8p, C.c_int, C.c_int, _u8p, C.c_int64]
            f("write_ppm").restype = C.c_int64
            f("read_ppm").argtypes = [_u8p, C.c_int64, _u8p, C.c_int64, _i32p, _i32p]
            f("palette_text").argtypes = [_f64p, C.c_int, C.c_char_p, C.c_int64]
            f("palette_text").restype = C.c_int64
            f("error_image").argtypes = [_u8p, _u8p, C.c_uint64, _u8p]
            f("run_bench").argtypes = [C.c_char_p, C.c_char_p]
            f("run_fkm").argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                     C.c_uint64, _f64p, _f64p, _u64p, _f64p, C.c_int]
            f("run_km_full").argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                         C.c_uint64, _f64p, _f64p, _u64p, _f64p, C.c_int]
        f("mse").argtypes = [_u8p, _u8p, C.c_uint64]
        f("mse").restype = C.c_double

    # -- generator ---------------------------------------------------------
    def mt64_stream(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._f("mt64_stream")(seed, _p(out, _u64p), n)
        return out

    # -- histogram ---------------------------------------------------------
    def build_histogram(self, rgb: np.ndarray, hash_expected: int = 0, hash_seed: int = 0) -> Histogram:
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8).reshape(-1, 3)
        n = rgb.shape[0]
        keys = np.zeros(max(n, 1), np.uint32)
        counts = np.zeros(max(n, 1), np.uint32)
        weights = np.zeros(max(n, 1), np.float64)
        if self.kind == "port":
            nu = self._f("build_histogram")(_p(rgb, _u8p), n, _p(keys, _u32p), _p(counts, _u32p),
                                            _p(weights, _f64p))
        else:
            nu = self._f("build_histogram")(_p(rgb, _u8p), n, _p(keys, _u32p), _p(counts, _u32p),
                                            _p(weights, _f64p), hash_expected, hash_seed)
        if nu < 0:
            raise ValueError("build_histogram: empty image")
        return Histogram(keys[:nu].copy(), counts[:nu].copy(), weights[:nu].copy(), n)

    # -- clustering --------------------------------------------------------
    def run_wsm(self, keys, counts, total: int, k: int, mode: int = 1, max_iters: int = 10, eps: float = 1e-4,
                cap: int = 100, seed: int = 1, trajectory: bool = False, labels: bool = False) -> WsmResult:
        keys = np.ascontiguousarray(keys, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        n = keys.shape[0]
        hcap = max(cap if mode == 1 else max_iters, 1)
        C_out = np.zeros(3 * k, np.float64)
        sse = np.zeros(1, np.float64)
        ev = np.zeros(1, np.uint64)
        hist = np.full(hcap, np.nan)
        traj = np.zeros((hcap, k, 3), np.float64) if trajectory else None
        ltraj = np.zeros((hcap, n), np.int32) if (labels and self.kind == "port") else None
        lab = np.zeros(n, np.int32) if (labels and self.kind == "port") else None
        args = [_p(keys, _u32p), _p(counts, _u32p), n, total, k, mode, max_iters, eps, cap, seed,
                _p(C_out, _f64p), _p(sse, _f64p), _p(ev, _u64p), _p(hist, _f64p), hcap,
                _p(traj, _f64p), hcap if trajectory else 0]
        if self.kind == "port":
            args += [_p(ltraj, _i32p), _p(lab, _i32p)]
        it = self._f("run_wsm")(*args)
        if it < 0:
            raise ValueError("run_wsm: invalid argument (k < 1 or k > N')")
        return WsmResult(C_out.reshape(k, 3), it, float(sse[0]), int(ev[0]), hist[:it].copy(),
                         traj[:it].copy() if traj is not None else None, lab,
                         ltraj[:it].copy() if ltraj is not None else None)

    def init_centers(self, keys, k: int, seed: int) -> np.ndarray:
        keys = np.ascontiguousarray(keys, np.uint32)
        C_out = np.zeros(3 * k, np.float64)
        if self.kind == "port":
            X = Histogram(keys, keys, keys).colors.copy()
            rc = self._f("init_centers")(_p(X, _f64p), keys.shape[0], k, seed, _p(C_out, _f64p), None)
        else:
            rc = self._f("init_centers")(_p(keys, _u32p), keys.shape[0], k, seed, _p(C_out, _f64p))
        if rc != 0:
            raise ValueError("init_centers: invalid k")
        return C_out.reshape(k, 3)

    def sort_means_step(self, keys, counts, total, centers, labels):
        """One fresh update_center_tables + assign_sort_means (reference only)."""
        assert self.kind == "reference"
        keys = np.ascontiguousarray(keys, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        C_in = np.ascontiguousarray(centers, np.float64).reshape(-1)
        k = C_in.shape[0] // 3
        lab = np.ascontiguousarray(labels, np.int32).copy()
        sse = np.zeros(1)
        ev = np.zeros(1, np.uint64)
        D = np.zeros(k * k)
        order = np.zeros(k * k, np.int32)
        self._f("sort_means_step")(_p(keys, _u32p), _p(counts, _u32p), keys.shape[0], total, _p(C_in, _f64p), k,
                                   _p(lab, _i32p), _p(sse, _f64p), _p(ev, _u64p), _p(D, _f64p),
                                   _p(order, _i32p))
        return lab, float(sse[0]), int(ev[0]), D.reshape(k, k), order.reshape(k, k)

    def update_centers(self, keys, counts, total, labels, prev):
        keys = np.ascontiguousarray(keys, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        lab = np.ascontiguousarray(labels, np.int32)
        P = np.ascontiguousarray(prev, np.float64).reshape(-1)
        k = P.shape[0] // 3
        out = np.zeros(3 * k)
        if self.kind == "port":
            X = Histogram(keys, counts, counts).colors.copy()
            W = counts.astype(np.float64) * (1.0 / float(total))
            self._f("update_centers")(_p(X, _f64p), _p(W, _f64p), keys.shape[0], _p(lab, _i32p), _p(P, _f64p), k,
                                      _p(out, _f64p))
        else:
            self._f("update_centers")(_p(keys, _u32p), _p(counts, _u32p), keys.shape[0], total, _p(lab, _i32p),
                                      _p(P, _f64p), k, _p(out, _f64p))
        return out.reshape(k, 3)

    # -- the point-set API (reference only) --------------------------------
    def init_centers_points(self, X, k: int, seed: int) -> np.ndarray:
        X = np.ascontiguousarray(X, np.float64)
        C_out = np.zeros(3 * k)
        if self._f("init_centers_points")(_p(X, _f64p), X.shape[0], k, seed, _p(C_out, _f64p)) != 0:
            raise ValueError("init_centers: invalid k")
        return C_out.reshape(k, 3)

    def points_assign(self, X, W, centers, memberships, naive: bool = False):
        X = np.ascontiguousarray(X, np.float64)
        W = np.ascontiguousarray(W, np.float64)
        Cc = np.ascontiguousarray(centers, np.float64).reshape(-1)
        m = np.ascontiguousarray(memberships, np.int32).copy()
        sse, ev, au = np.zeros(1), np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        rc = self._f("points_assign")(_p(X, _f64p), _p(W, _f64p), X.shape[0], _p(Cc, _f64p), Cc.shape[0] // 3,
                                      int(naive), _p(m, _i32p), _p(sse, _f64p), _p(ev, _u64p), _p(au, _u64p))
        if rc != 0:
            raise ValueError("assign: state does not match inputs")
        return m, float(sse[0]), int(ev[0]), int(au[0])

    def points_update(self, X, W, memberships, prev):
        X = np.ascontiguousarray(X, np.float64)
        W = np.ascontiguousarray(W, np.float64)
        m = np.ascontiguousarray(memberships, np.int32)
        P = np.ascontiguousarray(prev, np.float64).reshape(-1)
        out = np.zeros_like(P)
        self._f("points_update")(_p(X, _f64p), _p(W, _f64p), X.shape[0], _p(m, _i32p), _p(P, _f64p), P.shape[0] // 3,
                                 _p(out, _f64p))
        return out.reshape(-1, 3)

    def points_sse(self, X, W, centers, memberships) -> float:
        X = np.ascontiguousarray(X, np.float64)
        W = np.ascontiguousarray(W, np.float64)
        Cc = np.ascontiguousarray(centers, np.float64).reshape(-1)
        m = np.ascontiguousarray(memberships, np.int32)
        return float(self._f("points_sse")(_p(X, _f64p), _p(W, _f64p), X.shape[0], _p(Cc, _f64p), Cc.shape[0] // 3,
                                           _p(m, _i32p)))

    def run_wsm_points(self, X, W, k: int, mode: int = 1, max_iters: int = 10, eps: float = 1e-4, cap: int = 100,
                       seed: int = 1) -> WsmResult:
        X = np.ascontiguousarray(X, np.float64)
        W = np.ascontiguousarray(W, np.float64)
        hcap = max(cap if mode == 1 else max_iters, 1)
        C_out, sse, ev, hist = np.zeros(3 * k), np.zeros(1), np.zeros(1, np.uint64), np.full(hcap, np.nan)
        it = self._f("run_wsm_points")(_p(X, _f64p), _p(W, _f64p), X.shape[0], k, mode, max_iters, eps, cap, seed,
                                       _p(C_out, _f64p), _p(sse, _f64p), _p(ev, _u64p), _p(hist, _f64p), hcap)
        if it < 0:
            raise ValueError("run_wsm_points: invalid argument")
        return WsmResult(C_out.reshape(k, 3), it, float(sse[0]), int(ev[0]), hist[:it].copy())

    # -- post-processing ---------------------------------------------------
    def map_pixels(self, rgb: np.ndarray, centers: np.ndarray):
        shape = rgb.shape
        rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1, 3)
        C_in = np.ascontiguousarray(centers, np.float64).reshape(-1)
        k = C_in.shape[0] // 3
        out = np.zeros_like(rgb)
        idx = np.zeros(rgb.shape[0], np.uint8)
        if self.kind == "port":
            rc = self._f("map_pixels")(_p(rgb, _u8p), rgb.shape[0], _p(C_in, _f64p), k, _p(out, _u8p), _p(idx, _u8p))
        else:
            rc = self._f("map_pixels")(_p(rgb, _u8p), rgb.shape[0], _p(C_in, _f64p), k, _p(out, _u8p))
            idx = None
        if rc != 0:
            raise ValueError("map_pixels: empty palette")
        return out.reshape(shape), (idx.reshape(shape[:-1]) if idx is not None else None)

    def mse(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        if a.shape != b.shape:
            raise ValueError("mse: dimension mismatch")
        return float(self._f("mse")(_p(a, _u8p), _p(b, _u8p), a.size // 3))

    # -- whole path (reference only): generate_palette WSM + map + mse -----
    def quantize(self, img: np.ndarray, k: int, mode: int = 1, max_iters: int = 10, eps: float = 1e-4,
                 cap: int = 100, seed: int = 1):
        assert self.kind == "reference"
        h, w = img.shape[:2]
        img = np.ascontiguousarray(img, np.uint8)
        C_out = np.zeros(3 * k)
        it = np.zeros(1, np.int32)
        sse = np.zeros(1)
        ev = np.zeros(1, np.uint64)
        out = np.zeros_like(img)
        m = np.zeros(1)
        pms = np.zeros(1)
        mms = np.zeros(1)
        rc = self._f("quantize")(_p(img, _u8p), w, h, k, mode, max_iters, eps, cap, seed, _p(C_out, _f64p),
                                 _p(it, _i32p), _p(sse, _f64p), _p(ev, _u64p), _p(out, _u8p), _p(m, _f64p),
                                 _p(pms, _f64p), _p(mms, _f64p))
        if rc != 0:
            raise ValueError("quantize failed")
        return dict(centers=C_out.reshape(k, 3), iterations=int(it[0]), sse=float(sse[0]), dist_evals=int(ev[0]),
                    mapped=out, mse=float(m[0]), palette_ms=float(pms[0]), map_ms=float(mms[0]))

    # -- §8(f) f1: file formats (reference only) ---------------------------
    PPM_KINDS = {0: "ok", 1: "BadMagic", 2: "BadHeader", 3: "BadMaxval", 4: "Truncated", -1: "runtime"}

    def write_ppm(self, img: np.ndarray) -> bytes:
        assert self.kind == "reference"
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape[:2]
        n = self._f("write_ppm")(_p(img, _u8p), w, h, None, 0)
        out = np.zeros(n, np.uint8)
        self._f("write_ppm")(_p(img, _u8p), w, h, _p(out, _u8p), n)
        return out.tobytes()

    def read_ppm(self, data: bytes):
        """(kind, image or None) with kind in PPM_KINDS."""
        assert self.kind == "reference"
        buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
        w = np.zeros(1, np.int32)
        h = np.zeros(1, np.int32)
        cap = max(len(data) * 3, 16)
        out = np.zeros(cap, np.uint8)
        rc = self._f("read_ppm")(_p(buf, _u8p), len(data), _p(out, _u8p), cap, _p(w, _i32p), _p(h, _i32p))
        if rc != 0:
            return self.PPM_KINDS[rc], None
        return "ok", out[: 3 * int(w[0]) * int(h[0])].reshape(int(h[0]), int(w[0]), 3).copy()

    def palette_text(self, centers: np.ndarray) -> str:
        assert self.kind == "reference"
        c = np.ascontiguousarray(centers, np.float64).reshape(-1)
        k = c.size // 3
        n = self._f("palette_text")(_p(c, _f64p), k, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self._f("palette_text")(_p(c, _f64p), k, buf, n)
        return buf.raw[:n].decode()

    def run_km_full(self, img: np.ndarray, k: int, mode: int = 1, max_iters: int = 10, eps: float = 1e-4,
                    cap: int = 100, seed: int = 1):
        """run_km_full (kmeans.hpp:409-426): KM / KM-C over every pixel."""
        assert self.kind == "reference"
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape[:2]
        C_out = np.zeros(3 * k)
        sse = np.zeros(1)
        ev = np.zeros(1, np.uint64)
        hist = np.zeros(max(cap, max_iters) + 1)
        it = self._f("run_km_full")(_p(img, _u8p), w, h, k, mode, max_iters, eps, cap, seed, _p(C_out, _f64p),
                                    _p(sse, _f64p), _p(ev, _u64p), _p(hist, _f64p), hist.size)
        if it < 0:
            raise ValueError("run_km_full failed")
        return dict(centers=C_out.reshape(k, 3), iterations=int(it), sse=float(sse[0]), dist_evals=int(ev[0]),
                    sse_history=hist[:it].copy())

    def run_fkm(self, img: np.ndarray, k: int, k_prime: int = 8, mode: int = 1, max_iters: int = 10,
                eps: float = 1e-4, seed: int = 1):
        """generate_palette FKM / FKM-C (methods.hpp:163-178; hard cap 1000)."""
        assert self.kind == "reference"
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape[:2]
        C_out = np.zeros(3 * k)
        sse = np.zeros(1)
        ev = np.zeros(1, np.uint64)
        hist = np.zeros(1001)
        it = self._f("run_fkm")(_p(img, _u8p), w, h, k, k_prime, mode, max_iters, eps, seed, _p(C_out, _f64p),
                                _p(sse, _f64p), _p(ev, _u64p), _p(hist, _f64p), hist.size)
        if it < 0:
            raise ValueError("run_fkm failed")
        return dict(centers=C_out.reshape(k, 3), iterations=int(it), sse=float(sse[0]), dist_evals=int(ev[0]),
                    sse_history=hist[:it].copy())

    def run_bench(self, config_text: str, prefix: str) -> None:
        """run_bench + write_bench_outputs (bench.hpp:160-313), single thread."""
        assert self.kind == "reference"
        if self._f("run_bench")(config_text.encode(), prefix.encode()) != 0:
            raise ValueError("run_bench failed")

    def error_image(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        assert self.kind == "reference"
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        out = np.zeros_like(a)
        self._f("error_image")(_p(a, _u8p), _p(b, _u8p), a.size // 3, _p(out, _u8p))
        return out

    def quantize_many(self, imgs, k: int, nthreads: int, mode: int = 1, max_iters: int = 10, eps: float = 1e-4,
                      cap: int = 100, seed: int = 1):
        """Independent images on a native thread pool; returns (wall_ms, mses, iters)."""
        assert self.kind == "reference"
        imgs = [np.ascontiguousarray(i, np.uint8) for i in imgs]
        h, w = imgs[0].shape[:2]
        arr = (_u8p * len(imgs))(*[_p(i, _u8p) for i in imgs])
        mses = np.zeros(len(imgs))
        its = np.zeros(len(imgs), np.int32)
        ms = self._f("quantize_many")(arr, len(imgs), w, h, k, mode, max_iters, eps, cap, seed, nthreads,
                                      _p(mses, _f64p), _p(its, _i32p))
        return float(ms), mses, its
