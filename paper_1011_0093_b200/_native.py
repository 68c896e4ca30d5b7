"""ctypes binding of the C ABI (include/colorq_b200.h).

The CUDA library is built in-tree by ``__graft_entry__.build()`` (or
``make``) into ``paper_1011_0093_b200/lib/libcolorq_b200.so``. There is no
fallback: if the library is missing or no sm_100 device is present, every
call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

LIB_PATH = os.environ.get("CQB_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                          "libcolorq_b200.so")  # env: A/B diagnostics only

CQB_OK = 0
CQB_ERR_INVALID_ARGUMENT = 1
CQB_ERR_UNSUPPORTED = 2
CQB_ERR_CUDA = 3
CQB_ERR_OOM = 4
CQB_ERR_NCCL = 5
CQB_ERR_INTERNAL = 6
MAX_K = 256

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTS = (
    "cqb_create", "cqb_destroy", "cqb_last_error", "cqb_set_stream", "cqb_set_grid_limit", "cqb_device_info",
    "cqb_build_histogram", "cqb_run_wsm", "cqb_wsm_iterate", "cqb_quantize", "cqb_quantize_device",
    "cqb_fetch_results", "cqb_quantize_batch", "cqb_quantize_runs", "cqb_quantize_ex", "cqb_error_image", "cqb_run_km_full", "cqb_run_fkm",
    "cqb_map_pixels", "cqb_mse", "cqb_set_profiling", "cqb_stage_times",
    "cqb_loop_timeline", "cqb_block_times", "cqb_shard_prepare", "cqb_shard_step", "cqb_finalize_moments",
    "cqb_shard_reseed_candidate", "cqb_set_debug", "cqb_xch_window", "cqb_xch_open", "cqb_xch_emulate",
    "cqb_quantize_sharded", "cqb_xch_set_timeout", "cqb_init_centers", "cqb_points_tables", "cqb_points_assign",
    "cqb_points_update", "cqb_points_sse", "cqb_run_wsm_points", "cqb_hist_rows", "cqb_hist_merge", "cqb_hist_range",
    "cqb_quantize_sharded_samples",
)
IPC_HANDLE_BYTES = 64  # CQB_IPC_HANDLE_BYTES (cudaIpcMemHandle_t)
# cqb_stage_times intervals: memsets | K1 | K2b | init + bitmap scan + rank (+ gather) | loop | map tables+unique | map pixels
STAGES = ("reset", "hist_count", "bins_compact", "init_rank", "wsm_loop", "map_unique", "map_pixels")


class Termination(C.Structure):
    _fields_ = [("mode", C.c_int), ("max_iters", C.c_int), ("epsilon", C.c_double), ("hard_cap", C.c_int)]


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int), ("k", C.c_int), ("seed", C.c_uint64), ("sse", C.c_double), ("mse", C.c_double),
        ("elapsed_ms", C.c_double), ("map_ms", C.c_double), ("dist_evals", C.c_uint64), ("n_unique", C.c_uint64),
        ("empty_events", C.c_int), ("gpu_launches", C.c_int),
    ]


class CqbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[cqb {code}] {msg}")
        self.code = code


class CqbInvalidArgument(CqbError, ValueError):
    """Maps the reference's std::invalid_argument."""


_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p
_T = C.POINTER(Termination)
_R = C.POINTER(Report)

_lib = None
_lock = threading.Lock()


def load_library() -> C.CDLL:
    """Load the in-tree CUDA library (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"colorq_b200 CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.cqb_create.argtypes = [C.c_int, C.POINTER(_vp)]
        L.cqb_destroy.argtypes = [_vp]
        L.cqb_last_error.argtypes = [_vp]
        L.cqb_last_error.restype = C.c_char_p
        L.cqb_set_stream.argtypes = [_vp, _vp]
        L.cqb_set_grid_limit.argtypes = [_vp, C.c_int]
        L.cqb_device_info.argtypes = [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.cqb_build_histogram.argtypes = [_vp, _u8p, C.c_uint64, _u32p, _u32p, _f64p, _u32p, C.c_uint64, _u64p]
        L.cqb_run_wsm.argtypes = [_vp, _u32p, _u32p, C.c_uint64, C.c_uint64, C.c_int, _T, C.c_uint64, _f64p, _f64p,
                                  C.c_int, _f64p, C.c_int, _u8p, _R]
        L.cqb_wsm_iterate.argtypes = [_vp, _u32p, _u32p, C.c_uint64, C.c_uint64, C.c_int, _f64p, _u8p, C.c_int, _T,
                                      _f64p, _f64p, C.c_int, _R]
        L.cqb_quantize.argtypes = [_vp, _u8p, C.c_int, C.c_int, C.c_int, _T, C.c_uint64, _f64p, _f64p, C.c_int, _u8p,
                                   _u8p, _R]
        L.cqb_quantize_device.argtypes = [_vp, _vp, C.c_uint64, C.c_int, _T, C.c_uint64, _vp, _vp, C.c_int, _f64p,
                                          _f64p, C.c_int, _R]
        L.cqb_fetch_results.argtypes = [_vp, _f64p, _f64p, C.c_int, _R]
        L.cqb_quantize_ex.argtypes = [_vp, _u8p, C.c_int, C.c_int, C.c_int, _T, C.c_uint64, _f64p, _f64p, C.c_int,
                                      _u8p, _u8p, _u8p, _R]
        L.cqb_error_image.argtypes = [_vp, _u8p, _u8p, C.c_uint64, _u8p]
        L.cqb_run_km_full.argtypes = [_vp, _u8p, C.c_int, C.c_int, C.c_int, _T, C.c_uint64, _f64p, _f64p, C.c_int,
                                      _R]
        L.cqb_run_fkm.argtypes = [_vp, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, _T, C.c_uint64, _f64p, _f64p,
                                  C.c_int, _R]
        if hasattr(L, "cqb_quantize_runs"):  # (older builds in A/B runs lack the newest entry points)
            L.cqb_quantize_runs.argtypes = [_vp, _u8p, C.c_uint64, C.c_int, _T, C.c_int, _u64p, C.c_int, _f64p, _R]
        L.cqb_quantize_batch.argtypes = [_vp, C.c_int, C.POINTER(_vp), _u64p, C.c_int, _T, C.c_uint64,
                                         C.POINTER(_vp), C.POINTER(_vp), C.c_int, _f64p, _R]
        L.cqb_map_pixels.argtypes = [_vp, _u8p, C.c_uint64, _f64p, C.c_int, _u8p, _u8p, _u64p]
        L.cqb_mse.argtypes = [_vp, _u8p, _u8p, C.c_uint64, _f64p]
        L.cqb_set_profiling.argtypes = [_vp, C.c_int]
        L.cqb_stage_times.argtypes = [_vp, C.POINTER(C.c_float), C.c_int]
        L.cqb_loop_timeline.argtypes = [_vp, _u64p, C.c_int]
        L.cqb_block_times.argtypes = [_vp, _u64p, C.c_int]
        L.cqb_set_debug.argtypes = [_vp, C.c_int]
        L.cqb_shard_prepare.argtypes = [_vp, _u8p, C.c_uint64, C.c_int, C.c_uint64, _u64p, _f64p]
        L.cqb_shard_step.argtypes = [_vp, C.c_uint64, C.c_uint64, _f64p, C.c_int, _u64p, _u64p]
        L.cqb_finalize_moments.argtypes = [_vp, _u64p, _f64p, C.c_int, C.c_uint64, _f64p, _f64p,
                                           C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.cqb_shard_reseed_candidate.argtypes = [_vp, C.c_uint64, C.c_uint64, _f64p, _u32p, C.c_int, _f64p, _u32p,
                                                 _u32p]
        L.cqb_xch_window.argtypes = [_vp, C.c_int, C.c_int, _vp]
        L.cqb_xch_open.argtypes = [_vp, _vp]
        L.cqb_xch_emulate.argtypes = [_vp, C.c_int]
        _i32p = C.POINTER(C.c_int32)
        if hasattr(L, "cqb_run_wsm_points"):
            L.cqb_init_centers.argtypes = [_vp, C.c_uint64, C.c_int, C.c_uint64, _u32p]
            L.cqb_points_tables.argtypes = [_vp, _f64p, C.c_int, _f64p, _i32p]
            L.cqb_points_assign.argtypes = [_vp, _f64p, _f64p, C.c_uint64, _f64p, C.c_int, _f64p, _i32p, C.c_int,
                                            _i32p, _f64p, _u64p, _i32p, _f64p]
            L.cqb_points_update.argtypes = [_vp, _f64p, _f64p, C.c_uint64, _i32p, _f64p, C.c_int, _f64p]
            L.cqb_points_sse.argtypes = [_vp, _f64p, _f64p, C.c_uint64, _f64p, C.c_int, _i32p, _f64p]
            L.cqb_run_wsm_points.argtypes = [_vp, _f64p, _f64p, C.c_uint64, C.c_int, _T, C.c_uint64, _f64p, _f64p,
                                             C.c_int, _f64p, C.c_int, _i32p, _R]
        if hasattr(L, "cqb_xch_set_timeout"):
            L.cqb_xch_set_timeout.argtypes = [_vp, C.c_double]
        L.cqb_quantize_sharded.argtypes = [_vp, _vp, C.c_uint64, C.c_int, _T, C.c_uint64, _vp, _vp, _u64p]
        L.cqb_hist_rows.argtypes = [_vp, _vp, C.c_uint64, C.c_int, C.c_int, _vp, C.c_uint64, _u64p, _u64p]
        L.cqb_hist_merge.argtypes = [_vp, _vp, C.c_uint64, _vp, C.c_uint64, _u64p]
        L.cqb_hist_range.argtypes = [_vp, _vp, C.c_uint64, C.c_int, C.c_int, _vp, C.c_uint64, _u64p]
        L.cqb_quantize_sharded_samples.argtypes = [_vp, _vp, C.c_uint64, _vp, C.c_uint64, C.c_int, _T, C.c_uint64,
                                                   _vp, _vp, _u64p]
        _lib = L
        return L


class Context:
    """One device context (stream + arena). Not shared across threads."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = _vp()
        rc = self.lib.cqb_create(device, C.byref(h))
        if rc != CQB_OK:
            raise CqbError(rc, f"cqb_create(device={device}) failed (see stderr)")
        self.h = h
        self.device = device

    def check(self, rc: int) -> None:
        if rc == CQB_OK:
            return
        msg = self.lib.cqb_last_error(self.h).decode(errors="replace")
        if rc == CQB_ERR_INVALID_ARGUMENT:
            raise CqbInvalidArgument(rc, msg)
        raise CqbError(rc, msg)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.cqb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def context(device: int = 0) -> Context:
    """Thread-local context per device (the re-entrancy contract)."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]
