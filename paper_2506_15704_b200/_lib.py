"""ctypes binding of liblfps_b200.so (include/lfps_b200.h).

The library is built in-tree (paper_2506_15704_b200/lib/liblfps_b200.so, by
``__graft_entry__.build()`` or ``make -C paper_2506_15704_b200/csrc``).  There
is no CPU fallback: if the library is missing or no CUDA device is visible,
every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DeviceError

# LFPS_LIB selects another in-tree build of the same sources (tools/build_variant.sh
# experiments); the default is the library __graft_entry__.build() makes
LIB_PATH = os.environ.get("LFPS_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "liblfps_b200.so")
ABI_VERSION = 9
FLAG_EXPORT_SETS = 1
FLAG_TRACE = 2
FLAG_SPLIT = 8
FLAG_GRAPH = 16
FLAG_PREFETCHED = 64

# per-session device error codes (include/lfps_b200.h)
ERR_NAMES = {
    1: "non-finite logits in sparsity estimate",
    2: "non-finite sparsity ratio",
    3: "float division by zero (kappa == 0 in compute_thresholds)",
    4: "selection weights must sum to 1",
    5: "each prefill weight vector must sum to 1 over its non-sink range",
    6: "zero-norm prefill query",
    7: "softmax input contains non-finite scores",
}

EXPORTS = ("lfps_abi_version", "lfps_last_error", "lfps_workspace_layout",
           "lfps_bootstrap_tables", "lfps_bootstrap_stats", "lfps_decode_step",
           "lfps_decode_step_host_out", "lfps_decode_step_host_io", "lfps_step_input_bytes",
           "lfps_decode_prefetch", "lfps_wait_output",
           "lfps_exact_topk_step", "lfps_overlap", "lfps_decode_launches", "lfps_slash_capacity",
           "lfps_exact_launches", "lfps_kv_pool_page_bytes", "lfps_kv_pool_create",
           "lfps_kv_pool_reserve", "lfps_kv_pool_release", "lfps_kv_pool_mapped_bytes",
           "lfps_kv_pool_destroy", "lfps_profile_enable", "lfps_profile_collect",
           "lfps_workspace_release", "lfps_bootstrap_stats_requests", "lfps_stage_logits", "lfps_stage_thresholds",
           "lfps_stage_candidates", "lfps_stage_topk", "lfps_stage_attend", "lfps_stage_update",
           "lfps_stage_grow", "lfps_stage_init_tables", "lfps_stage_head_stats",
           "lfps_stage_gate")


class Dims(C.Structure):
    _fields_ = [("batch", C.c_int32), ("kv_heads", C.c_int32), ("group", C.c_int32),
                ("d", C.c_int32), ("n_max", C.c_int32), ("m_cap", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("r", C.c_double), ("epsilon", C.c_double), ("a", C.c_double),
                ("k_fraction", C.c_double), ("sqrt_d", C.c_double), ("sqrt_d_f32", C.c_float),
                ("s", C.c_int32), ("sink_count", C.c_int32), ("local_window", C.c_int32),
                ("bypass_mode", C.c_int32), ("exhaustive", C.c_int32),
                ("n_offsets", C.c_int32), ("offsets", C.c_int32 * 16), ("flags", C.c_int32)]


class State(C.Structure):
    _fields_ = [("k_cache", C.c_void_p), ("v_cache", C.c_void_p), ("n_ctx", C.c_void_p),
                ("ver", C.c_void_p), ("sla", C.c_void_p), ("scale", C.c_void_p),
                ("sla_base", C.c_void_p), ("clamp_count", C.c_void_p),
                ("mean_key", C.c_void_p), ("mean_value", C.c_void_p),
                ("sigma_hat_sq", C.c_void_p), ("block_table", C.c_void_p),
                ("block_rows", C.c_int32), ("max_blocks", C.c_int32)]


class WsLayout(C.Structure):
    _fields_ = [("total_bytes", C.c_size_t), ("rho", C.c_size_t), ("bypass", C.c_size_t),
                ("err", C.c_size_t), ("out", C.c_size_t), ("thr", C.c_size_t),
                ("counts", C.c_size_t), ("bits", C.c_size_t), ("probe_idx", C.c_size_t),
                ("probe_score", C.c_size_t), ("c2_idx", C.c_size_t), ("c2_score", C.c_size_t), ("uw", C.c_size_t),
                ("scratch", C.c_size_t), ("bsum", C.c_size_t), ("bmax", C.c_size_t),
                ("dirty", C.c_size_t), ("valid", C.c_size_t), ("wstat", C.c_size_t), ("trace", C.c_size_t),
                ("done", C.c_size_t), ("hot", C.c_size_t),
                ("thr_next", C.c_size_t),
                ("nblk", C.c_int32), ("dirty_words", C.c_int32), ("words", C.c_int32),
                ("list_cap", C.c_int32)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int32), ("total_ms", C.c_double)]


class Workspace(C.Structure):
    _fields_ = [("base", C.c_void_p), ("bytes", C.c_size_t)]


_lib = None
_lock = threading.Lock()


def _declare(lib):
    P = C.POINTER
    lib.lfps_abi_version.restype = C.c_int
    lib.lfps_last_error.restype = C.c_char_p
    lib.lfps_workspace_layout.argtypes = [P(Dims), P(WsLayout)]
    lib.lfps_slash_capacity.argtypes = [P(Dims)]
    lib.lfps_bootstrap_tables.argtypes = [P(Dims), P(Params), P(State), P(Workspace), C.c_void_p,
                                          C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
    lib.lfps_bootstrap_stats.argtypes = [P(Dims), P(Params), P(State), P(Workspace), C.c_void_p,
                                         C.c_void_p]
    lib.lfps_decode_step.argtypes = [P(Dims), P(Params), P(State), P(Workspace), C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.lfps_decode_step_host_out.argtypes = [P(Dims), P(Params), P(State), P(Workspace),
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p]
    lib.lfps_decode_step_host_io.argtypes = [P(Dims), P(Params), P(State), P(Workspace),
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_void_p]
    lib.lfps_decode_prefetch.argtypes = [P(Dims), P(Params), P(State), P(Workspace), C.c_void_p,
                                         C.c_void_p]
    lib.lfps_wait_output.argtypes = [P(Workspace)]
    lib.lfps_step_input_bytes.argtypes = [P(Dims)]
    lib.lfps_step_input_bytes.restype = C.c_int64
    lib.lfps_kv_pool_page_bytes.argtypes = []
    lib.lfps_kv_pool_page_bytes.restype = C.c_int64
    lib.lfps_kv_pool_create.argtypes = [P(Dims), P(C.c_void_p), P(C.c_void_p), P(C.c_void_p)]
    lib.lfps_kv_pool_reserve.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64]
    lib.lfps_kv_pool_release.argtypes = [C.c_void_p, C.c_int32]
    lib.lfps_kv_pool_mapped_bytes.argtypes = [C.c_void_p]
    lib.lfps_kv_pool_mapped_bytes.restype = C.c_int64
    lib.lfps_kv_pool_destroy.argtypes = [C.c_void_p]
    for name in ("lfps_kv_pool_create", "lfps_kv_pool_reserve", "lfps_kv_pool_release",
                 "lfps_kv_pool_destroy"):
        getattr(lib, name).restype = C.c_int
    lib.lfps_exact_topk_step.argtypes = [P(Dims), P(Params), P(State), P(Workspace), C.c_void_p,
                                         C.c_void_p, C.c_void_p]
    lib.lfps_overlap.argtypes = [P(Dims), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
    lib.lfps_profile_enable.argtypes = [C.c_int]
    lib.lfps_workspace_release.argtypes = [P(Workspace)]
    lib.lfps_bootstrap_stats_requests.argtypes = [P(Dims), P(Params), P(State), P(Workspace),
                                                  C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
    lib.lfps_bootstrap_stats_requests.restype = C.c_int
    lib.lfps_workspace_release.restype = C.c_int
    # per-head stage API (k_stages.cu): device pointers as c_void_p
    V, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    stage = {
        "lfps_stage_logits": [V, I32, V, I32, V, V, V],
        "lfps_stage_thresholds": [V, V, I32, D, D, I32, V, V, V],
        "lfps_stage_candidates": [I32, V, V, I32, D, V, V, I32, V, I32, I64, I32, I32, I32, V, V,
                                  V],
        "lfps_stage_topk": [V, V, I32, I32, V, V, V],
        "lfps_stage_attend": [V, V, I32, V, I32, V, V, V, V, V],
        "lfps_stage_update": [V, V, I32, I32, V, V, I32, I32, D, D, V, V, V],
        "lfps_stage_grow": [V, V, I32, I32, I32, V],
        "lfps_stage_init_tables": [V, I32, I32, D, V, V, V],
        "lfps_stage_head_stats": [V, V, I32, I32, I32, V, V, V, V, V, V, V],
        "lfps_stage_gate": [V, V, I32, I32, I32, I32, V, V, V, D, I32, V, V, V],
    }
    for name, args in stage.items():
        getattr(lib, name).argtypes = args
        getattr(lib, name).restype = C.c_int
    lib.lfps_decode_launches.argtypes = [C.c_void_p, C.c_int32]
    lib.lfps_profile_collect.argtypes = [P(KernelTime), C.c_int32, P(C.c_int32)]
    for name in ("lfps_profile_enable", "lfps_profile_collect", "lfps_workspace_layout",
                 "lfps_bootstrap_tables", "lfps_bootstrap_stats", "lfps_decode_step",
                 "lfps_decode_step_host_out", "lfps_decode_step_host_io", "lfps_exact_topk_step",
                 "lfps_overlap",
                 "lfps_decode_launches", "lfps_exact_launches", "lfps_slash_capacity"):
        getattr(lib, name).restype = C.c_int


def load_library(path: str = LIB_PATH):
    """Load (once) and return the CDLL; raises DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is not built: run __graft_entry__.build() or "
                "make -C paper_2506_15704_b200/csrc (there is no CPU fallback)")
        lib = C.CDLL(path)
        _declare(lib)
        if lib.lfps_abi_version() != ABI_VERSION:
            raise DeviceError(f"ABI mismatch: library {lib.lfps_abi_version()} != {ABI_VERSION}")
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load_library().lfps_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise DeviceError(f"{what} failed ({rc}): {msg}")


def slash_capacity(dims: Dims) -> int:
    cap = load_library().lfps_slash_capacity(C.byref(dims))
    check(min(cap, 0), "slash_capacity")
    return cap


def workspace_layout(dims: Dims) -> WsLayout:
    lay = WsLayout()
    check(load_library().lfps_workspace_layout(C.byref(dims), C.byref(lay)), "workspace_layout")
    return lay


def profile_enable(on: bool) -> None:
    check(load_library().lfps_profile_enable(1 if on else 0), "profile_enable")


def profile_collect() -> dict:
    """{kernel name: (launches, total_ms)} since the last collect."""
    buf = (KernelTime * 64)()
    n = C.c_int32(0)
    check(load_library().lfps_profile_collect(buf, 64, C.byref(n)), "profile_collect")
    return {buf[i].name.decode(): (buf[i].launches, buf[i].total_ms) for i in range(n.value)}
