"""ctypes binding of liblrqk_b200.so (include/lrqk_b200.h).

The library is the only compute path: if it cannot be loaded, or no CUDA
device is present, every entry point raises instead of falling back to CPU
code.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LRQK_LIB_PATH") or os.path.join(_HERE, "liblrqk_b200.so")

F32, BF16 = 0, 1
SLOW_HBM, SLOW_HOST = 0, 1

ST_NONFINITE = 1
ST_SOLVE_FAILED = 2
ST_INDEX_RANGE = 4
ST_CAPACITY = 8
ST_JITTERED = 16
ST_FALLBACK = 32
ST_BARRIER = 64

OK, EINVAL, ECUDA, EUNSUPPORTED = 0, 1, 2, 3

_INT_FIELDS = ("batch", "n_q_heads", "n_kv_heads", "head_dim", "dim_stride", "rank", "rank_stride",
               "t_max", "k_budget", "lite_budget", "s_cap", "n_slots", "cand_cap", "dtype", "policy",
               "max_iter")
_FLOAT_FIELDS = ("lambda_1", "lambda_2", "tol")
BUFFER_NAMES = ("proxy", "B_Q", "B_K", "slow_k", "slow_v", "slot_k", "slot_v", "ctx_len", "res_idx",
                "res_slot", "res_cnt", "spare_slot", "miss_idx", "miss_slot", "miss_cnt", "c_miss",
                "c_total", "step_miss", "step_total", "q_hat", "k_hat", "eta", "keys", "hist",
                "sel_meta", "sure_idx", "cand", "red_scratch", "attn_scratch", "counters", "status", "pre",
                "fcand", "fcnt", "res_bits", "cmask", "proxy_rowmajor")


class LayerStruct(C.Structure):
    """Mirror of lrqk_layer_t."""

    _fields_ = ([(n, C.c_int32) for n in _INT_FIELDS] + [(n, C.c_float) for n in _FLOAT_FIELDS]
                + [(n, C.c_void_p) for n in BUFFER_NAMES])


class PrefillStruct(C.Structure):
    """Mirror of lrqk_prefill_t."""

    _fields_ = [(n, C.c_int32) for n in ("n_heads", "group", "len", "head_dim", "dim_stride", "rank",
                                         "rank_stride", "dtype", "max_iter")] + \
               [(n, C.c_float) for n in ("lambda_q", "lambda_k", "tol")] + \
               [("want_objective", C.c_int32)] + \
               [(n, C.c_void_p) for n in ("Q", "K", "A_Q", "A_K", "B_Q", "B_K", "objective", "sweeps",
                                          "converged", "scratch", "status", "A_Q0", "A_K0")] + \
               [("init_shared", C.c_int32)]


class LibraryUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing; there is no CPU fallback."""


_lib = None

# exported symbols and their signatures (restype, argtypes)
_P = C.c_void_p
SIGNATURES = {
    "lrqk_abi_version": (C.c_int, []),
    "lrqk_sizeof_layer": (C.c_size_t, []),
    "lrqk_sizeof_prefill": (C.c_size_t, []),
    "lrqk_buffer_names": (C.c_char_p, []),
    "lrqk_last_error": (C.c_char_p, []),
    "lrqk_layer_buffer_bytes": (C.c_int, [C.POINTER(LayerStruct), C.POINTER(C.c_size_t), C.c_int]),
    "lrqk_red_chunks": (C.c_int, [C.POINTER(LayerStruct)]),
    "lrqk_attn_splits": (C.c_int, [C.POINTER(LayerStruct)]),
    "lrqk_seed_prompt": (C.c_int, [C.POINTER(LayerStruct), C.c_int32, _P]),
    "lrqk_decode_compress": (C.c_int, [C.POINTER(LayerStruct), _P, _P, _P, C.c_int, _P]),
    "lrqk_compress_prepare": (C.c_int, [C.POINTER(LayerStruct), _P]),
    "lrqk_score": (C.c_int, [C.POINTER(LayerStruct), _P]),
    "lrqk_select": (C.c_int, [C.POINTER(LayerStruct), _P]),
    "lrqk_gather_misses": (C.c_int, [C.POINTER(LayerStruct), _P]),
    "lrqk_attention": (C.c_int, [C.POINTER(LayerStruct), _P, _P, _P]),
    "lrqk_compress_prepare_layers": (C.c_int, [_P, C.POINTER(LayerStruct), C.c_int32, _P]),
    "lrqk_select_attend": (C.c_int, [C.POINTER(LayerStruct), _P, _P, _P]),
    "lrqk_score_attend": (C.c_int, [C.POINTER(LayerStruct), _P, _P, _P]),
    "lrqk_set_fused": (C.c_int, [C.c_int]),
    "lrqk_workspace_size": (C.c_size_t, [C.POINTER(LayerStruct)]),
    "lrqk_score_append": (C.c_int, [C.POINTER(LayerStruct), _P]),
    "lrqk_cache_update": (C.c_int, [C.POINTER(LayerStruct), _P]),
    "lrqk_get_status": (C.c_int, [C.POINTER(LayerStruct), _P, _P]),
    "lrqk_counters": (C.c_int, [C.POINTER(LayerStruct), _P, _P, _P]),
    "lrqk_decode_step": (C.c_int, [C.POINTER(LayerStruct), _P, _P, _P, _P, C.c_int, _P]),
    "lrqk_advance": (C.c_int, [_P, C.c_int32, _P]),
    "lrqk_proxy_scores_f32": (C.c_int, [_P, C.c_int32, _P, _P, C.c_int32, C.c_int32, C.c_int32, _P]),
    "lrqk_select_scores": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P,
                                     C.c_size_t, _P]),
    "lrqk_select_scores_workspace": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "lrqk_prefill_scratch_bytes": (C.c_size_t, [C.POINTER(PrefillStruct)]),
    "lrqk_prefill_factorize": (C.c_int, [C.POINTER(PrefillStruct), _P]),
    "lrqk_read_status": (C.c_int, [_P, _P, _P]),
    "lrqk_host_alloc": (_P, [C.c_size_t]),
    "lrqk_host_free": (None, [_P]),
    "lrqk_host_device_ptr": (_P, [_P]),
    "lrqk_attention_rows": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P]),
    "lrqk_count_misses": (C.c_int, [_P, C.c_int32, _P, C.c_int32, C.c_int32, _P, _P]),
    "lrqk_line_search": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P]),
    "lrqk_gemm_f64": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, _P, C.c_int32,
                                _P, C.c_int32, C.c_double, _P, C.c_int32, _P, C.c_size_t, _P]),
    "lrqk_gemm_f64_workspace": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
    "lrqk_symmetrize_f64": (C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    "lrqk_dot_f64": (C.c_int, [_P, _P, C.c_int64, _P, _P, _P]),
    "lrqk_axpby_f64": (C.c_int, [C.c_int64, C.c_double, _P, _P, C.c_double, _P, _P]),
    "lrqk_solve_spd_f64": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32, _P, C.c_int32, _P, _P, _P]),
    "lrqk_topk_f64": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P]),
    "lrqk_trace_enable": (C.c_int, [C.c_int]),
    "lrqk_trace_read": (C.c_int, [_P, C.c_int]),
}


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryUnavailable(
            f"{path} is missing; build it with `make` (or __graft_entry__.build()). "
            "There is no CPU fallback for the LRQK path.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.lrqk_sizeof_layer() != C.sizeof(LayerStruct):
        raise LibraryUnavailable("lrqk_layer_t layout mismatch between header and binding")
    if lib.lrqk_sizeof_prefill() != C.sizeof(PrefillStruct):
        raise LibraryUnavailable("lrqk_prefill_t layout mismatch between header and binding")
    names = tuple(lib.lrqk_buffer_names().decode().split(","))
    if names != BUFFER_NAMES:
        raise LibraryUnavailable(f"buffer order mismatch: {names}")
    _lib = lib
    return lib


def lib():
    """The loaded library, requiring a CUDA device (used by every compute call)."""
    import torch

    if not torch.cuda.is_available():
        raise LibraryUnavailable("no CUDA device: the LRQK path runs only on the GPU (sm_100a)")
    return load_library()


def check(rc: int, what: str):
    if rc != OK:
        err = _lib.lrqk_last_error().decode() if _lib is not None else ""
        kind = {EINVAL: "invalid argument", ECUDA: "CUDA error", EUNSUPPORTED: "unsupported shape"}.get(rc, rc)
        raise RuntimeError(f"{what}: {kind} {err}".strip())


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
