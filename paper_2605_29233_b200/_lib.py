"""ctypes binding of ``libbb200.so`` (the C-ABI declared in include/bb200.h).

Loading fails loudly when the library is missing: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, ContractError, RunawayError, StateError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BB_LIB_PATH") or os.path.join(_HERE, "libbb200.so")  # (override: A/B builds)

BB_OK = 0
BB_ERR_CONFIG, BB_ERR_CONTRACT, BB_ERR_STATE, BB_ERR_RUNAWAY = -1, -2, -3, -4
BB_ERR_CUDA, BB_ERR_NOMEM = -10, -11

_lib = None

vp, i32, i64, f32 = C.c_void_p, C.c_int, C.c_longlong, C.c_float
i32p, i64p = C.POINTER(C.c_int), C.POINTER(C.c_longlong)



class ModelDesc(C.Structure):
    """bb_model_desc (include/bb200.h)"""
    _fields_ = [(n, C.c_int) for n in ("arch", "vocab_size", "layers", "d_model", "n_heads", "n_kv_heads",
                                       "head_dim", "d_ff", "max_len", "qkv_bias", "dtype")] + \
               [("rope_theta", C.c_float), ("norm_eps", C.c_float), ("gamma", C.c_float), ("radius", C.c_int),
                ("head_scale", C.c_float), ("spike_cut", C.c_float), ("spike_gain", C.c_float)]


class Weights(C.Structure):
    """bb_weights (include/bb200.h)"""
    _fields_ = [(n, C.c_void_p) for n in ("emb", "pos", "wqkv", "bqkv", "wo", "wgu", "wd", "ln1", "ln2", "lnf",
                                          "head")]


class SessionDesc(C.Structure):
    """bb_session_desc (include/bb200.h)"""
    _fields_ = [("n_requests", C.c_int), ("n_branches", C.c_int), ("block_sizes", C.c_int * 8),
                ("prompt_len", C.c_int), ("gen_len", C.c_int), ("tau_conf", C.c_float),
                ("tau_merge", C.c_float), ("tau_sync", C.c_float), ("refresh_interval", C.c_int),
                ("merge_enabled", C.c_int), ("sync_enabled", C.c_int), ("page_size", C.c_int),
                ("pages_per_item", C.c_int), ("trace", C.c_int), ("event_capacity", C.c_int),
                ("diagnostics", C.c_int), ("test_flags", C.c_int), ("logits", C.c_int), ("seam", C.c_int),
                ("hard_cap", C.c_int)]


ARCH_REF, ARCH_LLADA = 0, 1
DTYPE_F32, DTYPE_BF16, DTYPE_BF16X2 = 0, 1, 2
VIEW_TOKENS, VIEW_TARGET, VIEW_PROMPT, VIEW_CTRL, VIEW_BRANCH, VIEW_EVENTS = 0, 1, 2, 3, 4, 5
VIEW_COVERED, VIEW_PM_M, VIEW_PM_S, VIEW_PAGES, VIEW_REFC = 6, 7, 8, 9, 10
VIEW_HEAD_MASKED, VIEW_HEAD_M, VIEW_HEAD_S, VIEW_HEAD_ARG, VIEW_SLOT_POS, VIEW_SLOT_BR = 11, 12, 13, 14, 15, 16
VIEW_INIT_GEN = 17
# per-request control words (csrc/bb_state.cuh: enum Ctrl)
(C_STATUS, C_WINNER, C_EOS, C_ITER, C_SINCE_REFRESH, C_NFE0, C_NFE1, C_NFE2, C_NEV, C_REFRESH_DUE,
 C_EV_OVERFLOW, C_ACTIVE_MASK, C_REFRESH_MASK, C_NCOPY, C_NPMCOPY, C_MERGES, C_SYNCS, C_COMMITS,
 C_REFRESHES, C_BLOCK_ROWS, C_COW_PAGES, C_SHARED_PAGES, C_LAST_ACTIVE) = range(23)
C_WORDS = 32
B_START, B_END, B_DONE, B_DEC, B_MERGED, B_SIZE = range(6)
B_WORDS = 8
EVW = 20
EV_KINDS = ("init", "block_forward", "decode", "merge", "sync", "refresh", "eos_pending", "eos_ready", "finish")
E_KIND, E_BRANCH, E_NFE0, E_NFE1, E_NFE2, E_A0, E_A1, E_A2, E_A3, E_PROB, E_DEC = range(11)
MAXB = 8

# name -> (restype, argtypes)
SIGNATURES = {
    "bb_version": (i32, []),
    "bb_model_create": (i32, [C.POINTER(ModelDesc), C.POINTER(Weights), C.POINTER(vp)]),
    "bb_model_destroy": (i32, [vp]),
    "bb_session_workspace_bytes": (i32, [vp, C.POINTER(SessionDesc), C.POINTER(C.c_size_t)]),
    "bb_session_create": (i32, [vp, C.POINTER(SessionDesc), vp, C.c_size_t, C.POINTER(vp)]),
    "bb_session_destroy": (i32, [vp]),
    "bb_session_view": (i32, [vp, i32, i64p, i64p]),
    "bb_session_info": (i32, [vp, i32p, i32]),
    "bb_session_ctrl": (i32, [vp, i32p, vp]),
    "bb_session_gemm_stats": (i32, [vp, C.POINTER(C.c_ulonglong), i32, vp]),
    "bb_session_phase_stats": (i32, [vp, vp, i32, vp]),
    "bb_session_counters": (i32, [vp, i64p]),
    "bb_session_klog": (i32, [vp, C.POINTER(C.c_ulonglong), i32, i32, i64p, vp]),
    "bb_prefill": (i32, [vp, vp]),
    "bb_block_step": (i32, [vp, vp]),
    "bb_refresh": (i32, [vp, vp]),
    "bb_iteration": (i32, [vp, i32, i32, vp]),
    "bb_run": (i32, [vp, i32, i32, vp, i32p]),
    "bb_run_vanilla": (i32, [vp, i32, i32, vp, i32p]),
    "bb_prefill_part": (i32, [vp, i32, vp]),
    "bb_block_step_part": (i32, [vp, i32, vp]),
    "bb_kv_gather": (i32, [vp, i32, i32, vp, vp]),
    "bb_fresh_kv": (i32, [vp, i32, i32, vp, vp]),
    "bb_seam_init": (i32, [vp, vp]),
    "bb_seam_forward": (i32, [vp, i32, i32, i32, vp]),
    "bb_kv_scatter": (i32, [vp, i32, i32, vp, vp]),
    "bb_head_logits": (i32, [vp, vp, vp, vp]),
    "bb_sqdiff_norm": (i32, [vp, vp, vp, i64, vp, vp]),
    "bb_commit_probs": (i32, [vp, i32, i32, vp, vp, f32, vp, vp, vp]),
    "bb_merge_sync_maps": (i32, [i32, i32, i32, i32, vp, vp, vp, vp, i32, f32, f32, i32, i32, vp, i32, vp, vp, vp,
                                 vp]),
    "bb_fill_hash_uniform": (i32, [vp, i32, i64, C.c_ulonglong, i32, f32, i64, i32, i32, vp]),
    "bb_debug_gemm_tc": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, i32, vp, i64p, vp, vp, f32, f32, f32, vp]),
    "bb_debug_gemm_simt": (i32, [vp, vp, vp, i32, i32, i32, vp]),
}


def lib():
    """Load libbb200.so (building it first if it is absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import _build
        _build.build()
    _lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(_lib, name)
        fn.restype = res
        fn.argtypes = args
    return _lib


def check(rc: int, what: str = "bb call"):
    if rc == BB_OK:
        return
    if rc == BB_ERR_CONFIG:
        raise ConfigError(f"{what}: invalid configuration")
    if rc == BB_ERR_CONTRACT:
        raise ContractError(f"{what}: contract violated")
    if rc == BB_ERR_STATE:
        raise StateError(f"{what}: invalid state")
    if rc == BB_ERR_RUNAWAY:
        raise RunawayError(f"{what}: exceeded the hard forward cap")
    raise RuntimeError(f"{what}: CUDA library error {rc}")
