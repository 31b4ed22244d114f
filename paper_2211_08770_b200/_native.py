"""ctypes declarations of the C ABI in include/tt_b200.h (argument marshalling only).

The shared library is built in-tree (paper_2211_08770_b200/_lib/libtt_b200.so) by
``_build.build_library``.  There is no fallback: if the library is missing this module
raises, and every product entry point fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libtt_b200.so")

TT_STATUS = {
    0: "TT_OK", 1: "TT_EINVAL", 2: "TT_ESHAPE", 3: "TT_EINDEX", 4: "TT_ENOMEM", 5: "TT_ECUDA",
    6: "TT_ENOCONV", 7: "TT_ESINGULAR_GRAM", 8: "TT_ELINDEP", 9: "TT_ENUMDEFECT", 10: "TT_ENOTSUP",
    11: "TT_ECOMM",
}
COMM_ID_BYTES = 128
KINDS = {"cgs": 0, "mgs": 1, "cgs2": 2, "mgs2": 3, "gram": 4, "householder": 5}

EXPORTED = [
    "tt_ctx_create", "tt_ctx_destroy", "tt_ctx_set_stream", "tt_last_error", "tt_status_string",
    "tt_ctx_launch_count", "tt_ctx_sync", "tt_ctx_profile", "tt_ctx_profile_query", "tt_tensor_view", "tt_tensor_free", "tt_upload", "tt_download",
    "tt_sum", "tt_axpy", "tt_matvec", "tt_dot_batch", "tt_gram", "tt_gram_blocks", "tt_element", "tt_norm",
    "tt_round", "tt_round_batch", "tt_orth",
    "tt_round_batch_strided", "tt_batch_shape", "tt_batch_ranks", "tt_batch_view", "tt_batch_download", "tt_batch_arena", "tt_batch_free",
    "tt_round_batch_host",
    "tt_comm_nccl_id", "tt_ctx_comm_nccl", "tt_ctx_comm_ops", "tt_ctx_comm_detach", "tt_ctx_comm_info",
    "tt_plan_slice", "tt_plan_lpt", "tt_plan_gram_blocks", "tt_ctx_round_hook",
]

# tt_comm_ops callbacks (include/tt_b200.h)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
BROADCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)


class CommOps(C.Structure):
    _fields_ = [("allgather", ALLGATHER_FN), ("broadcast", BROADCAST_FN), ("user", C.c_void_p)]


class TTView(C.Structure):
    _fields_ = [("d", C.c_int32), ("n", C.POINTER(C.c_int64)), ("r", C.POINTER(C.c_int64)),
                ("core", C.POINTER(C.c_void_p)), ("norm", C.c_double)]


class RoundOpts(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_rank", C.c_int64), ("floor_c", C.c_double),
                ("qrcp_theta", C.c_double), ("rank_revealing", C.c_int32)]


class RoundInfo(C.Structure):
    _fields_ = [("norm", C.c_double), ("scale", C.c_double), ("tau", C.c_double),
                ("qrcp_steps", C.c_int64), ("resumes", C.c_int64)]


class OrthOpts(C.Structure):
    _fields_ = [("round", RoundOpts), ("hh_beta_literal", C.c_int32), ("want_loo", C.c_int32),
                ("hh_mask", C.c_int32)]


class OrthReport(C.Structure):
    _fields_ = [("rounding_calls", C.c_int64), ("fail_index", C.c_int32),
                ("loo_per_step", C.POINTER(C.c_double)), ("max_rank_per_call", C.POINTER(C.c_int64)),
                ("householder_u", C.POINTER(C.c_void_p))]


ROUND_HOOK_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_double), C.POINTER(TTView),
                            C.POINTER(RoundOpts))


class TTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{TT_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = TT_STATUS.get(status, str(status))


_lib = None


def load() -> C.CDLL:
    """Load libtt_b200.so (raises if it was not built; there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                           "(the CUDA library is the only implementation)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
    VP = C.POINTER(TTView)
    sig = {
        "tt_ctx_create": (C.c_int, [C.c_int, P, C.POINTER(P)]),
        "tt_ctx_destroy": (C.c_int, [P]),
        "tt_ctx_set_stream": (C.c_int, [P, P]),
        "tt_last_error": (C.c_char_p, [P]),
        "tt_status_string": (C.c_char_p, [C.c_int]),
        "tt_ctx_launch_count": (i64, [P]),
        "tt_ctx_sync": (C.c_int, [P]),
        "tt_ctx_profile": (C.c_int, [P, i32]),
        "tt_ctx_profile_query": (C.c_int, [P, i32, C.c_char_p, i32, C.POINTER(i64), C.POINTER(dbl),
                                           C.POINTER(dbl), C.POINTER(dbl)]),
        "tt_tensor_view": (C.c_int, [P, VP]),
        "tt_tensor_free": (C.c_int, [P, P]),
        "tt_upload": (C.c_int, [P, VP, C.POINTER(P)]),
        "tt_download": (C.c_int, [P, P, C.POINTER(P)]),
        "tt_sum": (C.c_int, [P, i32, C.POINTER(dbl), VP, C.POINTER(P)]),
        "tt_axpy": (C.c_int, [P, dbl, VP, VP, C.POINTER(P)]),
        "tt_matvec": (C.c_int, [P, VP, VP, C.POINTER(P)]),
        "tt_dot_batch": (C.c_int, [P, i32, VP, VP, P]),
        "tt_gram": (C.c_int, [P, i32, VP, P]),
        "tt_gram_blocks": (C.c_int, [P, i32, VP, i32, C.POINTER(i32), P]),
        "tt_element": (C.c_int, [P, VP, i32, C.POINTER(i64), P]),
        "tt_norm": (C.c_int, [P, VP, C.POINTER(dbl)]),
        "tt_round": (C.c_int, [P, i32, C.POINTER(dbl), VP, C.POINTER(RoundOpts), C.POINTER(P),
                               C.POINTER(RoundInfo)]),
        "tt_round_batch": (C.c_int, [P, i32, C.POINTER(i32), C.POINTER(C.POINTER(dbl)), C.POINTER(VP),
                                     C.POINTER(RoundOpts), C.POINTER(P), C.POINTER(i64)]),
        "tt_round_batch_strided": (C.c_int, [P, i32, i32, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(P),
                                             C.POINTER(i64), C.POINTER(dbl), C.POINTER(dbl),
                                             C.POINTER(RoundOpts), C.POINTER(P)]),
        "tt_batch_shape": (C.c_int, [P, C.POINTER(i32), C.POINTER(i32)]),
        "tt_batch_ranks": (C.c_int, [P, C.POINTER(i64), C.POINTER(dbl)]),
        "tt_batch_view": (C.c_int, [P, i32, VP]),
        "tt_batch_download": (C.c_int, [P, P, P, i64, C.POINTER(i64)]),
        "tt_batch_arena": (C.c_int, [P, i32, C.POINTER(P), C.POINTER(i64)]),
        "tt_batch_free": (C.c_int, [P, P]),
        "tt_orth": (C.c_int, [P, C.c_int, i32, VP, C.POINTER(OrthOpts), C.POINTER(P), C.POINTER(dbl),
                              C.POINTER(OrthReport)]),
        "tt_round_batch_host": (C.c_int, [P, i32, i32, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(P),
                                          C.POINTER(i64), C.POINTER(dbl), C.POINTER(dbl), C.POINTER(RoundOpts),
                                          i32, P, i64, C.POINTER(i64), C.POINTER(i64), C.POINTER(dbl)]),
        "tt_comm_nccl_id": (C.c_int, [C.POINTER(C.c_uint8)]),
        "tt_ctx_comm_nccl": (C.c_int, [P, i32, i32, C.POINTER(C.c_uint8)]),
        "tt_ctx_comm_ops": (C.c_int, [P, i32, i32, C.POINTER(CommOps)]),
        "tt_ctx_comm_detach": (C.c_int, [P]),
        "tt_ctx_comm_info": (C.c_int, [P, C.POINTER(i32), C.POINTER(i32)]),
        "tt_plan_slice": (C.c_int, [i64, i32, i32, C.POINTER(i64), C.POINTER(i64)]),
        "tt_plan_lpt": (C.c_int, [i32, C.POINTER(dbl), i32, C.POINTER(i32)]),
        "tt_plan_gram_blocks": (C.c_int, [i32, i32, i32, i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
        "tt_ctx_round_hook": (C.c_int, [P, ROUND_HOOK_FN, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
