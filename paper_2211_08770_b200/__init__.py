"""B200-native hot path of arXiv 2211.08770 (TT-format orthogonalization).

TT-rounding of rank-inflated TT-sums, batched TT inner products / Gram matrices and the
six orthogonalization drivers (CGS, MGS, CGS2, MGS2, Gram, Householder), implemented as
hand-written sm_100a CUDA behind the C ABI of include/tt_b200.h.  This package is the
binding (argument marshalling) plus the multi-GPU sharding helpers; it never imports the
CPU oracle and has no CPU fallback.
"""
from . import _native  # noqa: F401
from .api import (  # noqa: F401
    DEFAULT_FLOOR_C,
    BatchTT,
    Context,
    DeviceTT,
    LibTT,
    RoundTrace,
    compression_gain,
    compression_ratio,
    krylov_set,
    laplacian_cores,
    storage_count,
    ttm_device,
    tt_dot_batch,
    tt_element,
    tt_gram,
    tt_gram_blocks,
    tt_matvec,
    tt_norm,
    tt_orth,
    tt_round,
    tt_round_batch,
    tt_round_batch_host,
    tt_round_batch_strided,
    tt_sum,
)
