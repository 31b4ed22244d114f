"""Seeded synthetic TT inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the paper's method (no TT-rounding, TT-dot, TT-sum,
Gram-Schmidt or Householder step).  It only draws Gaussian numbers from a fixed
``numpy.random.Generator(PCG64(seed))`` in a fixed order and builds inputs whose exact
answers follow from the construction.
"""
from .generate import (  # noqa: F401
    CONFIGS,
    ConfigSpec,
    SharedTailSet,
    config_spec,
    make_shared_tail_set,
    make_batch_sums,
    make_batch_sums_stacked,
    make_fuzz_batch,
    make_random_tt,
    tt_ranks_capped,
)
