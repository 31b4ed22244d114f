"""Helpers for the GPU parity tests (call the CUDA path through the C ABI binding)."""
import numpy as np
import pytest

from oracle import rounding, tt


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


_CTX = None


def ctx():
    global _CTX
    if _CTX is None:
        from paper_2211_08770_b200 import _build
        _build.build_library()
        import paper_2211_08770_b200 as P
        _CTX = P.Context(0)
    return _CTX


def dev(cores, norm=float("nan")):
    import paper_2211_08770_b200 as P
    return P.DeviceTT.from_numpy(cores, norm=norm)


def diff_norm(x, y):
    """||x - y|| through an exact (delta = 0) oracle rounding of the difference (sweep norm).
    Never sqrt(<a,a> - 2<a,b> + <b,b>)."""
    _, info = rounding.tt_round(tt.tt_sum([x, y], [1.0, -1.0]), 0.0)
    return info.norm


# Window hits accepted by rank_window_ok across the session: (test id, split, gpu rank,
# oracle rank, |tail - tau| / window).  conftest.py prints them at the end of the run.
WINDOW_HITS = []
WINDOW_CHECKS = [0]


def window(cpu_info, floor_c):
    """ranks may differ only at a split where some rho between the two
    choices has |tail_rho - tau| <= 1e-12 tau + c_floor u s(x) (the second term is the fp
    resolution of singular values after cancellation; c_floor = the run's floor constant, 64 --
    SURVEY A12's starting value -- for paper-pure runs with the floor off)."""
    c = floor_c if floor_c > 0.0 else 64.0
    return 1e-12 * cpu_info.tau + c * rounding.U_ROUND * cpu_info.scale


def rank_window_ok(gpu_ranks, cpu_info, floor_c=rounding.DEFAULT_FLOOR_C, tag=""):
    """Ranks identical, or every disputed split inside the C6 window (each hit recorded)."""
    WINDOW_CHECKS[0] += 1
    if list(gpu_ranks) == list(cpu_info.ranks):
        return True
    win = window(cpu_info, floor_c)
    hits = []
    for k, (g, c) in enumerate(zip(gpu_ranks[1:-1], cpu_info.ranks[1:-1])):
        if g == c:
            continue
        S = cpu_info.sigmas[k]
        lo, hi = min(g, c), max(g, c)
        # some rho in [lo, hi] must have its tail within the window of tau
        gaps = [abs(np.sqrt(np.sum(S[rho:] ** 2)) - cpu_info.tau) for rho in range(lo, hi + 1)]
        if min(gaps) > win:
            return False
        hits.append((tag, k + 1, g, c, min(gaps) / win))
    WINDOW_HITS.extend(hits)
    return True


def assert_round_parity(g, gpu_ranks, terms, coeffs, delta, floor_c, norms, info=None, ref=None,
                        max_rank=None, tol=1e-10, tag=""):
    """The kernel-level TT-round parity of SURVEY C6 item 1 on one rounding: ranks identical or
    inside the window; reconstruction within tol s(x) of the oracle's -- where ranks differ, of
    the oracle's rounding truncated to the GPU's ranks (same per-split rank; force_ranks)."""
    if info is None:
        ref, info = rounding.tt_round_sum(terms, coeffs, delta, floor_c=floor_c, term_norms=norms,
                                          max_rank=max_rank)
    assert rank_window_ok(gpu_ranks, info, floor_c, tag), (tag, list(gpu_ranks), info.ranks)
    if list(gpu_ranks) != list(info.ranks):
        ref, _ = rounding.tt_round_sum(terms, coeffs, delta, floor_c=floor_c, term_norms=norms,
                                       max_rank=max_rank, force_ranks=list(gpu_ranks))
    dn = diff_norm(g, ref)
    assert dn <= tol * info.scale, (tag, dn, info.scale)
    return info
