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


def rank_window_ok(gpu_ranks, cpu_info, slack_rel=1e-9):
    """Ranks must be identical unless the oracle's tail at the disputed rank lies within the
    documented window of tau."""
    if list(gpu_ranks) == list(cpu_info.ranks):
        return True
    for k, (g, c) in enumerate(zip(gpu_ranks[1:-1], cpu_info.ranks[1:-1])):
        if g == c:
            continue
        S = cpu_info.sigmas[k]
        lo = min(g, c)
        tail = np.sqrt(np.sum(S[lo:] ** 2))
        if abs(tail - cpu_info.tau) > slack_rel * cpu_info.tau + 64 * rounding.U_ROUND * cpu_info.scale:
            return False
    return True
