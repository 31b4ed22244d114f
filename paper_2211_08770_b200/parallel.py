"""Multi-GPU sharding of the naturally parallel parts of the hot path.

* Gram matrix (Alg. 5 lines 2-6): the lower triangle of pair indices is tiled into b x b
  pair blocks, blocks are assigned to ranks by longest-processing-time (pair counts), each
  rank evaluates its blocks with ``tt_gram_blocks`` (one launch of the TT-dot kernel), the
  packed results are exchanged with ONE all-gather (NCCL over NVLink on GPUs), every rank
  unpacks the symmetric matrix.
* Batches of independent roundings (C4): contiguous slices per rank, no collective on the
  data path; only the rank metadata is all-gathered.

A single rounding sweep and the MGS / Householder step chains never shard (north star).
The partition / pack / unpack logic is pure Python so it is testable with gloo on CPU.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np

Block = Tuple[int, int, int, int]  # (i0, j0, bi, bj)


def gram_pair_blocks(m: int, b: int) -> List[Block]:
    """Blocks covering every pair (i, j) with i >= j (diagonal blocks are full squares)."""
    out = []
    for I in range(0, m, b):
        for J in range(0, I + 1, b):
            out.append((I, J, min(b, m - I), min(b, m - J)))
    return out


def assign_blocks(blocks: Sequence[Block], world: int) -> List[List[Block]]:
    """Greedy LPT assignment by pair count (bi * bj); deterministic."""
    order = sorted(range(len(blocks)), key=lambda k: (-blocks[k][2] * blocks[k][3], k))
    load = [0] * world
    parts: List[List[Block]] = [[] for _ in range(world)]
    for k in order:
        r = min(range(world), key=lambda q: (load[q], q))
        parts[r].append(blocks[k])
        load[r] += blocks[k][2] * blocks[k][3]
    for p in parts:
        p.sort()
    return parts


def unpack_blocks(m: int, parts: Sequence[Sequence[Block]], packed: Sequence[np.ndarray]) -> np.ndarray:
    """Assemble the symmetric m x m Gram matrix from every rank's packed block values."""
    G = np.zeros((m, m))
    for blocks, buf in zip(parts, packed):
        o = 0
        for i0, j0, bi, bj in blocks:
            blk = np.asarray(buf[o:o + bi * bj]).reshape(bi, bj)
            o += bi * bj
            G[i0:i0 + bi, j0:j0 + bj] = blk
            G[j0:j0 + bj, i0:i0 + bi] = blk.T
    return G


def sharded_gram(m: int, block_fn: Callable[[List[Block]], "object"], block: int = 5, group=None):
    """Gram matrix sharded over the ranks of ``group`` (torch.distributed).

    block_fn(blocks) returns this rank's packed values (a 1-D torch tensor on the rank's
    device, e.g. ``tt_gram_blocks``).  One all_gather of equal-sized (padded) buffers."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    parts = assign_blocks(gram_pair_blocks(m, block), world)
    mine = block_fn(parts[rank])
    sizes = [sum(bi * bj for _, _, bi, bj in p) for p in parts]
    cap = max(sizes)
    buf = torch.zeros(cap, dtype=torch.float64, device=mine.device)
    buf[: mine.numel()] = mine
    if world > 1:
        out = torch.empty(world * cap, dtype=torch.float64, device=mine.device)
        dist.all_gather_into_tensor(out, buf, group=group)
        allbuf = out.cpu().numpy().reshape(world, cap)
    else:
        allbuf = buf.cpu().numpy().reshape(1, cap)
    return unpack_blocks(m, parts, [allbuf[r, : sizes[r]] for r in range(world)])


def batch_slice(B: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous slice [start, end) of B independent items for `rank` (balanced)."""
    base, rem = divmod(B, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def sharded_round_batch(items, round_fn: Callable, group=None):
    """Round this rank's slice of independent TT-sums; all-gather the output ranks (metadata
    only).  Returns (my results, [ranks of every item in global order])."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    s, e = batch_slice(len(items), world, rank)
    outs = round_fn(items[s:e])
    d1 = len(outs[0].ranks) if outs else 0
    mine = torch.tensor([r for o in outs for r in o.ranks], dtype=torch.int64)
    if world > 1:
        d1 = max(d1, 1)
        cap = (len(items) // world + 1) * d1
        buf = torch.zeros(cap, dtype=torch.int64)
        buf[: mine.numel()] = mine
        dev = "cuda" if (dist.get_backend(group) == "nccl") else "cpu"
        buf = buf.to(dev)
        out = torch.empty(world * cap, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(out, buf, group=group)
        out = out.cpu().numpy().reshape(world, cap)
        ranks = []
        for r in range(world):
            a, b = batch_slice(len(items), world, r)
            ranks += [list(out[r, k * d1:(k + 1) * d1]) for k in range(b - a)]
    else:
        ranks = [list(o.ranks) for o in outs]
    return outs, ranks


def dot_slice(P: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous slice [start, end) of a batch of P dot products for `rank`."""
    return batch_slice(P, world, rank)


def sharded_dots(P: int, dot_fn: Callable[[int, int], "object"], group=None) -> np.ndarray:
    """A batch of P TT-dots split over the ranks of ``group``: rank r evaluates the contiguous
    slice dot_slice(P, world, r) with dot_fn(start, end) (a 1-D float64 torch tensor on the
    rank's device, e.g. ``tt_dot_batch`` of those pairs), ONE all-gather of equal-sized
    (padded) buffers, every rank returns all P values in order (north star: "CGS projection
    dot products are split ... and combined with NCCL all-gather")."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if P == 0:
        return np.zeros(0)
    s, e = dot_slice(P, world, rank)
    mine = dot_fn(s, e) if e > s else None
    cap = -(-P // world)
    dev = mine.device if mine is not None else ("cuda" if dist.is_initialized() and dist.get_backend(group) == "nccl"
                                                 else "cpu")
    buf = torch.zeros(cap, dtype=torch.float64, device=dev)
    if mine is not None:
        buf[: e - s] = mine
    if world > 1:
        out = torch.empty(world * cap, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(out, buf, group=group)
        allbuf = out.cpu().numpy().reshape(world, cap)
    else:
        allbuf = buf.cpu().numpy().reshape(1, cap)
    vals = []
    for r in range(world):
        a, b = dot_slice(P, world, r)
        vals.append(allbuf[r, : b - a])
    return np.concatenate(vals)


def cgs_sharded(ctx, kind: str, A, delta: float, floor_c: float = None, group=None):
    """TT-CGS / TT-CGS2 (PAPER.md Algs. 1 and 3) with the projection dots of every step split
    over the ranks (sharded_dots + one all-gather per pass); the roundings are replicated on
    every rank (deterministic: identical results everywhere).  Same schedule as tt_orth's
    lazy drivers: per pass the coefficients c_j = <p, q_j> (j < i), R(j, i) += c_j, then
    p = round(p - sum_j c_j q_j); R(i, i) = ||p||, q_i = p / R(i, i).  Returns (Q, R, calls)."""
    from . import api as P

    if kind not in ("cgs", "cgs2"):
        raise ValueError("cgs_sharded: kind must be 'cgs' or 'cgs2'")
    fc = P.DEFAULT_FLOOR_C if floor_c is None else floor_c
    passes = 2 if kind == "cgs2" else 1
    m = len(A)
    R = np.zeros((m, m))
    Q = []
    calls = 0
    for i in range(m):
        base = A[i]
        for _ in range(passes):
            if i > 0:
                fn = lambda s, e: P.tt_dot_batch(ctx, [base] * (e - s), Q[s:e])  # noqa: E731
                c = sharded_dots(i, fn, group)
            else:
                c = np.zeros(0)
            R[:i, i] += c
            base, _ = P.tt_round(ctx, [base] + Q, [1.0] + [-float(v) for v in c], delta, floor_c=fc)
            calls += 1
        nrm = P.tt_norm(ctx, base)
        R[i, i] = nrm
        q = P.tt_sum(ctx, [base], [1.0 / nrm])
        Q.append(q)
    return Q, R, calls
