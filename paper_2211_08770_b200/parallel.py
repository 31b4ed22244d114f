"""Multi-GPU plumbing for the naturally sharded parts of the hot path.

Everything that computes lives in the library (include/tt_b200.h, csrc/comm.cu): a context holds a
communicator, and with one attached ``tt_gram`` splits the Gram pair blocks by LPT and all-gathers
them, ``tt_orth`` splits every driver dot batch (projection coefficients, Gram rows) into slices and
all-gathers them, and shards the independent phase-2 roundings of TT-Gram / TT-Householder by LPT
(owner rounds, ranks all-gathered, q_i broadcast).  Batches of independent roundings need no
communicator: rank r rounds ``plan_slice(B, world, r)``.  A single rounding sweep never shards.

This module only attaches communicators and exposes the library's shard plans:
* ``attach_nccl`` -- the library-owned NCCL communicator (the 128-byte unique id travels over the
  torch.distributed process group, the one out-of-band channel the launcher provides);
* ``attach_host`` -- caller-supplied collectives that exchange through the host over a
  torch.distributed group (gloo): lets several processes share one GPU in the tests, since their
  kernels never wait on one another (every exchange is a host-side rendezvous).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

from . import _native as N

Block = Tuple[int, int, int, int]  # (i0, j0, bi, bj)


# ----------------------------------------------------------------------------- shard plans (host)
def plan_slice(P: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced slice [start, end) of P independent items for `rank` (tt_plan_slice)."""
    lib = N.load()
    s, e = C.c_int64(), C.c_int64()
    st = lib.tt_plan_slice(int(P), int(world), int(rank), C.byref(s), C.byref(e))
    if st != 0:
        raise N.TTError(st, "tt_plan_slice")
    return s.value, e.value


batch_slice = plan_slice


def plan_lpt(costs: Sequence[float], world: int) -> List[int]:
    """Owner rank of each item by longest-processing-time on `costs` (tt_plan_lpt)."""
    lib = N.load()
    P = len(costs)
    cost = (C.c_double * max(P, 1))(*[float(c) for c in costs])
    own = (C.c_int32 * max(P, 1))()
    st = lib.tt_plan_lpt(P, cost, int(world), own)
    if st != 0:
        raise N.TTError(st, "tt_plan_lpt")
    return list(own[:P])


def plan_gram_blocks(m: int, b: int, world: int) -> Tuple[List[Block], List[int]]:
    """The pair blocks of an m x m Gram matrix and their LPT owners (tt_plan_gram_blocks)."""
    lib = N.load()
    nb = C.c_int32()
    st = lib.tt_plan_gram_blocks(int(m), int(b), int(world), 0, None, None, C.byref(nb))
    if st != 0:
        raise N.TTError(st, "tt_plan_gram_blocks")
    blk = (C.c_int32 * (4 * nb.value))()
    own = (C.c_int32 * nb.value)()
    st = lib.tt_plan_gram_blocks(int(m), int(b), int(world), nb.value, blk, own, C.byref(nb))
    if st != 0:
        raise N.TTError(st, "tt_plan_gram_blocks")
    return [tuple(blk[4 * q:4 * q + 4]) for q in range(nb.value)], list(own)


# ----------------------------------------------------------------------------- communicators
def _world(group=None):
    import torch.distributed as dist
    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def attach_nccl(ctx, group=None) -> None:
    """Attach the library's own NCCL communicator over the ranks of `group` (collective)."""
    import torch.distributed as dist
    world, rank = _world(group)
    lib = ctx.lib
    idbuf = (C.c_uint8 * N.COMM_ID_BYTES)()
    if rank == 0:
        ctx.check(lib.tt_comm_nccl_id(idbuf))
    if world > 1:
        obj = [bytes(idbuf) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        idbuf = (C.c_uint8 * N.COMM_ID_BYTES).from_buffer_copy(obj[0])
    ctx.check(lib.tt_ctx_comm_nccl(ctx.handle, world, rank, idbuf))


class HostCollectives:
    """tt_comm_ops over a torch.distributed group: device bytes are copied to the host, exchanged
    with the group's backend (gloo) and copied back.  `device` is where the library's buffers
    live ("cuda:k" in the library; "cpu" when the callbacks are exercised on their own)."""

    def __init__(self, group=None, device: str = "cuda"):
        self.group = group
        self.device = device
        self._ag = N.ALLGATHER_FN(self._allgather)
        self._bc = N.BROADCAST_FN(self._broadcast)
        self.ops = N.CommOps(self._ag, self._bc, None)

    def _tensor(self, ptr: int, nbytes: int):
        import torch
        if self.device == "cpu":
            buf = (C.c_uint8 * nbytes).from_address(ptr)
            return torch.frombuffer(buf, dtype=torch.uint8, count=nbytes) if nbytes else torch.empty(0, dtype=torch.uint8)

        class _Arr:
            pass
        a = _Arr()
        a.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                      "strides": None, "stream": None}
        return torch.as_tensor(a, device=self.device)

    def _allgather(self, user, send, recv, nbytes, stream) -> int:
        try:
            import torch
            import torch.distributed as dist
            world, _ = _world(self.group)
            src = self._tensor(send, nbytes).cpu()
            out = torch.empty(world * nbytes, dtype=torch.uint8)
            dist.all_gather_into_tensor(out, src, group=self.group)
            self._tensor(recv, world * nbytes).copy_(out)
            if self.device != "cpu":
                torch.cuda.synchronize(self.device)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    def _broadcast(self, user, buf, nbytes, root, stream) -> int:
        try:
            import torch
            import torch.distributed as dist
            t = self._tensor(buf, nbytes).cpu()
            src = dist.get_global_rank(self.group, root) if self.group is not None else root
            dist.broadcast(t, src=src, group=self.group)
            self._tensor(buf, nbytes).copy_(t)
            if self.device != "cpu":
                torch.cuda.synchronize(self.device)
            return 0
        except Exception:  # noqa: BLE001
            return 1


def attach_host(ctx, group=None) -> HostCollectives:
    """Attach host-exchanged collectives over `group` (keep the returned object alive while
    attached: it owns the callbacks)."""
    world, rank = _world(group)
    hc = HostCollectives(group, device=f"cuda:{ctx.device}")
    ctx.check(ctx.lib.tt_ctx_comm_ops(ctx.handle, world, rank, C.byref(hc.ops)))
    ctx._host_collectives = hc
    return hc


def detach(ctx) -> None:
    ctx.check(ctx.lib.tt_ctx_comm_detach(ctx.handle))
    ctx._host_collectives = None


def comm_info(ctx) -> Tuple[int, int]:
    nr, rk = C.c_int32(), C.c_int32()
    ctx.check(ctx.lib.tt_ctx_comm_info(ctx.handle, C.byref(nr), C.byref(rk)))
    return nr.value, rk.value
