"""Host-side multi-GPU logic (CPU, no GPU): the library's shard plans (tt_plan_*, C host code) and
the host-exchanged collectives of parallel.HostCollectives at world size 2 over gloo.

The device paths that use them (sharded tt_gram, driver dot slices, LPT phase-2 roundings) are
checked on the GPU in tests/test_gpu_comm.py."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_08770_b200 import parallel


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2211_08770_b200 import _build
    _build.build_library()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gram_blocks_cover_lower_triangle_once():
    for m, b in [(1, 5), (7, 3), (50, 4), (50, 5), (13, 13)]:
        blocks, owners = parallel.plan_gram_blocks(m, b, 3)
        cover = np.zeros((m, m), int)
        for i0, j0, bi, bj in blocks:
            assert j0 <= i0
            cover[i0:i0 + bi, j0:j0 + bj] += 1
        lower = np.tril(np.ones((m, m), int))
        assert np.all(cover[lower == 1] == 1)
        assert set(owners) <= {0, 1, 2}


def test_lpt_balance_and_determinism():
    blocks, owners = parallel.plan_gram_blocks(50, 4, 8)
    loads = np.zeros(8)
    for (i0, j0, bi, bj), o in zip(blocks, owners):
        loads[o] += bi * bj
    assert loads.sum() == sum(bi * bj for _, _, bi, bj in blocks)
    assert loads.max() - loads.min() <= 16  # one block's worth
    # LPT on increasing costs (Householder phase 2: rounding cost grows like (31 i)^3)
    cost = [float((31 * i) ** 3) for i in range(1, 101)]
    own = parallel.plan_lpt(cost, 8)
    per = np.zeros(8)
    for c, o in zip(cost, own):
        per[o] += c
    assert per.max() <= sum(cost) / 8 + max(cost)  # Graham's LPT bound (list-scheduling form)
    assert per.max() / per.mean() < 1.02
    assert own == parallel.plan_lpt(cost, 8)  # deterministic: every rank derives the same map
    # ties keep index order: equal costs are dealt round-robin
    assert parallel.plan_lpt([1.0] * 5, 2) == [0, 1, 0, 1, 0]
    assert parallel.plan_lpt([], 4) == []


def test_slices():
    for P, W in [(4096, 8), (49, 8), (10, 3), (2, 4), (0, 3), (5, 5)]:
        sl = [parallel.plan_slice(P, W, r) for r in range(W)]
        assert sl[0][0] == 0 and sl[-1][1] == P
        assert all(sl[r][1] == sl[r + 1][0] for r in range(W - 1))
        assert max(e - s for s, e in sl) - min(e - s for s, e in sl) <= 1


def test_plan_errors():
    from paper_2211_08770_b200 import _native as N
    with pytest.raises(N.TTError):
        parallel.plan_slice(5, 2, 2)
    lib = N.load()
    nb = ctypes.c_int32()
    blk = (ctypes.c_int32 * 4)()
    own = (ctypes.c_int32 * 1)()
    assert lib.tt_plan_gram_blocks(9, 3, 2, 1, blk, own, ctypes.byref(nb)) == 1  # cap too small
    assert nb.value == 6


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hc = parallel.HostCollectives(None, device="cpu")
        # all-gather through the C callback signature (host buffers stand in for device ones)
        send = (ctypes.c_double * 3)(*[10.0 * rank + k for k in range(3)])
        recv = (ctypes.c_double * (3 * world))()
        rc1 = hc.ops.allgather(None, ctypes.addressof(send), ctypes.addressof(recv), 24, None)
        gathered = list(recv)
        # broadcast from rank 1
        buf = (ctypes.c_double * 2)(*([7.0, 8.0] if rank == 1 else [0.0, 0.0]))
        rc2 = hc.ops.broadcast(None, ctypes.addressof(buf), 16, 1, None)
        # every rank derives the same plans
        blocks, owners = parallel.plan_gram_blocks(23, 4, world)
        mine = [b for b, o in zip(blocks, owners) if o == rank]
        q.put((rank, rc1, rc2, gathered, list(buf), mine, owners))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None, None, None, None, None))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_collectives_and_plans():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rc1, rc2, gathered, buf, mine, owners in res:
        assert rc1 == 0, rc1
        assert rc2 == 0
        assert gathered == [0.0, 1.0, 2.0, 10.0, 11.0, 12.0]
        assert buf == [7.0, 8.0]
    assert res[0][6] == res[1][6]
    cover = np.zeros((23, 23), int)
    for r in res:
        for i0, j0, bi, bj in r[5]:
            cover[i0:i0 + bi, j0:j0 + bj] += 1
    assert np.all(cover[np.tril(np.ones((23, 23), int)) == 1] == 1)
