"""Multi-process (gloo, world size 2, CPU) tests of the sharding logic in parallel.py.

The block values are computed with the oracle's TT-dot here (the GPU path computes them
with tt_gram_blocks); what is under test is partition + all-gather + unpack."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_08770_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_blocks_cover_lower_triangle_once():
    for m, b in [(1, 5), (7, 3), (50, 5), (13, 13)]:
        cover = np.zeros((m, m), int)
        for i0, j0, bi, bj in parallel.gram_pair_blocks(m, b):
            cover[i0:i0 + bi, j0:j0 + bj] += 1
        lower = np.tril(np.ones((m, m), int))
        assert np.all(cover[lower == 1] == 1)


def test_lpt_balance():
    blocks = parallel.gram_pair_blocks(50, 5)
    parts = parallel.assign_blocks(blocks, 8)
    loads = [sum(bi * bj for _, _, bi, bj in p) for p in parts]
    assert sum(loads) == sum(bi * bj for _, _, bi, bj in blocks)
    assert max(loads) - min(loads) <= 25
    assert sorted(b for p in parts for b in p) == sorted(blocks)


def test_dot_slices():
    for P, W in [(49, 8), (1, 2), (0, 3), (5, 5)]:
        sl = [parallel.dot_slice(P, W, r) for r in range(W)]
        assert sl[0][0] == 0 and sl[-1][1] == P and sum(e - s for s, e in sl) == P


def test_batch_slices():
    for B, W in [(4096, 8), (10, 3), (2, 4)]:
        sl = [parallel.batch_slice(B, W, r) for r in range(W)]
        assert sl[0][0] == 0 and sl[-1][1] == B
        assert all(sl[r][1] == sl[r + 1][0] for r in range(W - 1))
        assert max(e - s for s, e in sl) - min(e - s for s, e in sl) <= 1


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import orth, tt
        from ttinputs import make_shared_tail_set
        st = make_shared_tail_set(3, 5, 2, 9, 100.0, seed=42)
        A = st.tensors

        def block_fn(blocks):
            vals = []
            for i0, j0, bi, bj in blocks:
                for s in range(bi):
                    for t in range(bj):
                        vals.append(tt.tt_dot(A[i0 + s], A[j0 + t]))
            return torch.tensor(vals, dtype=torch.float64)

        G = parallel.sharded_gram(9, block_fn, block=2)
        ref = orth.gram_matrix(A)
        ok_gram = float(np.max(np.abs(G - ref)))

        class R:
            def __init__(self, ranks):
                self.ranks = ranks
        items = list(range(7))
        outs, ranks = parallel.sharded_round_batch(items, lambda xs: [R([1, x, 1]) for x in xs])
        # CGS projection dots <a_8, a_j>, j < 8, split over the ranks and all-gathered
        dots = parallel.sharded_dots(8, lambda s, e: torch.tensor([tt.tt_dot(A[8], A[j]) for j in range(s, e)],
                                                                  dtype=torch.float64))
        ok_dots = float(np.max(np.abs(dots - np.array([tt.tt_dot(A[8], A[j]) for j in range(8)]))))
        # fewer dots than ranks (P = 1): the idle rank contributes an empty slice
        one = parallel.sharded_dots(1, lambda s, e: torch.tensor([tt.tt_dot(A[1], A[0])], dtype=torch.float64))
        ok_dots = max(ok_dots, float(abs(one[0] - tt.tt_dot(A[1], A[0]))) if len(one) == 1 else 1.0)
        q.put((rank, max(ok_gram, ok_dots), ranks))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_gram_and_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, ranks in res:
        assert not isinstance(err, str), err
        assert err <= 1e-15
        assert ranks == [[1, x, 1] for x in range(7)]
