"""GPU checks of the library's sharded paths (include/tt_b200.h "multi-GPU"):
tt_gram by LPT pair blocks + all-gather, tt_orth with every driver dot batch split into slices +
all-gather, and the LPT-sharded phase-2 roundings of TT-Gram and
TT-Householder with ranks all-gathered and q_i broadcast from its owner.

* world 1 through the library's own NCCL communicator (one GPU in this pool): the NCCL calls
  themselves run (all-gather, grouped broadcasts) on the sharded code path;
* world 2 as two processes on the one GPU exchanging through the host (gloo, tt_comm_ops): the
  kernels of the two processes never wait on one another (every exchange is a host rendezvous),
  so this is the multi-rank data flow without a second GPU.

Each sharded result is compared with the same process's unsharded call: R and G to 1e-12
relative (the sharded dots differ from the unsharded ones only in the batching of the same
kernels), every q_i to 1e-10 s(q_i) through an exact oracle rounding of the difference, Table 1
counts and per-call ranks identical, and across the two ranks bitwise equality."""
import os
import socket

import numpy as np
import pytest

from oracle import tt
from ttinputs import make_shared_tail_set

from gpu_util import cuda_ok, diff_norm

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

KINDS = ["cgs", "mgs", "cgs2", "gram", "householder"]


def _set():
    return make_shared_tail_set(5, 6, 3, 9, 1e2, seed=7171)


def _compare(ctx_sh, ctx_ref, st, delta=1e-10):
    """Run tt_gram and tt_orth on both contexts; return the sharded results (host arrays)."""
    import paper_2211_08770_b200 as P
    out = {}
    A1 = [P.DeviceTT.from_numpy(a) for a in st.tensors]
    G1 = P.tt_gram(ctx_sh, A1).cpu().numpy()
    G0 = P.tt_gram(ctx_ref, A1).cpu().numpy()
    assert np.linalg.norm(G1 - G0) <= 1e-12 * np.linalg.norm(G0)
    assert np.array_equal(G1, G1.T)
    out["G"] = G1
    for kind in KINDS:
        Q1, R1, rep1 = P.tt_orth(ctx_sh, kind, A1, delta)
        Q0, R0, rep0 = P.tt_orth(ctx_ref, kind, A1, delta)
        assert rep1["rounding_calls"] == rep0["rounding_calls"], kind
        assert rep1["max_rank_per_call"] == rep0["max_rank_per_call"], kind
        assert np.linalg.norm(R1 - R0) <= 1e-12 * np.linalg.norm(R0), kind
        qs = [q.to_numpy() for q in Q1]
        for i, (q1, q0) in enumerate(zip(qs, Q0)):
            assert diff_norm(q1, q0.to_numpy()) <= 1e-10, (kind, i)
            assert abs(Q1[i].norm - q0.norm) <= 1e-12, (kind, i)
        out[kind] = (R1, qs)
    return out


def test_nccl_world1_sharded_paths():
    """The library-owned NCCL communicator at world size 1: tt_gram and all drivers take the
    sharded code path (NCCL all-gather and grouped broadcasts) and equal the plain calls."""
    import paper_2211_08770_b200 as P
    from paper_2211_08770_b200 import parallel
    c_sh, c_ref = P.Context(0), P.Context(0)
    parallel.attach_nccl(c_sh)
    assert parallel.comm_info(c_sh) == (1, 0)
    _compare(c_sh, c_ref, _set())
    parallel.detach(c_sh)
    assert parallel.comm_info(c_sh) == (1, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2211_08770_b200 as P
        from paper_2211_08770_b200 import parallel
        c_sh, c_ref = P.Context(0), P.Context(0)
        parallel.attach_host(c_sh)
        assert parallel.comm_info(c_sh) == (world, rank)
        out = _compare(c_sh, c_ref, _set())
        q.put((rank, None, {k: (v if k == "G" else (v[0], [np.concatenate([c.ravel() for c in x]) for x in v[1]]))
                            for k, v in out.items()}))
    except Exception as e:  # noqa: BLE001 -- report instead of hanging the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


def test_host_comm_world2_sharded_paths():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    for rank, err, _ in res:
        assert err is None, err
    a, b = res[0][2], res[1][2]
    assert np.array_equal(a["G"], b["G"])
    for kind in KINDS:
        assert np.array_equal(a[kind][0], b[kind][0]), kind
        for x, y in zip(a[kind][1], b[kind][1]):
            assert np.array_equal(x, y), kind
