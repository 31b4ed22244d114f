import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_2211_08770_b200 as P
from ttinputs import make_batch_sums_stacked
B=4096
cores, coeffs = make_batch_sums_stacked(B)
ctx = P.Context(0)
host = [[torch.from_numpy(c).pin_memory() for c in term] for term in cores]
norms = np.ones((B,4))
dc = [[x.cuda() for x in term] for term in host]
res = P.tt_round_batch_strided(ctx, dc, coeffs, 1e-6, norms=norms); n = res.total_doubles(); del res
out = torch.empty(n + 4096, dtype=torch.float64).pin_memory()
torch.cuda.synchronize()
for chunks in (1, 2, 4, 8):
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out, rk, nr, cnt = P.tt_round_batch_host(ctx, host, coeffs, 1e-6, norms=norms, chunks=chunks, out_host=out)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"chunks={chunks} wall {1e3*(t1-t0):.1f} ms", flush=True)
# raw copy speeds
torch.cuda.synchronize(); t0=time.perf_counter()
d2 = [[x.to('cuda', non_blocking=True) for x in term] for term in host]; torch.cuda.synchronize(); t1=time.perf_counter()
print(f"H2D 8.7GB {1e3*(t1-t0):.1f} ms")
g = torch.empty(n, dtype=torch.float64, device='cuda'); torch.cuda.synchronize(); t0=time.perf_counter()
out[:n].copy_(g, non_blocking=True); torch.cuda.synchronize(); t1=time.perf_counter()
print(f"D2H {n*8/1e9:.1f}GB {1e3*(t1-t0):.1f} ms")
torch.cuda.synchronize(); t0=time.perf_counter()
res = P.tt_round_batch_strided(ctx, dc, coeffs, 1e-6, norms=norms); torch.cuda.synchronize(); t1=time.perf_counter()
print(f"compute only {1e3*(t1-t0):.1f} ms")
