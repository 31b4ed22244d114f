import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2211_08770_b200 as P
from ttinputs import make_batch_sums_stacked
ctx = P.Context(0)
B = 4096
cores, coeffs = make_batch_sums_stacked(B)
host = [[torch.from_numpy(c).pin_memory() for c in term] for term in cores]
norms = np.ones((B, 4))
dev = [[h.cuda() for h in term] for term in host]
half = [[x[:2048] for x in term] for term in dev]
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(ctx.stream); return e
for it in range(3):
    torch.cuda.synchronize()
    e0 = ev()
    with torch.cuda.stream(ctx.stream):
        for term_d, term_h in zip(dev, host):
            for d_, h_ in zip(term_d, term_h):
                d_[:2048].copy_(h_[:2048], non_blocking=True)
    e1 = ev()
    r = P.tt_round_batch_strided(ctx, half, coeffs[:2048], 1e-6, norms=norms[:2048])
    e2 = ev()
    r2 = P.tt_round_batch_strided(ctx, dev, coeffs, 1e-6, norms=norms)
    e3 = ev()
    torch.cuda.synchronize()
    print(f"h2d half {e0.elapsed_time(e1):.1f} ms, round 2048 {e1.elapsed_time(e2):.1f} ms, round 4096 {e2.elapsed_time(e3):.1f} ms")
    del r, r2
out = None
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, rk, nr, cnt = P.tt_round_batch_host(ctx, host, coeffs, 1e-6, norms=norms, chunks=2, out_host=out)
    print(f"host call {1e3*(time.perf_counter()-t0):.1f} ms")
