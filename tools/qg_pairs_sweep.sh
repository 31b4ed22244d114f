for pp in 1 0.5 0.25; do
  echo "pairs_per_warp=$pp"
  TT_B200_QG_PAIRS=$pp CONFIG=C5 DRIVER=householder CGS2_M=20 python - <<'PY'
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2211_08770_b200 as P
from ttinputs import CONFIGS, make_shared_tail_set
c = CONFIGS["C5"]
st = make_shared_tail_set(c.d, c.n, c.r, 20, c.kappa, c.seed)
ctx = P.Context(0)
A = [P.DeviceTT.from_numpy(a) for a in st.tensors]
P.tt_orth(ctx, "householder", A[:3], c.delta)
ctx.profile(True)
t0 = time.time()
P.tt_orth(ctx, "householder", A, c.delta)
torch.cuda.synchronize()
rep = ctx.profile_report()
print("wall %.2f s" % (time.time() - t0), {k: round(v["ms"], 1) for k, v in rep.items() if k.startswith("qrcp")})
PY
done
