"""One driver run on a BASELINE config prefix, for TT_B200_RR_DEBUG / ncu captures.

  CONFIG=C3 DRIVER=cgs2 CGS2_M=8 python tools/cgs2_dbg.py
"""
import os
import sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2211_08770_b200 as P
from ttinputs import CONFIGS, make_shared_tail_set
c = CONFIGS[os.environ.get("CONFIG", "C3")]
st = make_shared_tail_set(c.d, c.n, c.r, int(os.environ.get("CGS2_M", "8")), c.kappa, c.seed)
ctx = P.Context(0)
A = [P.DeviceTT.from_numpy(a) for a in st.tensors]
Q, R, rep = P.tt_orth(ctx, os.environ.get("DRIVER", "cgs2"), A, c.delta)
print(rep["max_rank_per_call"])
