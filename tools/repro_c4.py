"""Round one C4 item (4 unit-norm TTs, d=10, n=32, r=16) on the GPU; used for debugging."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2211_08770_b200 as P  # noqa: E402
from ttinputs import make_batch_sums  # noqa: E402

items = make_batch_sums(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
ctx = P.Context(0)
for terms, coeffs in items:
    out, info = P.tt_round(ctx, [P.DeviceTT.from_numpy(t, norm=1.0) for t in terms], coeffs, 1e-6)
    print(out.ranks, info)
