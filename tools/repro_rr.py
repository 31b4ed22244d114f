"""Replay the roundings of an oracle driver run on the GPU with and without the
rank-revealing right-to-left sweep (debugging aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2211_08770_b200 as P  # noqa: E402
from oracle import orth  # noqa: E402
from ttinputs import CONFIGS, make_shared_tail_set  # noqa: E402
from gpu_util import dev, diff_norm  # noqa: E402

cfg, kind, m = sys.argv[1], sys.argv[2], int(sys.argv[3])
c = CONFIGS[cfg]
st = make_shared_tail_set(c.d, c.n, c.r, m, c.kappa, c.seed)
ref = orth.orth(kind, st.tensors, c.delta)
ctx = P.Context(0)
for t, (terms, coefs, norms) in enumerate(zip(ref.terms, ref.coeffs, ref.term_norms)):
    info = ref.infos[t]
    row = [t, len(terms), max(info.formal_ranks), max(info.ranks)]
    for rr in (True, False):
        out, gi = P.tt_round(ctx, [dev(x, nr) for x, nr in zip(terms, norms)], list(coefs), c.delta,
                             rank_revealing=rr)
        dn = diff_norm(out.to_numpy(), ref.outputs[t]) / info.scale if out.ranks == info.ranks else float("nan")
        row += [max(out.ranks), f"{(gi['norm'] - info.norm) / info.scale:.2e}", f"{dn:.2e}"]
    print(*row)
