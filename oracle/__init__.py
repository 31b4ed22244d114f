"""CPU fp64 ORACLE for the TT-orthogonalization hot path of arXiv 2211.08770.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or execute this
package.  The product path (``paper_2211_08770_b200``) never imports it and fails loudly
when its CUDA library is missing.

Plain, slow, obviously-correct numpy code written from the paper (PAPER.md, cited per
function as ``PAPER.md:<line>`` with the section / algorithm / equation).  LAPACK
routines (``numpy.linalg.qr`` = Householder QR, ``numpy.linalg.svd``) serve as single
steps; nothing is blocked, fused or reordered beyond the paper's listings.  Where the
paper is silent or garbled the reading of SURVEY.md §8(c) is taken; every reading is
listed in DESIGN.md ("Readings of the paper").

The oracle shares no code with the CUDA path; only ``ttinputs`` (seeded input draws,
none of the method's arithmetic) serves both.

Parity pins (tests/test_oracle_*.py, marker "not gpu") fix every function below against
something other than itself; see DESIGN.md "Oracle pins".  Functions with no pin:
none are left unpinned; LOO values in noise-dominated regimes (CGS/Gram at u*kappa^2 >~ 1)
have no closed form and are only checked for their order of magnitude ("parity unpinned"
for those values, SURVEY.md §8(c) C5 last row).
"""
from . import tt, dense, rounding, orth, metrics  # noqa: F401
