"""Development aid: one wide-block solve (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14471_b200 import api, synth  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 100
p = synth.random_sur(64, 100000, [nb] * 64, seed=3)
sur = api.sur_from_problem(p)
op = api.sur_preconditioner(sur)
api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=1e-14, max_iter=6, diag_every=0, xv_mode="qr"), want_trace=False)
