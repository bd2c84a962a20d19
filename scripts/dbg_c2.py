"""Debug aid: c2 (singular Omega) GPU vs oracle -- stop iteration, b distance, growth margins."""
import numpy as np
import oracle
from paper_2510_14471_b200 import api, synth

p = synth.make_problem(2, M=1000)
o = oracle.solve(p, "oracle", cfg=oracle.make_config(tol_rel=p.tol_rel, max_iter=p.max_iter))
for mode in ("x", "qr"):
    sur = api.sur_from_problem(p)
    op = api.sur_preconditioner(sur)
    g = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=p.tol_rel, max_iter=p.max_iter, xv_mode=mode, diag_every=1))
    cg = np.asarray(g.trace.rows["c"]); co = np.asarray(o.trace["c"])
    print(mode, g.solution.iterations, g.solution.termination.name, o.iterations, o.termination,
          "b rel", np.linalg.norm(g.solution.b - o.b) / np.linalg.norm(o.b),
          "cbest gpu", cg[1:].min(), int(np.argmin(cg[1:])) + 1, "orc", co[1:].min(), int(np.argmin(co[1:])) + 1)
