"""Development aid: trace-level comparison of a MVRGLM solve, GPU vs oracle variants."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle
from paper_2510_14471_b200 import api, synth

p = synth.random_mv(5, 60, 8, seed=42)
p.z_scale = np.linspace(0.5, 2.0, p.G)
p.c_scale = np.linspace(3.0, 0.25, p.G)
p.max_iter = 3 * (p.k + 1) + 10
cfg = oracle.make_config(tol_rel=p.tol_rel, max_iter=p.max_iter)
o = oracle.solve_mv(p, cfg=cfg)
L = oracle.lib("oracle")
L.orc_set_sum_mode(1)
o1 = oracle.solve_mv(p, cfg=cfg)
L.orc_set_sum_mode(0)
mv = api.mv_from_problem(p)
op = api.mvrglm_preconditioner(mv, p.z_scale, p.c_scale)
for mode in ("x", "qr"):
    g = api.pcg_aug(mv, op, config=api.PcgConfig(tol_rel=p.tol_rel, max_iter=p.max_iter, xv_mode=mode, diag_every=1))
    print(mode, g.solution.iterations, g.solution.termination.name, g.trace.breakdown_iteration, "oracle", o.iterations,
          o.termination, "pair", o1.iterations, o1.termination)
    n = min(len(g.trace.rows), len(o.trace))
    for i in range(n):
        print(i, "%.6e %.6e %.6e | aug %.6e %.6e | dual %.3e %.3e" % (
            g.trace.rows["c"][i], o.trace["c"][i], o1.trace["c"][i] if i < len(o1.trace) else np.nan,
            g.trace.rows["aug_residual_norm"][i], o.trace["aug_residual_norm"][i],
            g.trace.rows["dual_feas_norm"][i], o.trace["dual_feas_norm"][i]))
