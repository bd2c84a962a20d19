"""Debug aid: operator applies and the c trace of one small problem, GPU vs oracle."""
import numpy as np
import oracle
from paper_2510_14471_b200 import api, synth

p = synth.random_sur(3, 200, [5, 7, 4], seed=21)
sur = api.sur_from_problem(p)
op = api.sur_preconditioner(sur)
rng = np.random.default_rng(1)
x = rng.standard_normal(p.M * p.G)
v = rng.standard_normal(int(np.sum(p.nb)))
for name, f, arg in (("pi", op.apply_pi, x), ("xstar_t", op.apply_xstar_t, x), ("xstar", op.apply_xstar, v)):
    a = f(arg)
    b = oracle.sur_apply(p, name, arg)
    print(name, np.abs(a - b).max() / np.abs(b).max())
sa = op.sigma_apply(x)
sb = oracle.kron_apply(p.omega, x, p.M)
print("sigma", np.abs(sa - sb).max())
print("omega", p.omega.shape, np.linalg.eigvalsh(p.omega)[[0, -1]], "scale", getattr(p, "scale", None))
o = oracle.solve(p, "oracle", cfg=oracle.make_config(tol_rel=1e-6))
for mode in ("x", "qr"):
    for diag in (1, 0):
        g = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=1e-6, xv_mode=mode, diag_every=diag))
        print(mode, diag, g.solution.iterations, g.solution.termination, o.iterations, o.termination)
g = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=1e-6))
cg = g.trace.rows["c"]; co = o.trace["c"]
k = min(len(cg), len(co))
print("c gpu", cg[:k])
print("c orc", co[:k])
print("sigma_scale", g.sigma_scale, o.sigma_scale if hasattr(o, "sigma_scale") else None)
