"""Quick GPU-vs-oracle parity probe (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2510_14471_b200 import synth, api

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

def run(c, **kw):
    p = synth.make_problem(c, **kw)
    t = time.time(); o = oracle.solve(p, "oracle"); to = time.time() - t
    sur = api.sur_from_problem(p)
    t = time.time(); op = api.sur_preconditioner(sur); tq = time.time() - t
    Qo, Ro = oracle.sur_setup(p)
    Qg, Rg = op.factors()
    # Q up to column signs: compare projectors via Q Q' applied to a probe
    xi = np.random.default_rng(0).standard_normal(p.M * p.G)
    pi_o = oracle.sur_apply(p, "pi", xi); pi_g = op.apply_pi(xi)
    xt_o = oracle.sur_apply(p, "xstar_t", xi); xt_g = op.apply_xstar_t(xi)
    v = np.random.default_rng(1).standard_normal(p.n)
    xs_o = oracle.sur_apply(p, "xstar", v); xs_g = op.apply_xstar(v)
    sg_o = oracle.kron_apply(p.omega, xi, p.M); sg_g = op.sigma_apply(xi)
    print(f"c{c} {kw} setup {tq:.3f}s  pi {rel(pi_g,pi_o):.2e} xstar_t {rel(xt_g,xt_o):.2e} xstar {rel(xs_g,xs_o):.2e} "
          f"sigma bitwise={np.array_equal(sg_g, sg_o)} {rel(sg_g,sg_o):.2e}", flush=True)
    for mode in ("x", "qr"):
        cfg = api.PcgConfig(tol_rel=p.tol_rel, max_iter=p.max_iter, xv_mode=mode)
        t = time.time(); g = api.pcg_aug(sur, op, config=cfg, true_beta=p.beta); tg = time.time() - t
        print(f"   [{mode}] oracle it={o.iterations} {o.termination} ({to:.2f}s) | gpu it={g.solution.iterations} "
              f"{g.solution.termination.name} ({tg:.3f}s, dev {g.solve_ms:.1f} ms) rel b {rel(g.solution.b, o.b):.2e} "
              f"rel w {rel(g.solution.w, o.w):.2e} c0 {g.trace.rows['c'][0]:.6e}/{o.trace['c'][0]:.6e} "
              f"aug0 {g.trace.rows['aug_residual_norm'][0]:.6e}/{o.trace['aug_residual_norm'][0]:.6e} "
              f"dual1 {g.trace.rows['dual_feas_norm'][1]:.4e}/{o.trace['dual_feas_norm'][1]:.4e} "
              f"sigscale {g.sigma_scale:.12e}/{o.sigma_scale:.12e}", flush=True)

if __name__ == "__main__":
    run(0)
    run(1, M=400)
    run(2, M=1000)
    run(3, M=600, N=40)
    run(4, M=2000, G=32)
