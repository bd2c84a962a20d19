"""Every solver path on the B200 at the BASELINE configs' full shapes (development / evidence aid; not the
driver's bench): GPU wall time of one complete solve (setup + iterations + recovery) through the C-ABI from
host buffers, the iteration count and termination, and -- where a CPU solve finishes in bounded time -- the
oracle (bitwise the reference) on the same inputs with the relative difference of b.

    python scripts/bench_paths.py [--cpu] > profiles/r01_paths.json   (one JSON line per path)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14471_b200 import api, synth  # noqa: E402

CPU = "--cpu" in sys.argv


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t0


def emit(**kw):
    print(json.dumps(kw), flush=True)


def sur_path(name, p, cfg_kw, cpu_ok):
    sur = api.sur_from_problem(p)
    cfg = api.PcgConfig(tol_rel=p.tol_rel, max_iter=p.max_iter, diag_every=0, xv_mode="qr", **cfg_kw)
    api.pcg_aug(sur, config=cfg, want_trace=False)  # warm-up (context, kernels)

    def solve():
        op = api.sur_preconditioner(sur)
        g = api.pcg_aug(sur, op, config=cfg, want_trace=False)
        op.close()
        return g
    g, dt = timed(solve)
    rec = dict(path=name, G=p.G, M=p.M, n=p.n, gpu_s=dt, iterations=g.solution.iterations,
               termination=g.solution.termination.name, gpu_it_per_s=g.solution.iterations / dt)
    if CPU and cpu_ok:
        import oracle
        o, ct = timed(lambda: oracle.solve(p, cfg=oracle.make_config(tol_rel=p.tol_rel, max_iter=p.max_iter),
                                           trace=False))
        rec.update(cpu_s=ct, cpu_iterations=o.iterations, cpu_termination=o.termination, rel_b=rel(g.solution.b, o.b),
                   speedup=ct / dt)
    emit(**rec)


def main():
    # SUR configs 1-3 (BASELINE.json:configs[1..3]) through the SUR operator
    sur_path("sur_c1", synth.make_problem(1), {}, True)
    sur_path("sur_c2", synth.make_problem(2), {}, True)
    c3 = synth.make_problem(3)
    sur_path("sur_c3", c3, {}, False)
    # config 3 as the multivariate model: mv_reduce on the device, then MVRGLM (K2 auxiliary, the harness's
    # choice) on the N0-row model; and sur_reduce (Remark 1) then the SUR solve
    mv = synth.make_mv_problem(3)
    mvm = api.mv_from_problem(mv)
    api.mv_reduce(mvm)  # warm-up

    def mv_route():
        red, _ = api.mv_reduce(mvm)
        zs, cs = api.auxiliary_scales(mv.omega, "k2", z0=red.z0)
        g = api.pcg_aug(red, api.mvrglm_preconditioner(red, zs, cs),
                        config=api.PcgConfig(tol_rel=1e-12, max_iter=3 * (mv.k + 1) + 10, diag_every=0),
                        want_trace=False)
        return g
    g, dt = timed(mv_route)
    emit(path="c3_mv_reduce_mvrglm_k2", G=mv.G, M0=mv.M0, N0=mv.N0, k=mv.k, gpu_s=dt,
         iterations=g.solution.iterations, termination=g.solution.termination.name)
    sur3 = api.sur_from_problem(c3)

    def red_route():
        red, rec = api.sur_reduce(sur3)
        g = api.pcg_aug(red, config=api.PcgConfig(tol_rel=c3.tol_rel, diag_every=0), want_trace=False)
        return g, rec
    (g, rec), dt = timed(red_route)
    emit(path="c3_sur_reduce_then_sur", G=c3.G, M=c3.M, reduced_rows=rec.reduced_rows, gpu_s=dt,
         iterations=g.solution.iterations, termination=g.solution.termination.name)
    # PCG-NE comparison solver on config 1
    p1 = synth.make_problem(1)
    op1 = api.sur_preconditioner(api.sur_from_problem(p1))
    g, dt = timed(lambda: api.pcg_normal_equations(op1, api.PcgConfig(tol_rel=1e-12, max_iter=2000),
                                                    want_trace=False))
    emit(path="pcg_ne_c1", G=p1.G, M=p1.M, n=p1.n, gpu_s=dt, iterations=g.solution.iterations,
         termination=g.solution.termination.name)


if __name__ == "__main__":
    main()
