"""Full-shape parity artefacts (GPU box): every BASELINE config at its real shape against the oracle.

    python scripts/parity_fullshape.py [--out profiles/r02_parity_fullshape.jsonl] [--only c4full,c4m20k,c1,c2,c3]

One JSON line per case (the GPU through the C-ABI; the oracle -- bitwise the reference -- on the same inputs,
multi-threaded).  c4: the bench's own device-generated inputs and knobs (D2H copy to the oracle); c1-c3: the
host generator (synth.make_problem).  tests/test_gpu_fullshape.py holds the same bars.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import witness  # noqa: E402
from paper_2510_14471_b200 import api, synth  # noqa: E402

rel = witness.rel


def host_case(c, mode="qr", variants=0, **kw):
    p = synth.make_problem(c, **kw)
    sur = api.sur_from_problem(p)
    t0 = time.perf_counter()
    op = api.sur_preconditioner(sur)
    g = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=p.tol_rel, max_iter=p.max_iter, xv_mode=mode, diag_every=0),
                    true_beta=p.beta, want_w=False)
    t_gpu = time.perf_counter() - t0
    op.close()
    cfg = oracle.make_config(tol_rel=p.tol_rel, max_iter=p.max_iter)
    t0 = time.perf_counter()
    o = oracle.solve(p, cfg=cfg, beta_true=p.beta)
    t_orc = time.perf_counter() - t0
    out = witness.compare(g, o)
    out.update({"config": c, "G": p.G, "M": p.M, "n": p.n, "nb_min": int(p.nb.min()), "nb_max": int(p.nb.max()),
                "xv_mode": mode, "inputs": "host generator (synth.make_problem)", "gpu_solve_s": t_gpu,
                "gpu_solve_ms_device": g.solve_ms, "oracle_s": t_orc, "oracle_threads": oracle.threads(),
                "rel_b_vs_beta_gpu": rel(g.solution.b, p.beta), "rel_b_vs_beta_oracle": rel(o.b, p.beta)})
    if variants:
        vs = []
        lib = oracle.lib("oracle")
        lib.orc_set_sum_mode(1)
        try:
            v = oracle.solve(p, cfg=cfg, beta_true=p.beta)
        finally:
            lib.orc_set_sum_mode(0)
        vs.append(("pairwise", v))
        for seed in range(1, variants + 1):
            q = synth.SurProblem(p.name, p.G, p.M, p.nb,
                                 np.asfortranarray(p.X * (1.0 + 1e-15 * np.random.default_rng(seed).standard_normal(p.X.shape))),
                                 p.Y, p.omega, p.beta, p.tol_rel, p.max_iter)
            vs.append((f"perturb{seed}", oracle.solve(q, cfg=cfg, beta_true=p.beta)))
        out["envelope"] = [{"variant": k, "iterations": v.iterations, "termination": v.termination,
                            "rel_b_vs_reference": rel(v.b, o.b), "rel_b_vs_beta": rel(v.b, p.beta)} for k, v in vs]
        out["envelope_spread"] = max(e["rel_b_vs_reference"] for e in out["envelope"])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_parity_fullshape.jsonl"))
    ap.add_argument("--only", default="c4m20k,c1,c2,c3w,c4full,c3")
    a = ap.parse_args()
    cases = {
        "c4m20k": lambda: witness.device_parity(4, M=20000, max_iter=200),
        "c4full": lambda: witness.device_parity(4, max_iter=3),
        "c1": lambda: host_case(1),
        "c2": lambda: host_case(2, variants=3),
        "c3w": lambda: host_case(3, M=5000, variants=2),
        "c3": lambda: host_case(3, variants=1),
    }
    with open(a.out, "a") as f:
        for name in a.only.split(","):
            t0 = time.perf_counter()
            try:
                r = cases[name]()
            except Exception as e:  # record and go on: each case is independent
                r = {"error": f"{type(e).__name__}: {e}"}
            r["case"] = name
            r["wall_s"] = time.perf_counter() - t0
            line = json.dumps(r)
            print(line, flush=True)
            f.write(line + "\n")
            f.flush()


if __name__ == "__main__":
    main()
