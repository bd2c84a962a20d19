"""oracle.witness -- TEST INFRASTRUCTURE ONLY: the GPU solve against the oracle on the SAME inputs.

Used by tests/ (the full-shape parity tests), by scripts/parity_fullshape.py (the committed full-shape
artefacts under profiles/) and by bench.py's parity-witness line (after the timed region).  The GPU side
runs through the product's C-ABI exactly as the bench does (device-resident inputs, the bench's knobs);
the oracle (gls_oracle.c, bitwise the reference) runs on a D2H copy of the very same X and Y.

The bar is the north star's: same termination and iteration count, ||b_gpu - b_ref|| / ||b_ref|| <= 1e-10;
the early trace values c_i (r'Pi r, proj/src/pcg.cpp:156-157) are compared too.
"""
from __future__ import annotations

import time
from typing import Optional

import numpy as np

import oracle


def rel(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


BENCH_KNOBS = dict(xv_mode="qr", diag_every=0, kron_fma=True, sw_mode=1)


def gpu_solve_device(dp, max_iter: Optional[int] = None, knobs: Optional[dict] = None, device: int = 0):
    """The bench's solve of a DeviceProblem: from_device handle + PcgConfig(knobs)."""
    from paper_2510_14471_b200 import api
    knobs = dict(BENCH_KNOBS if knobs is None else knobs)
    op = api.GpuSurPreconditioner.from_device(dp.G, dp.M_local, dp.nb, dp.X.data_ptr(), dp.M_local, dp.Y.data_ptr(),
                                              dp.M_local, dp.omega, device=device)
    mi = dp.max_iter if max_iter is None else max_iter
    t0 = time.perf_counter()
    g = api.pcg_aug(None, op, config=api.PcgConfig(tol_rel=dp.tol_rel, max_iter=mi, **knobs), true_beta=dp.beta,
                    want_w=False)
    dt = time.perf_counter() - t0
    op.close()
    return g, dt


def compare(g, o, c_rows: int = 4) -> dict:
    """Verdict dict of a GPU AugSolveResult against an oracle SolveOut."""
    cg = np.asarray(g.trace.rows["c"])
    co = np.asarray(o.trace["c"])
    k = min(c_rows, len(cg), len(co))
    c_rel = [abs(float(cg[i]) - float(co[i])) / max(abs(float(co[i])), 1e-300) for i in range(k)]
    out = {
        "iterations_gpu": int(g.solution.iterations), "iterations_oracle": int(o.iterations),
        "termination_gpu": g.solution.termination.name, "termination_oracle": o.termination,
        "rel_b": rel(g.solution.b, o.b), "c_rows_rel": c_rel,
    }
    out["strict"] = bool(out["iterations_gpu"] == out["iterations_oracle"] and
                         out["termination_gpu"] == out["termination_oracle"] and out["rel_b"] <= 1e-10)
    return out


def device_parity(config: int = 4, M: Optional[int] = None, G: Optional[int] = None, max_iter: Optional[int] = None,
                  knobs: Optional[dict] = None, c_rows: int = 4, device: int = 0, threads: int = 0) -> dict:
    """Device-generated config (the bench's generator) solved on the GPU with the bench's knobs and by the
    oracle on a D2H copy of the same inputs."""
    from paper_2510_14471_b200 import devsynth
    dp = devsynth.device_problem(config, M=M, G=G, device=device)
    mi = dp.max_iter if max_iter is None else max_iter
    g, t_gpu = gpu_solve_device(dp, max_iter=mi, knobs=knobs, device=device)
    hp = dp.to_host_problem()
    del dp
    if threads:
        oracle.set_threads(threads)
    t0 = time.perf_counter()
    o = oracle.solve(hp, "oracle", cfg=oracle.make_config(tol_rel=hp.tol_rel, max_iter=mi), beta_true=hp.beta)
    t_orc = time.perf_counter() - t0
    out = compare(g, o, c_rows)
    out.update({"config": config, "G": hp.G, "M": hp.M, "n": int(hp.nb.sum()), "max_iter": mi,
                "knobs": dict(BENCH_KNOBS if knobs is None else knobs), "inputs": "device Philox (bench generator), "
                "D2H copy to the oracle", "gpu_solve_s": t_gpu, "oracle_s": t_orc,
                "oracle_threads": oracle.threads()})
    return out
