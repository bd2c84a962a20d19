"""bench.py -- GLS-PCG (PCG-Aug, SUR) iterations/s on BASELINE config 4 (G=256, M=1e6, n_i=32, fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C] [--xv qr|x]

A step is one complete GLS solve of the config on inputs resident in HBM: the setup QR of every
block (sur_preconditioner) + PCG-Aug to tol 1e-10 with the config's 200-iteration cap + the b
recovery.  `value` = PCG iterations completed / second over the K timed steps (CUDA events on the
solver stream, barrier + synchronize on both sides, max over ranks).  `e2e` = the same metric through
the C-ABI with HOST buffers (pinned X, Y copied in by glsgpu_sur_create every step, b copied out).

--impl reference times the reference's own CPU implementation (oracle/_ref, the unmodified gls_core
compiled from the reference sources; single-threaded as written) on a bounded row sample of the same
config, extrapolated linearly in M (every per-iteration and setup cost of the reference is linear in M).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2510_14471_b200 import synth  # noqa: E402

METRIC = "GLS-PCG iterations/s and solve time (fp64); achieved HBM GB/s vs peak"
UNIT = "iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--rows", type=int, default=0, help="override M (development only)")
    ap.add_argument("--xv", default="qr", choices=["qr", "x"])
    ap.add_argument("--fused", default="off", choices=["on", "off"],
                    help="Sigma pr inside pass C with an element-wise pass A (fused_c; needs --sw direct; parity-tested, "
                         "slower at c4 -- DESIGN.md s10)")
    ap.add_argument("--sw", default="direct", choices=["direct", "recurrence"],
                    help="Sigma w: formed where read (sw_mode 1) or the reference's recurrence; both parity-tested")
    ap.add_argument("--kron", default="fma", choices=["fma", "exact"],
                    help="Kronecker pass arithmetic (glsgpu_pcg_config::kron_fma); both are parity-tested")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0)
    return ap.parse_args()


def workload(c: int, M: int):
    meta = synth.config_meta(c)
    prob = synth.make_problem(c, M=M, with_data=False)
    return meta, prob


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc or not os.path.exists(self.path):
            return None
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                s, m, pw = float(parts[0]), float(parts[1]), float(parts[2])
            except ValueError:
                continue
            if pw > 300:  # under load
                sm.append(s)
            mx.append(m)
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                               parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not mx:
            return None
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples_under_load": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------------- CPU baseline
def cpu_sample(c: int, kind: str, rows: int, k1: int, k2: int):
    """Time the CPU implementation on a row sample at two iteration caps; return per-iteration and
    setup seconds at the sample size (slope / intercept)."""
    import oracle
    p = synth.make_problem(c, M=rows)
    times = []
    for k in (k1, k2):
        cfg = oracle.make_config(tol_rel=p.tol_rel, max_iter=k)
        t0 = time.perf_counter()
        out = oracle.solve(p, kind, cfg=cfg, beta_true=p.beta)
        times.append((time.perf_counter() - t0, out.iterations))
    (t1, i1), (t2, i2) = times
    per_it = (t2 - t1) / max(i2 - i1, 1)
    setup = max(t1 - per_it * i1, 0.0)
    return per_it, setup, p, sum(t for t, _ in times)


def cpu_value(c: int, M: int, max_iter: int, kind: str, rows: int):
    k1, k2 = (2, 6) if kind == "ref" else (3, 10)
    per_it, setup, p, spent = cpu_sample(c, kind, rows, k1, k2)
    scale = M / rows
    iters = max_iter if max_iter else 200
    step_s = setup * scale + iters * per_it * scale
    return {
        "value": iters / step_s,
        "unit": UNIT,
        "cores": 1,
        "kind": "reference" if kind == "ref" else "port",
        "sample": (f"config {c} with M={rows} rows (of {M}); solves capped at {k1} and {k2} iterations; "
                   f"per-iteration {per_it * 1e3:.1f} ms and setup {setup:.2f} s at the sample, scaled x{scale:.0f} "
                   f"(linear in M) to a {iters}-iteration solve: EXTRAPOLATED; {spent:.1f} s of CPU work; "
                   + ("literal pcg_aug(embed_sur(sur), *sur_preconditioner(sur)) of the unmodified reference"
                      if kind == "ref" else "structured restatement of run_aug (bitwise-equal to the reference)")),
    }


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    meta = synth.config_meta(args.config)
    M = args.rows or meta["M"]
    max_iter = meta["max_iter"] or 200
    import oracle
    kind = "ref" if oracle.have("ref") else "oracle"
    rows = args.cpu_rows or (48 if kind == "ref" else 1000)
    vals = []
    for s in range(args.warmup + args.steps):
        v = cpu_value(args.config, M, max_iter, kind, rows)
        if s >= args.warmup:
            vals.append(v)
    value = statistics.mean(v["value"] for v in vals)
    cb = dict(vals[-1])
    cb["value"] = value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * max_iter / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy Philox; BASELINE config shapes/distributions)",
        "config": {"workload": f"c{args.config}", "G": meta["G"], "M": M, "parallelism": "none (1 CPU thread)"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    from paper_2510_14471_b200 import api
    from paper_2510_14471_b200 import _lib as L
    import ctypes as C

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = local
    lib = L.load()
    meta = synth.config_meta(args.config)
    M = args.rows or meta["M"]
    G = meta["G"]
    seed = 1000 + args.config
    prob = synth.make_problem(args.config, M=M, with_data=False)
    nb = np.ascontiguousarray(prob.nb, dtype=np.int64)
    n = int(nb.sum())
    max_iter = meta["max_iter"]
    tol = meta["tol"]

    # ---- synthetic inputs generated on the device (counter-based Philox normals; BASELINE distributions);
    # with N ranks each rank draws its own row shard of the SAME global matrices
    if prob.name.startswith("c3"):
        raise SystemExit("bench: config 3 uses host generation; run config 4 (the bench workload)")
    row0, Ml = api.row_partition(M, world, rank) if world > 1 else (0, M)
    X = torch.empty((n, Ml), dtype=torch.float64, device=f"cuda:{dev}")   # column-major Ml x n, ld = Ml
    Y = torch.empty((G, Ml), dtype=torch.float64, device=f"cuda:{dev}")
    rc = lib.glsgpu_synth_normal(C.c_void_p(X.data_ptr()), Ml, n, Ml, row0, M, seed, 0, dev)
    assert rc == 0, lib.glsgpu_last_error_message()
    beta = synth._rng(seed, 1).standard_normal(n)
    omega = prob.omega
    oh = synth.omega_half(omega)
    rc = lib.glsgpu_synth_response(G, Ml, row0, M, nb.ctypes.data_as(C.POINTER(C.c_int64)), C.c_void_p(X.data_ptr()),
                                   Ml, beta.ctypes.data_as(C.POINTER(C.c_double)),
                                   oh.ctypes.data_as(C.POINTER(C.c_double)), seed, C.c_void_p(Y.data_ptr()), Ml, dev)
    assert rc == 0, lib.glsgpu_last_error_message()
    torch.cuda.synchronize()

    if world > 1:
        obj = [api.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        op = api.GpuSurPreconditioner.from_device_sharded(G, Ml, M, nb, X.data_ptr(), Ml, Y.data_ptr(), Ml, omega,
                                                          obj[0], rank, world, device=dev)
    else:
        op = api.GpuSurPreconditioner.from_device(G, M, nb, X.data_ptr(), M, Y.data_ptr(), M, omega, device=dev)
    fma = args.kron == "fma"
    cfg = api.PcgConfig(tol_rel=tol, max_iter=max_iter, xv_mode=args.xv, diag_every=0, kernel_timing=False,
                        kron_fma=fma, sw_mode=1 if args.sw == "direct" else 0, fused_c=1 if args.fused == "on" else 0)
    stream = torch.cuda.ExternalStream(op.stream_ptr(), device=f"cuda:{dev}")

    setup_ms = []

    def step(timing=False):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        op.refactor()
        e1.record(stream)
        cfg.kernel_timing = timing
        r = api.pcg_aug(None, op, config=cfg, true_beta=beta, want_w=False)
        if timing:
            setup_ms.append(e0.elapsed_time(e1))
        return r

    for _ in range(args.warmup):
        step()
    # ---- timed region
    results = []
    kstats = {}
    launches0 = op.launch_count()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            r = step(timing=True)
            results.append(r)
            for s in op.kernel_stats():
                d = kstats.setdefault(s["name"], {"launches": 0, "total_ms": 0.0, "bytes_per_launch": s["bytes_per_launch"]})
                d["launches"] += s["launches"]
                d["total_ms"] += s["total_ms"]
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = op.launch_count() - launches0
    elapsed_ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([elapsed_ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    iters = sum(r.solution.iterations for r in results)
    value = iters / (elapsed_ms / 1e3)
    last = results[-1]

    # ---- roofline of the dominant kernel (largest algorithmic bytes per launch)
    peak, peak_src = peaks()
    dom_name = max(kstats, key=lambda k: kstats[k]["bytes_per_launch"]) if kstats else None
    roof = None
    if dom_name and kstats[dom_name]["launches"]:
        d = kstats[dom_name]
        avg_ms = d["total_ms"] / d["launches"]
        achieved = d["bytes_per_launch"] / (avg_ms / 1e3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get(dom_name)
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": dom_name, "bytes_per_launch": d["bytes_per_launch"],
                "avg_launch_ms": avg_ms, "peak_source": peak_src}
    iter_ms = 0.0
    b_iter = 8.0 * (2.0 * M * n + 14.0 * M * G)
    passes = {}
    for k, d in kstats.items():
        if d["launches"]:
            avg = d["total_ms"] / d["launches"]
            passes[k] = {"avg_ms": avg, "GB/s": d["bytes_per_launch"] / (avg / 1e3) / 1e9}
            iter_ms += avg

    # ---- e2e through the C-ABI with host buffers (pinned X, Y -> device every step; b -> host)
    e2e = None
    if not args.no_e2e:
        Xh = torch.empty((n, Ml), dtype=torch.float64, pin_memory=True)
        Yh = torch.empty((G, Ml), dtype=torch.float64, pin_memory=True)
        Xh.copy_(X)
        Yh.copy_(Y)
        torch.cuda.synchronize()
        op.close()
        del X, Y, op
        torch.cuda.empty_cache()
        e_iters, e_time = 0, 0.0
        ksteps = max(1, min(args.steps, 2))
        ecfg = api.PcgConfig(tol_rel=tol, max_iter=max_iter, xv_mode=args.xv, diag_every=0, kron_fma=fma,
                             sw_mode=1 if args.sw == "direct" else 0, fused_c=1 if args.fused == "on" else 0)
        for s in range(ksteps + 1):
            if world > 1:
                obj = [api.nccl_unique_id() if rank == 0 else None]
                torch.distributed.broadcast_object_list(obj, src=0)
                torch.distributed.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if world > 1:
                # the C-ABI's sharded entry takes device buffers: this rank's host shard goes in first
                Xd = Xh.to(f"cuda:{dev}", non_blocking=True)
                Yd = Yh.to(f"cuda:{dev}", non_blocking=True)
                torch.cuda.synchronize()
                op2 = api.GpuSurPreconditioner.from_device_sharded(G, Ml, M, nb, Xd.data_ptr(), Ml, Yd.data_ptr(), Ml,
                                                                   omega, obj[0], rank, world, device=dev)
                r2 = api.pcg_aug(None, op2, config=ecfg, want_w=False)
                op2.close()
                del Xd, Yd
            else:
                # create once (step 0, untimed warm-up), then per step: new host data through the C-ABI
                # (glsgpu_sur_update: H2D of X and Y pipelined with the TSQR), the solve, b back to the host
                if s == 0:
                    sur = api.SurModel(X=Xh.numpy().T, nb=nb, y=Yh.numpy().T, sigma0=omega)
                    op2 = api.GpuSurPreconditioner(sur, device=dev)
                else:
                    op2.update(Xh.numpy().T, Yh.numpy().T)
                r2 = api.pcg_aug(sur, op2, config=ecfg, want_w=False)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([dt], device=f"cuda:{dev}")
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                dt = float(t.item())
            if s > 0:  # first e2e step is a warm-up (allocator / context)
                e_iters += r2.solution.iterations
                e_time += dt
        if world == 1:
            op2.close()
        e2e = {"value": e_iters / e_time, "unit": UNIT, "h2d_bytes_per_step": int(8 * (M * n + M * G)),
               "d2h_bytes_per_step": int(8 * n + 48 * (r2.trace.rows.size)), "steps": ksteps,
               "timer": ("host wall clock (max over ranks) around: H2D of the step's X and Y from pinned memory "
                         "pipelined with the TSQR (glsgpu_sur_update; 1 GPU) or create (N > 1) + solve + b D2H")}
        del Xh, Yh

    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        try:
            cpu = cpu_value(args.config, M, max_iter, "oracle", args.cpu_rows or 1000)
        except Exception as e:  # the CPU baseline is a reported number, never the product
            cpu = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device counter-based Philox N(0,1) X, beta, Z; Omega = L L' + 0.1 I; BASELINE c4)",
            "config": {"workload": f"c{args.config}: G={G}, M={M}, n_i={int(nb[0])}, n={n}, tol {tol:g}, "
                                   f"max_iter {max_iter}; step = setup QR + PCG-Aug solve + recovery",
                       "G": G, "M": M, "n": n, "xv_mode": args.xv, "kron_arith": args.kron, "sigma_w": args.sw, "fused_c": args.fused, "trace_diagnostics": "row 0 + final row",
                       "l2": "inputs (65.5 GB X/Q) far larger than L2", "parallelism": f"rows x{world}"},
            "iterations_per_step": [r.solution.iterations for r in results],
            "termination": last.solution.termination.name,
            "iter_ms": iter_ms, "b_iter_bytes": b_iter,
            "setup_qr_ms": statistics.mean(setup_ms) if setup_ms else None,
            "solve_ms": statistics.mean(r.solve_ms for r in results),
            "iter_GBps_algorithmic": b_iter / (iter_ms / 1e3) / 1e9 if iter_ms else None,
            "passes": passes,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
