"""Development aid: where a config's SUR solve spends its time (setup vs passes).  python scripts/c3_profile.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14471_b200 import api, synth  # noqa: E402

p = synth.make_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
sur = api.sur_from_problem(p)
print("widths min/max", int(p.nb.min()), int(p.nb.max()), "n", p.n, flush=True)
t0 = time.perf_counter()
op = api.sur_preconditioner(sur)
t1 = time.perf_counter()
op.refactor()
t2 = time.perf_counter()
g = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=p.tol_rel, diag_every=0, xv_mode="qr", kernel_timing=True),
                want_trace=False)
t3 = time.perf_counter()
print(f"create {1e3 * (t1 - t0):.1f} ms, refactor {1e3 * (t2 - t1):.1f} ms, solve {1e3 * (t3 - t2):.1f} ms "
      f"({g.solution.iterations} it, device {g.solve_ms:.1f} ms)")
for k in op.kernel_stats():
    if k["launches"]:
        print(k["name"], k["launches"], f"{k['total_ms'] / k['launches']:.3f} ms/launch",
              f"{k['bytes_per_launch'] / (k['total_ms'] / k['launches']) / 1e6:.0f} GB/s")
