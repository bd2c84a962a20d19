"""Development aid: streaming-pass bandwidth for narrow (n_i = 32, tile-contiguous Q) vs wide blocks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14471_b200 import api, synth  # noqa: E402

for nb in (32, 33, 64, 100, 127):
    p = synth.random_sur(64, 100000, [nb] * 64, seed=3)
    sur = api.sur_from_problem(p)
    op = api.sur_preconditioner(sur)
    g = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=1e-14, max_iter=30, diag_every=0, xv_mode="qr",
                                                  kernel_timing=True), want_trace=False)
    st = {k["name"]: (k["total_ms"] / k["launches"], k["bytes_per_launch"] / (k["total_ms"] / k["launches"]) / 1e6)
          for k in op.kernel_stats() if k["launches"]}
    print(nb, {k: (round(v[0], 3), round(v[1])) for k, v in st.items()}, flush=True)
    op.close()
