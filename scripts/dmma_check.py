"""Development aid: the DMMA pass A (k_kron_mma) against the DFMA one (k_kron_ws<true>) on c4-shaped inputs:
the same FMA chain, so the solves must agree bitwise."""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, ".")
if len(sys.argv) > 1:
    from paper_2510_14471_b200 import api, synth
    G = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    p = synth.make_problem(4, M=int(sys.argv[1]), G=G)
    g = api.pcg_aug(api.sur_from_problem(p), config=api.PcgConfig(tol_rel=1e-10, max_iter=200, xv_mode="qr",
                                                                    diag_every=0, kron_fma=1))
    np.save(sys.argv[3], np.concatenate([[g.solution.iterations], g.solution.b]))
    sys.exit(0)
for M, G in ((300, 256), (1000, 160), (2000, 256)):
    a = subprocess.run([sys.executable, __file__, str(M), str(G), "/tmp/a.npy"], env=dict(os.environ))
    b = subprocess.run([sys.executable, __file__, str(M), str(G), "/tmp/b.npy"], env=dict(os.environ, GLSGPU_NO_DMMA="1"))
    x, y = np.load("/tmp/a.npy"), np.load("/tmp/b.npy")
    print(f"M={M} G={G}: iterations {int(x[0])} vs {int(y[0])}, bitwise {np.array_equal(x, y)}, "
          f"max|diff| {np.max(np.abs(x - y)):.3e}", flush=True)
