import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_14471_b200 import api, synth
p = synth.make_problem(0)
P = 2
Xf = torch.from_numpy(np.ascontiguousarray(p.X.T)).cuda(); Yf = torch.from_numpy(np.ascontiguousarray(p.Y.T)).cuda()
for M_al in (False, True):
    parts = [api.row_partition(p.M, P, r) for r in range(P)] if not M_al else [(0, 512), (512, 488)]
    sh = [(Xf[:, a:a+m].contiguous(), Yf[:, a:a+m].contiguous(), m) for a, m in parts]
    for mode in ("x", "qr"):
        for mi in (1,):
            grp = api.LocalGroup(P); out = [None]*P; err = [None]*P
            def w(r):
                try:
                    Xr, Yr, m = sh[r]
                    op = api.GpuSurPreconditioner.from_device_local_group(grp, r, p.G, m, p.M, p.nb, Xr.data_ptr(), m, Yr.data_ptr(), m, p.omega)
                    g = api.pcg_aug(None, op, config=api.PcgConfig(tol_rel=p.tol_rel, max_iter=mi, xv_mode=mode, diag_every=1), true_beta=p.beta, want_w=True)
                    out[r] = g
                except Exception as e:
                    err[r] = e
            ts = [threading.Thread(target=w, args=(r,)) for r in range(P)]
            [t.start() for t in ts]; [t.join() for t in ts]
            xtw = 0
            for r in range(P):
                a, m = parts[r]
                W = out[r].solution.w.reshape(p.G, m)
                off = 0; v = []
                for b, k in enumerate(p.nb):
                    v.append(p.X[a:a+m, off:off+k].T @ W[b]); off += k
                xtw = xtw + np.concatenate(v)
            print("aligned" if M_al else "unaligned", mode, "max_iter", mi, "err", err, "host |X'w|", np.linalg.norm(xtw),
                  "trace dual r0", out[0].trace.rows["dual_feas_norm"][-1], "r1", out[1].trace.rows["dual_feas_norm"][-1])
