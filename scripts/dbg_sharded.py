"""Debug: 2-rank in-process group, c0: factors and the QR-mode dual."""
import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_14471_b200 import api, synth
p = synth.make_problem(0)
P = 2
Xf = torch.from_numpy(np.ascontiguousarray(p.X.T)).cuda(); Yf = torch.from_numpy(np.ascontiguousarray(p.Y.T)).cuda()
parts = [api.row_partition(p.M, P, r) for r in range(P)]
sh = [(Xf[:, a:a+m].contiguous(), Yf[:, a:a+m].contiguous(), m) for a, m in parts]
for mode in ("x", "qr"):
    grp = api.LocalGroup(P); out = [None]*P; err = [None]*P
    def w(r):
        try:
            Xr, Yr, m = sh[r]
            op = api.GpuSurPreconditioner.from_device_local_group(grp, r, p.G, m, p.M, p.nb, Xr.data_ptr(), m, Yr.data_ptr(), m, p.omega)
            g = api.pcg_aug(None, op, config=api.PcgConfig(tol_rel=p.tol_rel, max_iter=6, xv_mode=mode, diag_every=1), true_beta=p.beta)
            Q, R = op.factors()
            out[r] = (g, Q, R)
        except Exception as e:
            err[r] = e
    ts = [threading.Thread(target=w, args=(r,)) for r in range(P)]
    [t.start() for t in ts]; [t.join() for t in ts]
    print(mode, "errors", err)
    Q = np.concatenate([o[1] for o in out], axis=0); R = out[0][2]
    off = roff = 0
    for bi, k in enumerate(p.nb[:3]):
        Qi = Q[:, off:off+k]; Ri = R[roff:roff+k*k].reshape(k, k, order="F")
        print(mode, "blk", bi, "orth", np.abs(Qi.T@Qi-np.eye(k)).max(), "QR-X", np.abs(Qi@Ri - p.X[:, off:off+k]).max(),
              "R0==R1", np.array_equal(out[0][2], out[1][2]))
        off += k; roff += k*k
    for r in range(P):
        print(mode, "rank", r, "dual", out[r][0].trace.rows["dual_feas_norm"][:5], "c", out[r][0].trace.rows["c"][:3])
