"""Debug: QR-mode trace dual_feas_norm on the colpass (non-TMA) path vs the stream path, sharded vs not."""
import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_14471_b200 import api, synth
p = synth.make_problem(0)
X = torch.from_numpy(np.ascontiguousarray(p.X.T)).cuda(); Y = torch.from_numpy(np.ascontiguousarray(p.Y.T)).cuda()
for mode in ("x", "qr"):
    cfg = api.PcgConfig(tol_rel=p.tol_rel, max_iter=8, xv_mode=mode, diag_every=1)
    g_host = api.pcg_aug(api.sur_from_problem(p), config=cfg, true_beta=p.beta)
    op_dev = api.GpuSurPreconditioner.from_device(p.G, p.M, p.nb, X.data_ptr(), p.M, Y.data_ptr(), p.M, p.omega)
    g_dev = api.pcg_aug(None, op_dev, config=cfg, true_beta=p.beta)
    grp = api.LocalGroup(1)
    op_g = api.GpuSurPreconditioner.from_device_local_group(grp, 0, p.G, p.M, p.M, p.nb, X.data_ptr(), p.M, Y.data_ptr(), p.M, p.omega)
    g_grp = api.pcg_aug(None, op_g, config=cfg, true_beta=p.beta)
    op_n = api.GpuSurPreconditioner.from_device_sharded(p.G, p.M, p.M, p.nb, X.data_ptr(), p.M, Y.data_ptr(), p.M, p.omega, api.nccl_unique_id(), 0, 1)
    g_n = api.pcg_aug(None, op_n, config=cfg, true_beta=p.beta)
    for col in ("c", "aug_residual_norm", "dual_feas_norm", "rmse"):
        print(mode, col, "host", g_host.trace.rows[col][:4], "\n   dev", g_dev.trace.rows[col][:4], "\n   grp", g_grp.trace.rows[col][:4], "\n   nccl1", g_n.trace.rows[col][:4])
