"""The library's row-sharded path with more than one rank, and the staged (pipelined) update path.

Row sharding: rank r owns a contiguous row range of every block; per iteration the
ranks all-gather their partial sums and reduce them in rank order; the setup QR is a TSQR whose top level spans
the ranks (k_stack_r + a replicated QR of the stacked R's).  Only one GPU is available to these tests, and ranks
whose kernels wait on one another must not share a GPU (B200_PROFILING.md), so the ranks here are an in-process
group on one device (glsgpu_sur_create_sharded_local, TEST-ONLY): one host thread per rank, the all-gathers done
by device-to-device copies ordered with CUDA events and host barriers.  Everything else -- every kernel, the
cross-rank TSQR, the rank-order sums, the device-side scalar control -- is the product's sharded code path.
"""
import threading

import numpy as np
import pytest

import oracle
from paper_2510_14471_b200 import api, synth

pytestmark = pytest.mark.gpu

B_TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def require_device():
    assert api.device_count() > 0, "no CUDA device: the GPU tests must run on the B200 box (no CPU fallback exists)"


def run_group(p, P, cfg, partition=None):
    """Solve p with P in-process ranks on device 0; returns per-rank (result, Q_local, R)."""
    import torch
    Xf = torch.from_numpy(np.ascontiguousarray(p.X.T)).cuda()   # (n, M) == M x n column-major
    Yf = torch.from_numpy(np.ascontiguousarray(p.Y.T)).cuda()
    parts = partition or [api.row_partition(p.M, P, r) for r in range(P)]
    shards = [(Xf[:, r0:r0 + ml].contiguous(), Yf[:, r0:r0 + ml].contiguous(), ml) for r0, ml in parts]
    torch.cuda.synchronize()
    grp = api.LocalGroup(P)
    out, err = [None] * P, [None] * P

    def worker(r):
        try:
            Xr, Yr, ml = shards[r]
            op = api.GpuSurPreconditioner.from_device_local_group(grp, r, p.G, ml, p.M, p.nb, Xr.data_ptr(), ml,
                                                                  Yr.data_ptr(), ml, p.omega)
            g = api.pcg_aug(None, op, config=cfg, true_beta=p.beta, want_w=True)
            Q, R = op.factors()
            g.factor_method = op.factor_info()[0]
            out[r] = (g, Q, R)
            op.close()
        except Exception as e:  # noqa: BLE001 -- reported below
            err[r] = e

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=900)
    grp.close()
    assert all(not t.is_alive() for t in ts), "a rank thread hung"
    for e in err:
        if e is not None:
            raise e
    return out, parts


# the last field: the setup every rank must have taken -- CholeskyQR2 with all-gathered Grams when every rank's shard
# is on the TMA passes (32-row aligned), the cross-rank Householder TSQR otherwise
CASES = [
    ("c4_G24_M2048_P2_aligned", lambda: synth.make_problem(4, M=2048, G=24), 2, None, "cholqr2"),
    ("c1_G20_M1280_P2_wide_aligned", lambda: synth.make_problem(1, M=1280, G=20), 2, None, "cholqr2"),
    ("c4_G24_M3000_P2", lambda: synth.make_problem(4, M=3000, G=24), 2, None, None),
    ("c4_G24_M3000_P3_uneven", lambda: synth.make_problem(4, M=3000, G=24), 3, [(0, 700), (700, 1500), (2200, 800)],
     "tsqr"),
    ("c1_G20_M1200_P2_wide", lambda: synth.make_problem(1, M=1200, G=20), 2, None, None),
    ("c0_P2", lambda: synth.make_problem(0), 2, None, None),
]


@pytest.mark.parametrize("mode", ["qr", "x"])
@pytest.mark.parametrize("name,mk,P,part,method", CASES, ids=[c[0] for c in CASES])
def test_sharded_ranks_match_oracle(name, mk, P, part, method, mode):
    p = mk()
    mx = p.max_iter or 400
    cfg = api.PcgConfig(tol_rel=p.tol_rel, max_iter=mx, xv_mode=mode, diag_every=1)
    out, parts = run_group(p, P, cfg, part)
    g0 = out[0][0]
    methods = {g.factor_method for g, _, _ in out}
    assert len(methods) == 1, methods  # the collectives of the two factorisations differ: all ranks take the same
    if method is not None:
        assert methods == {method}, methods
    # every rank takes bitwise the same decisions and holds the same replicated b and R
    for g, _, R in out[1:]:
        assert g.solution.iterations == g0.solution.iterations
        assert g.solution.termination == g0.solution.termination
        assert np.array_equal(g.solution.b, g0.solution.b)
        assert np.array_equal(g.trace.rows["c"], g0.trace.rows["c"])
        assert np.array_equal(R, out[0][2])
    # against the oracle (bitwise the reference) on the unsharded model: the north-star bar
    o = oracle.solve(p, "oracle", cfg=oracle.make_config(tol_rel=p.tol_rel, max_iter=mx), beta_true=p.beta)
    assert g0.solution.termination.name == o.termination
    assert g0.solution.iterations == o.iterations, (g0.solution.iterations, o.iterations)
    assert rel(g0.solution.b, o.b) <= B_TOL, rel(g0.solution.b, o.b)
    # the cross-rank TSQR: the stacked local Q's are orthonormal per block and Q R = w X; |R_kk| as the reference
    Q = np.concatenate([q for _, q, _ in out], axis=0)
    Qo, Ro = oracle.sur_setup(p)
    off = roff = 0
    for k in p.nb:
        Qi = Q[:, off:off + k]
        Ri = out[0][2][roff:roff + k * k].reshape(k, k, order="F")
        assert np.max(np.abs(Qi.T @ Qi - np.eye(k))) < 1e-13
        assert np.max(np.abs(Qi @ Ri - p.X[:, off:off + k])) < 1e-12 * max(1.0, np.abs(p.X[:, off:off + k]).max())
        Roi = Ro[roff:roff + k * k].reshape(k, k, order="F")
        assert np.allclose(np.abs(np.diag(Ri)), np.abs(np.diag(Roi)), rtol=1e-12)
        off += k
        roff += k * k
    # the trace diagnostics of the sharded run equal the unsharded device run's
    op1 = api.sur_preconditioner(api.sur_from_problem(p))
    g1 = api.pcg_aug(None, op1, config=cfg, true_beta=p.beta)
    assert g1.solution.iterations == g0.solution.iterations
    assert rel(g0.solution.b, g1.solution.b) <= 1e-12
    k = min(5, len(g1.trace.rows))
    for col in ("c", "aug_residual_norm", "rmse"):
        assert np.allclose(g0.trace.rows[col][:k], g1.trace.rows[col][:k], rtol=1e-10, equal_nan=True), col
    # |X'w| sits at the roundoff level (w stays feasible): equal in absolute terms at that level
    scale = float(np.nanmax(g1.trace.rows["aug_residual_norm"][:k]))
    assert np.allclose(g0.trace.rows["dual_feas_norm"][:k], g1.trace.rows["dual_feas_norm"][:k], rtol=0,
                       atol=1e-10 * scale)
    # w is this rank's rows of the unsharded w
    W = np.concatenate([out[r][0].solution.w.reshape(p.G, parts[r][1]) for r in range(P)], axis=1).ravel()
    assert rel(W, g1.solution.w) <= 1e-9


def test_sharded_refuses_w1():
    p = synth.make_problem(4, M=600, G=8)
    cfg = api.PcgConfig(tol_rel=p.tol_rel, max_iter=20, xv_mode="qr")
    import torch
    grp = api.LocalGroup(1)
    X = torch.from_numpy(np.ascontiguousarray(p.X.T)).cuda()
    Y = torch.from_numpy(np.ascontiguousarray(p.Y.T)).cuda()
    op = api.GpuSurPreconditioner.from_device_local_group(grp, 0, p.G, p.M, p.M, p.nb, X.data_ptr(), p.M,
                                                          Y.data_ptr(), p.M, p.omega)
    with pytest.raises(api.GlsError):
        api.pcg_aug(None, op, w1=np.ones(op.m), config=cfg)
    op.close()
    grp.close()


# ------------------------------------------------------------------------------------------ staged updates
def test_stage_overlaps_and_matches_update():
    """glsgpu_sur_stage / _update_staged: a solve while the next model uploads (xv_mode QR never reads X) is
    bitwise the solve without staging; the staged model then solves bitwise as a fresh handle; X-reading
    paths refuse while X belongs to the next model."""
    import torch
    p1 = synth.make_problem(4, M=1500, G=24)
    p2 = synth.make_problem(4, M=1500, G=24, seed=77)
    p2.omega = p1.omega
    cfg = api.PcgConfig(tol_rel=1e-10, max_iter=200, xv_mode="qr", diag_every=1)
    op = api.sur_preconditioner(api.sur_from_problem(p1))
    ref1 = api.pcg_aug(None, op, config=cfg, true_beta=p1.beta)
    X2 = torch.from_numpy(np.ascontiguousarray(p2.X.T)).pin_memory()
    Y2 = torch.from_numpy(np.ascontiguousarray(p2.Y.T)).pin_memory()
    op.stage(X2, Y2)
    during = api.pcg_aug(None, op, config=cfg, true_beta=p1.beta)
    assert during.solution.iterations == ref1.solution.iterations
    assert np.array_equal(during.solution.b, ref1.solution.b)
    assert np.array_equal(during.trace.rows["aug_residual_norm"], ref1.trace.rows["aug_residual_norm"], equal_nan=True)
    with pytest.raises(api.GlsError):
        api.pcg_aug(None, op, config=api.PcgConfig(tol_rel=1e-10, max_iter=5, xv_mode="x"))
    with pytest.raises(api.GlsError):
        op.refactor()
    with pytest.raises(api.GlsError):
        op.stage(X2, Y2)  # one staged upload at a time
    op.update_staged()
    g2 = api.pcg_aug(None, op, config=cfg, true_beta=p2.beta)
    f2 = api.pcg_aug(api.sur_from_problem(p2), config=cfg, true_beta=p2.beta)
    assert g2.solution.iterations == f2.solution.iterations
    assert np.array_equal(g2.solution.b, f2.solution.b)
    # X is resident again: X-mode solves work
    api.pcg_aug(None, op, config=api.PcgConfig(tol_rel=1e-10, max_iter=5, xv_mode="x"))
    op.close()


def test_qr_mode_diagnostics_from_q():
    """In xv_mode QR the trace diagnostics read Q and R instead of X (X est = Q s / w, X'w = R'Q'w / w): the
    same values as the X-side diagnostics to rounding."""
    p = synth.make_problem(1, M=500, G=16)
    p.scale = np.linspace(0.5, 2.0, p.G)
    sur = api.sur_from_problem(p)
    op = api.sur_preconditioner(sur, block_scale=p.scale)
    gx = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=1e-12, max_iter=60, xv_mode="x", diag_every=1),
                     true_beta=p.beta)
    gq = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=1e-12, max_iter=60, xv_mode="qr", diag_every=1),
                     true_beta=p.beta)
    for col in ("aug_residual_norm", "rmse"):
        a, b = gq.trace.rows[col][:20], gx.trace.rows[col][:20]
        assert np.allclose(a, b, rtol=1e-9, atol=1e-9 * np.nanmax(np.abs(b)), equal_nan=True), col
    # |X'w| is a roundoff-level quantity (w stays feasible): the two forms agree at that level
    scale = float(np.nanmax(gx.trace.rows["aug_residual_norm"][:20]))
    assert np.allclose(gq.trace.rows["dual_feas_norm"][:20], gx.trace.rows["dual_feas_norm"][:20], rtol=0,
                       atol=1e-10 * scale)


def test_host_sharded_single_rank_update_and_stage():
    """glsgpu_sur_create_sharded_host + update / stage on a 1-rank NCCL communicator (the N > 1 e2e path)."""
    import torch
    p1 = synth.make_problem(4, M=2000, G=16)
    p2 = synth.make_problem(4, M=2000, G=16, seed=5)
    p2.omega = p1.omega
    cfg = api.PcgConfig(tol_rel=1e-10, max_iter=100, xv_mode="qr", diag_every=0)
    op = api.GpuSurPreconditioner.from_host_sharded(p1.G, p1.M, p1.M, p1.nb, p1.X, p1.Y, p1.omega,
                                                    api.nccl_unique_id(), 0, 1)
    g1 = api.pcg_aug(None, op, config=cfg)
    f1 = api.pcg_aug(api.sur_from_problem(p1), config=cfg)
    assert g1.solution.iterations == f1.solution.iterations
    assert rel(g1.solution.b, f1.solution.b) <= 1e-12
    op.update(p2.X, p2.Y)
    g2 = api.pcg_aug(None, op, config=cfg)
    X1 = torch.from_numpy(np.ascontiguousarray(p1.X.T)).pin_memory()
    Y1 = torch.from_numpy(np.ascontiguousarray(p1.Y.T)).pin_memory()
    op.stage(X1, Y1)
    op.update_staged()
    g1b = api.pcg_aug(None, op, config=cfg)
    assert np.array_equal(g1b.solution.b, g1.solution.b)
    f2 = api.pcg_aug(api.sur_from_problem(p2), config=cfg)
    assert rel(g2.solution.b, f2.solution.b) <= 1e-12
    op.close()
