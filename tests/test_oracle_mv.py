"""CPU tests of the MVRGLM row: the oracle's restatement of
pcg_aug(embed_mvrglm(mv), *mvrglm_preconditioner(mv[, z_scale, c_scale]), ...) and of mv_reduce, pinned
BITWISE to the reference itself (oracle/_ref) and to the reference-generated fixtures tests/golden/mv_*.npz
(tests/golden/make_golden.py --mv); plus the host-side model checks and the harness's K1 / K2 auxiliary
choice (proj/src/experiments.cpp:826-851).
"""
import glob
import os

import numpy as np
import pytest

import oracle
from paper_2510_14471_b200 import api, synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _same(a, b):
    return np.array_equal(a, b, equal_nan=True)


def golden_mv(z):
    G, M0, N0 = int(z["G"]), int(z["M0"]), int(z["N0"])
    roff, ridx = z["roff"], z["ridx"]
    restr = [np.asarray(ridx[roff[i]:roff[i + 1]], dtype=np.int64) for i in range(G)]
    p = synth.MvProblem("golden", G, M0, N0, np.asfortranarray(z["Z0"]), np.asfortranarray(z["Y"]),
                        np.asfortranarray(z["omega"]), restr, z["beta"], float(z["tol_rel"]), int(z["max_iter"]))
    if z["z_scale"].size:
        p.z_scale = z["z_scale"]
    if z["c_scale"].size:
        p.c_scale = z["c_scale"]
    w1 = z["w1"] if z["w1"].size else None
    z1 = z["z1"] if z["z1"].size else None
    return p, w1, z1


def assert_bitwise(o, r):
    assert o.iterations == r.iterations and o.termination == r.termination
    assert o.breakdown_iteration == r.breakdown_iteration and o.w1_projected == r.w1_projected
    assert o.residual_seminorm == r.residual_seminorm
    assert _same(o.b, r.b) and _same(o.w, r.w)
    for f in ("iter", "c", "aug_residual_norm", "dual_feas_norm", "rmse"):
        assert _same(o.trace[f], r.trace[f]), f
    assert o.sigma_scale == r.sigma_scale


MV_GOLDEN = sorted(glob.glob(os.path.join(GOLDEN, "mv_*.npz")))


@pytest.mark.parametrize("path", MV_GOLDEN, ids=os.path.basename)
def test_oracle_mv_matches_reference_golden(oracle_mod, path):
    z = np.load(path)
    p, w1, z1 = golden_mv(z)
    o = oracle.solve_mv(p, cfg=oracle.make_config(tol_rel=p.tol_rel, max_iter=p.max_iter), w1=w1, z1=z1,
                        beta_true=p.beta)
    assert o.iterations == int(z["iterations"]) and o.termination == str(z["termination"])
    assert o.breakdown_iteration == (None if int(z["breakdown_iteration"]) < 0 else int(z["breakdown_iteration"]))
    assert _same(o.b, z["b"]) and _same(o.w, z["w"])
    assert o.residual_seminorm == float(z["residual_seminorm"])
    for f in ("iter", "c", "aug_residual_norm", "dual_feas_norm", "rmse"):
        assert _same(o.trace[f], z["trace"][f]), f
    assert o.sigma_scale == float(z["sigma_scale"])


def test_golden_reduced_inputs_are_the_reference_mv_reduce(oracle_mod):
    """mv_c3red*: the stored reduced model is the reference's mv_reduce of the stored full model, and the
    oracle's restated mv_reduce reproduces it bitwise."""
    for name in ("mv_c3red.npz", "mv_c3red_k1.npz", "mv_c3red_k2.npz"):
        z = np.load(os.path.join(GOLDEN, name))
        full = synth.MvProblem("full", int(z["G"]), z["full_Z0"].shape[0], int(z["N0"]),
                               np.asfortranarray(z["full_Z0"]), np.asfortranarray(z["full_Y"]), z["omega"], [], None,
                               1e-10)
        R, QtY = oracle.mv_reduce(full)
        assert _same(R, z["Z0"]) and _same(QtY, z["Y"])


MV_CASES = [
    ("random", lambda: synth.random_mv(3, 30, 5, seed=31), None),
    ("scaled", lambda: synth.random_mv(4, 25, 6, seed=32), "custom"),
    ("c3_mv_M300", lambda: synth.make_mv_problem(3, M=300, G=6, N=12), None),
    ("c3_mv_M300_k1", lambda: synth.make_mv_problem(3, M=300, G=6, N=12), "k1"),
    ("c3_mv_M300_k2", lambda: synth.make_mv_problem(3, M=300, G=6, N=12), "k2"),
]


def _with_scales(p, how):
    if how == "custom":
        p.z_scale = np.linspace(0.5, 2.0, p.G)
        p.c_scale = np.linspace(3.0, 0.25, p.G)
    elif how in ("k1", "k2"):
        p.z_scale, p.c_scale = api.auxiliary_scales(p.omega, how, z0=p.Z0)
    return p


@pytest.mark.parametrize("name,mk,how", MV_CASES, ids=[c[0] for c in MV_CASES])
def test_oracle_mv_bitwise_equals_reference(oracle_mod, have_ref, name, mk, how):
    if not have_ref:
        pytest.skip("oracle/_ref/libglsref.so not built (needs /root/reference)")
    p = _with_scales(mk(), how)
    p.max_iter = 3 * (p.k + 1) + 10  # the harness's MVRGLM budget (experiments.cpp:553-554)
    o = oracle.solve_mv(p, "oracle", beta_true=p.beta)
    r = oracle.solve_mv(p, "ref", beta_true=p.beta)
    assert_bitwise(o, r)
    assert o.counters is None and r.counters[0] == p.G  # factorizations == G


def test_oracle_mv_probes_bitwise(oracle_mod, have_ref):
    if not have_ref:
        pytest.skip("reference not built")
    p = _with_scales(synth.random_mv(4, 20, 5, seed=33), "custom")
    r = np.random.default_rng(4)
    xi, v = r.standard_normal(p.m), r.standard_normal(p.n)
    for kind, vec in (("pi", xi), ("xstar_t", xi), ("xstar", v)):
        assert _same(oracle.mv_apply(p, kind, vec, "oracle"), oracle.mv_apply(p, kind, vec, "ref")), kind
    R, Q = oracle.mv_reduce(p)
    R2, Q2 = oracle.mv_reduce(p, "ref")
    assert _same(R, R2) and _same(Q, Q2)


def test_oracle_mv_embedded_operators(oracle_mod):
    """The structured X / X' / Sigma applies equal the dense embed_mvrglm matrices (structured.cpp:77-95)."""
    p = synth.random_mv(3, 12, 4, seed=34)
    G, M0, N0, m, k = p.G, p.M0, p.N0, p.G * p.M0, p.k
    X = np.zeros((m + k, G * N0))
    row = m
    for i in range(G):
        X[i * M0:(i + 1) * M0, i * N0:(i + 1) * N0] = p.Z0
        for c in p.restrictions[i]:
            X[row, i * N0 + c] = 1.0
            row += 1
    S = np.zeros((m + k, m + k))
    S[:m, :m] = np.kron(p.omega, np.eye(M0))
    r = np.random.default_rng(5)
    v, w = r.standard_normal(G * N0), r.standard_normal(m + k)
    assert np.allclose(oracle.mv_apply(p, "x", v), X @ v, rtol=1e-14, atol=1e-13)
    assert np.allclose(oracle.mv_apply(p, "xt", w), X.T @ w, rtol=1e-14, atol=1e-13)
    assert np.allclose(oracle.mv_apply(p, "sigma", w), S @ w, rtol=1e-14, atol=1e-13)
    # X* is a right inverse of X' on the parameter space; Pi annihilates range(X)
    xs = oracle.mv_apply(p, "xstar", v)
    assert np.allclose(X.T @ xs, v, rtol=1e-11, atol=1e-11)
    assert np.linalg.norm(oracle.mv_apply(p, "pi", X @ v)) <= 1e-11 * np.linalg.norm(X @ v)


def test_mv_error_paths(oracle_mod):
    p = synth.random_mv(3, 10, 4, seed=35)
    q = synth.MvProblem("bad", p.G, p.M0, p.N0, p.Z0, p.Y, p.omega, p.restrictions, p.beta, 1e-10,
                        z_scale=np.array([1.0, -1.0, 1.0]))
    with pytest.raises(oracle.OracleError) as e:
        oracle.solve_mv(q)
    assert e.value.kind == "SingularD"
    # rank-deficient stacked block: a duplicated Z0 column that no restriction separates
    Z = p.Z0.copy(order="F")
    Z[:, 1] = Z[:, 0]
    restr = [np.zeros(0, dtype=np.int64)] * p.G
    q = synth.MvProblem("bad", p.G, p.M0, p.N0, Z, p.Y, p.omega, restr, p.beta, 1e-10)
    with pytest.raises(oracle.OracleError) as e:
        oracle.solve_mv(q)
    assert e.value.kind == "RankDeficient" and "block 0" in str(e.value)


def test_make_mvrglm_validation_mirrors_reference():
    z0 = np.ones((5, 3))
    y = np.ones((5, 2))
    om = np.eye(2)
    with pytest.raises(api.DimensionMismatch, match="Z0 must be tall"):
        api.make_mvrglm(np.ones((2, 3)), np.ones((2, 2)), om, [[], []])
    with pytest.raises(api.DimensionMismatch, match="row mismatch"):
        api.make_mvrglm(z0, np.ones((4, 2)), om, [[], []])
    with pytest.raises(api.DimensionMismatch, match="G x G"):
        api.make_mvrglm(z0, y, np.eye(3), [[], []])
    with pytest.raises(api.DimensionMismatch, match="one list per equation"):
        api.make_mvrglm(z0, y, om, [[]])
    with pytest.raises(api.DimensionMismatch, match="out of range"):
        api.make_mvrglm(z0, y, om, [[3], []])
    with pytest.raises(api.DimensionMismatch, match="strictly increasing"):
        api.make_mvrglm(z0, y, om, [[1, 1], []])
    mv = api.make_mvrglm(z0, y, om, [[0, 2], [1]])
    roff, ridx = mv.csr()
    assert list(roff) == [0, 2, 3] and list(ridx) == [0, 2, 1] and mv.total_restrictions() == 3


def test_auxiliary_scales_follow_the_harness():
    """K1 = alpha I (alpha = max Omega_ii), K2 = diag(Omega); constraint rows scaled by |Z0|_F^2 / N0
    (experiments.cpp:826-847)."""
    om = np.array([[2.0, 0.3, 0.1], [0.3, 5.0, 0.2], [0.1, 0.2, 1.5]])
    z0 = np.arange(1.0, 13.0).reshape(4, 3, order="F")
    zs2 = float(np.sum(z0 * z0)) / 3.0
    k1z, k1c = api.auxiliary_scales(om, "k1", z0=z0)
    k2z, k2c = api.auxiliary_scales(om, "k2", z0=z0)
    assert np.array_equal(k1z, [5.0, 5.0, 5.0]) and np.allclose(k1c, 5.0 / zs2, rtol=1e-15)
    assert np.array_equal(k2z, [2.0, 5.0, 1.5]) and np.allclose(k2c, np.array([2.0, 5.0, 1.5]) / zs2, rtol=1e-15)
    assert np.array_equal(api.auxiliary_scales(om, "k1"), [5.0, 5.0, 5.0])


def test_mv_model_is_config3(oracle_mod):
    """make_mv_problem(3) and make_problem(3) are the same draws: the SUR of the kept columns
    (sur_from_exclusions, experiments.cpp:467-480) is config 3's SUR, and both routes estimate the same
    GLS coefficients."""
    mv = synth.make_mv_problem(3, M=240, G=6, N=10)
    sp = synth.make_problem(3, M=240, G=6, N=10)
    s2 = mv.to_sur()
    assert _same(s2.X, sp.X) and _same(s2.Y, sp.Y) and _same(s2.beta, sp.beta)
    o_sur = oracle.solve(s2, cfg=oracle.make_config(tol_rel=1e-13))
    mv.z_scale, mv.c_scale = api.auxiliary_scales(mv.omega, "k2", z0=mv.Z0)
    o_mv = oracle.solve_mv(mv, cfg=oracle.make_config(tol_rel=1e-12, max_iter=3 * (mv.k + 1) + 10))
    b = mv.gather_sur(o_mv.b)
    assert np.linalg.norm(b - o_sur.b) <= 1e-6 * np.linalg.norm(o_sur.b)
    # the restricted entries of the MVRGLM estimate are (numerically) zero
    full = o_mv.b.reshape(mv.G, mv.N0)
    for i, r in enumerate(mv.restrictions):
        assert np.max(np.abs(full[i, r]), initial=0.0) <= 1e-8 * np.max(np.abs(full))
