"""CPU tests of the PCG-NE comparison solver: the SUR-structured restatement of
pcg_normal_equations(embed_sur(sur), nullptr, cfg, true_beta) (proj/src/pcg.cpp:364-511) is bitwise the
reference (the dense m x m Cholesky of Sigma = Omega (x) I_M is L (x) I_M by the same loop), against the
reference-generated fixtures tests/golden/ne_*.npz and live against oracle/_ref."""
import glob
import os

import numpy as np
import pytest

import oracle
from paper_2510_14471_b200 import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _same(a, b):
    return np.array_equal(a, b, equal_nan=True)


def golden_problem(z):
    return synth.SurProblem("g", int(z["G"]), int(z["M"]), z["nb"], np.asfortranarray(z["X"]), np.asfortranarray(z["Y"]),
                            np.asfortranarray(z["omega"]), z["beta"], float(z["tol_rel"]), int(z["max_iter"]))


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "ne_*.npz"))), ids=os.path.basename)
def test_oracle_ne_matches_reference_golden(oracle_mod, path):
    z = np.load(path)
    p = golden_problem(z)
    o = oracle.solve_ne(p, cfg=oracle.make_config(tol_rel=p.tol_rel, max_iter=p.max_iter), beta_true=p.beta)
    assert o.iterations == int(z["iterations"]) and o.termination == str(z["termination"])
    assert _same(o.b, z["b"]) and _same(o.w, z["w"])
    assert o.residual_seminorm == float(z["residual_seminorm"])
    for f in ("iter", "c", "aug_residual_norm", "dual_feas_norm", "rmse"):
        assert _same(o.trace[f], z["trace"][f]), f


def test_oracle_ne_bitwise_live_and_singular_covariance(oracle_mod, have_ref):
    if not have_ref:
        pytest.skip("reference not built")
    p = synth.make_problem(0, M=50, G=5)
    o = oracle.solve_ne(p, beta_true=p.beta)
    r = oracle.solve_ne(p, "ref", beta_true=p.beta)
    assert o.iterations == r.iterations and _same(o.b, r.b) and _same(o.w, r.w)
    assert _same(o.trace["c"], r.trace["c"])
    q = synth.make_problem(2, M=40, G=10)
    L = np.random.default_rng(1).standard_normal((q.G, 3))
    q.omega = np.asfortranarray(L @ L.T)         # rank 3: not positive definite
    for kind in ("oracle", "ref"):
        with pytest.raises(oracle.OracleError) as e:
            oracle.solve_ne(q, kind)
        assert e.value.kind == "SingularCovariance"
