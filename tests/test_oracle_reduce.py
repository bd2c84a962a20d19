"""CPU tests of the sur_reduce row (the paper's Remark 1, structured.cpp:132-178).

The fixtures tests/golden/red_*.npz hold the reference's own reduction (oracle/_ref) and its pcg_aug on the
reduced model (tests/golden/make_golden.py --reduce).  The restatement (oracle) must reproduce the reduced
solve bitwise; the reduction must keep every Gram of the model (X_i'X_j and X_i'Y are invariant under the
rotation onto range(W)), which is what the device reduction is judged by (tests/test_gpu_reduce.py).
"""
import glob
import os

import numpy as np
import pytest

import oracle
from paper_2510_14471_b200 import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RED = sorted(glob.glob(os.path.join(GOLDEN, "red_*.npz")))


def golden_problem(z):
    return synth.SurProblem("g", int(z["G"]), int(z["M"]), z["nb"], np.asfortranarray(z["X"]),
                            np.asfortranarray(z["Y"]), np.asfortranarray(z["omega"]), z["beta"], float(z["tol_rel"]),
                            int(z["max_iter"]))


def reduced_problem(z, X_red=None, Y_red=None):
    q = int(z["q"])
    return synth.SurProblem("r", int(z["G"]), q, z["nb"], np.asfortranarray(z["X_red"] if X_red is None else X_red),
                            np.asfortranarray(z["Y_red"] if Y_red is None else Y_red), np.asfortranarray(z["omega"]),
                            z["beta"], float(z["tol_rel"]), int(z["max_iter"]))


@pytest.mark.parametrize("path", RED, ids=os.path.basename)
def test_oracle_solves_the_reference_reduction_bitwise(oracle_mod, path):
    z = np.load(path)
    red = reduced_problem(z)
    o = oracle.solve(red, cfg=oracle.make_config(tol_rel=red.tol_rel, max_iter=red.max_iter), beta_true=red.beta)
    assert o.iterations == int(z["iterations"]) and o.termination == str(z["termination"])
    assert np.array_equal(o.b, z["b"])
    assert np.array_equal(o.trace["c"], z["trace"]["c"])


@pytest.mark.parametrize("path", RED, ids=os.path.basename)
def test_reference_reduction_fixture_and_invariants(oracle_mod, have_ref, path):
    z = np.load(path)
    p = golden_problem(z)
    X, Y, Xr, Yr = p.X, p.Y, z["X_red"], z["Y_red"]
    # range(W) keeps every Gram of the model
    g, gr = X.T @ X, Xr.T @ Xr
    assert np.linalg.norm(gr - g) <= 1e-12 * np.linalg.norm(g)
    assert np.linalg.norm(Xr.T @ Yr - X.T @ Y) <= 1e-12 * np.linalg.norm(X.T @ Y)
    assert int(z["q"]) == np.linalg.matrix_rank(X)
    if have_ref:
        q, Xr2, Yr2, B = oracle.sur_reduce_ref(p, want_basis=True)
        assert q == int(z["q"]) and np.array_equal(Xr2, Xr) and np.array_equal(Yr2, Yr)
        assert np.max(np.abs(B.T @ B - np.eye(q))) < 1e-13
    # the estimator does not move (Remark 1): the reduced solve's b vs the unreduced solve's
    assert np.linalg.norm(z["b"] - z["b_full"]) <= 1e-7 * np.linalg.norm(z["b_full"])
