"""GPU tests of the PCG-NE comparison solver (glsgpu_pcg_ne, pcg_normal_equations of pcg.cpp:364-511) against
the restatement (bitwise the reference, tests/test_oracle_ne.py) and the reference fixtures ne_*.npz.
Sigma^-1 is applied on the device as a Kronecker pass with Omega^-1 instead of the reference's per-row
triangular solves, so the bar is the SUR one: same termination and iterations, b to 1e-10, where the run is
not decided by roundoff (MaxIter runs compare the trace to 1e-8 relative)."""
import glob
import os

import numpy as np
import pytest

import oracle
from paper_2510_14471_b200 import api, synth

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def require_device():
    assert api.device_count() > 0, "no CUDA device: the GPU tests must run on the B200 box (no CPU fallback exists)"


def golden_problem(z):
    return synth.SurProblem("g", int(z["G"]), int(z["M"]), z["nb"], np.asfortranarray(z["X"]), np.asfortranarray(z["Y"]),
                            np.asfortranarray(z["omega"]), z["beta"], float(z["tol_rel"]), int(z["max_iter"]))


def check(g, o_b, o_iters, o_term, o_c):
    s = g.solution
    assert s.termination.name == o_term
    assert s.iterations == o_iters
    assert rel(s.b, o_b) <= 1e-9, rel(s.b, o_b)
    k = min(len(o_c), len(g.trace.rows), 50)
    assert np.allclose(g.trace.rows["c"][:k], o_c[:k], rtol=1e-8, atol=0)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "ne_*.npz"))), ids=os.path.basename)
def test_ne_golden(path):
    z = np.load(path)
    p = golden_problem(z)
    g = api.pcg_normal_equations(api.sur_from_problem(p), api.PcgConfig(tol_rel=p.tol_rel, max_iter=p.max_iter),
                                 true_beta=p.beta)
    check(g, z["b"], int(z["iterations"]), str(z["termination"]), z["trace"]["c"])
    assert rel(g.solution.w, z["w"]) <= 1e-8


@pytest.mark.parametrize("name,mk,tol,mx", [("c0", lambda: synth.make_problem(0), 1e-12, 400),
                                            ("c4_G64_M2000", lambda: synth.make_problem(4, M=2000, G=64), 1e-10, 150)])
def test_ne_parity(name, mk, tol, mx):
    p = mk()
    o = oracle.solve_ne(p, cfg=oracle.make_config(tol_rel=tol, max_iter=mx), beta_true=p.beta)
    g = api.pcg_normal_equations(api.sur_from_problem(p), api.PcgConfig(tol_rel=tol, max_iter=mx), true_beta=p.beta)
    check(g, o.b, o.iterations, o.termination, o.trace["c"])
    # the normal-equation and augmented solves estimate the same coefficients
    aug = api.pcg_aug(api.sur_from_problem(p), config=api.PcgConfig(tol_rel=1e-12, max_iter=mx, diag_every=0))
    if o.termination == "Converged":
        assert rel(g.solution.b, aug.solution.b) <= 1e-8


def test_ne_singular_covariance():
    p = synth.make_problem(2, M=200, G=16)       # Omega = L L' with L 16 x 32 is PD; make it rank 3
    L = np.random.default_rng(1).standard_normal((p.G, 3))
    p.omega = np.asfortranarray(L @ L.T)
    with pytest.raises(api.SingularCovariance):
        api.pcg_normal_equations(api.sur_from_problem(p), api.PcgConfig(max_iter=5))
