"""GPU tests of the PCG-NE comparison solver (glsgpu_pcg_ne, pcg_normal_equations of pcg.cpp:364-511) against
the restatement (bitwise the reference, tests/test_oracle_ne.py) and the reference fixtures ne_*.npz.

The whole CG loop runs on the device (csrc/ne.cuh: graph-captured steps, device-side termination logic), and
Sigma^-1 is the reference's own per-row chol_solve with L = cholesky(Omega) (bitwise per row).  What differs
from the reference is only the summation order of the long sums (X' columns, n-vector dots), so the bar is
the SUR one: same termination and iterations, b to 1e-10 on converged runs; unconverged (MaxIter) runs of
the squared-condition normal equations carry the restatement's own drift under a change of summation order
and are judged against it."""
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


def oracle_pair(p, tol, mx):
    """The restatement (bitwise the reference) with sequential and with pairwise sums: runs that end at MaxIter
    without converging carry the normal equations' rounding drift (1e-6 .. 1e-5 in b between the two)."""
    cfg = oracle.make_config(tol_rel=tol, max_iter=mx)
    L = oracle.lib("oracle")
    o = oracle.solve_ne(p, cfg=cfg, beta_true=p.beta)
    L.orc_set_sum_mode(1)
    try:
        o1 = oracle.solve_ne(p, cfg=cfg, beta_true=p.beta)
    finally:
        L.orc_set_sum_mode(0)
    return o, o1


def check(g, o, o1):
    s = g.solution
    assert s.termination.name == o.termination
    assert s.iterations == o.iterations
    spread = rel(o1.b, o.b)
    bar = 1e-10 if o.termination == "Converged" and spread <= 1e-11 else max(1e-10, 10.0 * spread)
    assert rel(s.b, o.b) <= bar, (rel(s.b, o.b), spread)
    # the c trace agrees while it carries signal (relative to c1; rows at the roundoff floor carry none)
    c_g, c_o, c_1 = np.asarray(g.trace.rows["c"]), np.asarray(o.trace["c"]), np.asarray(o1.trace["c"])
    k = min(len(c_o), len(c_g), len(c_1))
    tol = 10.0 * np.abs(c_1[:k] - c_o[:k]) + 1e-6 * np.abs(c_o[:k]) + 1e-9 * c_o[0]
    sig = c_o[:k] >= 1e-5 * c_o[0]  # below, the normal equations carry their rounding noise
    bad = np.flatnonzero((np.abs(c_g[:k] - c_o[:k]) > tol) & sig)
    assert bad.size == 0, (bad[:5], c_g[bad[:5]], c_o[bad[:5]], c_1[bad[:5]])


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "ne_*.npz"))), ids=os.path.basename)
def test_ne_golden(path):
    z = np.load(path)
    p = golden_problem(z)
    g = api.pcg_normal_equations(api.sur_from_problem(p), api.PcgConfig(tol_rel=p.tol_rel, max_iter=p.max_iter),
                                 true_beta=p.beta)
    o, o1 = oracle_pair(p, p.tol_rel, p.max_iter)
    assert o.iterations == int(z["iterations"]) and np.array_equal(o.b, z["b"])  # the oracle is the fixture
    check(g, o, o1)
    assert rel(g.solution.w, z["w"]) <= max(1e-8, 10.0 * rel(o1.w, o.w))


@pytest.mark.parametrize("name,mk,tol,mx", [("c0", lambda: synth.make_problem(0), 1e-12, 400),
                                            ("c4_G64_M2000", lambda: synth.make_problem(4, M=2000, G=64), 1e-10, 150)])
def test_ne_parity(name, mk, tol, mx):
    p = mk()
    o, o1 = oracle_pair(p, tol, mx)
    g = api.pcg_normal_equations(api.sur_from_problem(p), api.PcgConfig(tol_rel=tol, max_iter=mx), true_beta=p.beta)
    check(g, o, o1)
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
