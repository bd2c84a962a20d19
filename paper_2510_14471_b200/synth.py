"""Seeded synthetic SUR problems with the shapes and distributions of BASELINE.json:configs.

There is no public dataset behind this path: every config is synthetic.  Each config
has a master seed 1000 + c and independent numpy Philox streams per ingredient (X, beta, L, Z,
widths / B-pattern), so a scaled-down variant (smaller M) of a config draws from the same
distributions.  Generation is host-side numpy (tests, parity runs, the CPU baseline sample); the
full-size c4 bench inputs (65.5 GB of X) are generated on the device by the library instead
(``glsgpu_synth_normal``), see bench.py.

Layouts follow the reference (proj/include/gls/dense_matrix.hpp:13-15): every matrix is
column-major.  X is the concatenation [X_0 | X_1 | ...] as one M x n Fortran-ordered array; Y is
M x G (equation b in column b, i.e. rows [b*M, (b+1)*M) of the stacked y of embed_sur,
proj/src/structured.cpp:107-119).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

__all__ = ["SurProblem", "MvProblem", "CONFIGS", "make_problem", "make_mv_problem", "omega_half", "config_meta"]


@dataclasses.dataclass
class SurProblem:
    name: str
    G: int
    M: int
    nb: np.ndarray            # int64 widths n_i
    X: np.ndarray             # (M, n) float64, Fortran order
    Y: np.ndarray             # (M, G) float64, Fortran order
    omega: np.ndarray         # (G, G) float64, Fortran order, symmetric
    beta: np.ndarray          # (n,) true coefficients
    tol_rel: float
    max_iter: int = 0         # 0 -> m - n + 1 (proj/src/pcg.cpp:34)
    scale: Optional[np.ndarray] = None  # per-block auxiliary variances (D = I when None)

    @property
    def n(self) -> int:
        return int(self.nb.sum())

    @property
    def m(self) -> int:
        return self.M * self.G


@dataclasses.dataclass
class MvProblem:
    """Multivariate model Y = Z0 B + U with exclusion restrictions (gls::MvRglm,
    proj/include/gls/structured.hpp:37-52): restrictions[i] lists the zero-forced rows of B[:, i]."""
    name: str
    G: int
    M0: int
    N0: int
    Z0: np.ndarray            # (M0, N0) float64, Fortran order
    Y: np.ndarray             # (M0, G) float64, Fortran order
    omega: np.ndarray         # (G, G) float64, symmetric
    restrictions: list        # G int64 arrays, strictly increasing, < N0
    beta: np.ndarray          # (G * N0,) true coefficients, zeros at the restricted entries
    tol_rel: float
    max_iter: int = 0
    z_scale: Optional[np.ndarray] = None  # per-equation auxiliary variances (observation rows)
    c_scale: Optional[np.ndarray] = None  # per-equation auxiliary variances (constraint rows)

    @property
    def k(self) -> int:
        return int(sum(len(r) for r in self.restrictions))

    @property
    def m(self) -> int:             # rows of embed_mvrglm: G M0 observation rows + k constraint rows
        return self.G * self.M0 + self.k

    @property
    def n(self) -> int:
        return self.G * self.N0

    def csr(self):
        """restrictions as CSR (roff[G + 1], ridx), the C-ABI / oracle form."""
        roff = np.zeros(self.G + 1, dtype=np.int64)
        roff[1:] = np.cumsum([len(r) for r in self.restrictions])
        ridx = (np.concatenate([np.asarray(r, dtype=np.int64) for r in self.restrictions])
                if roff[-1] else np.zeros(1, dtype=np.int64))
        return roff, np.ascontiguousarray(ridx, dtype=np.int64)

    def kept(self):
        """kept_columns (proj/src/experiments.cpp:453-465): the unrestricted rows of each B column."""
        return [np.setdiff1d(np.arange(self.N0), r) for r in self.restrictions]

    def to_sur(self) -> "SurProblem":
        """sur_from_exclusions (proj/src/experiments.cpp:467-480): X_i = Z0[:, kept_i]."""
        kept = self.kept()
        nb = np.array([len(k) for k in kept], dtype=np.int64)
        X = np.asfortranarray(np.concatenate([self.Z0[:, k] for k in kept], axis=1))
        beta = np.concatenate([self.beta[i * self.N0 + k] for i, k in enumerate(kept)])
        return SurProblem(self.name + "-sur", self.G, self.M0, nb, X, self.Y, self.omega, beta, self.tol_rel,
                          self.max_iter)

    def gather_sur(self, b_full: np.ndarray) -> np.ndarray:
        """gather_sur_params (proj/src/experiments.cpp:482-489): the kept entries of a G N0 estimate."""
        return np.concatenate([b_full[i * self.N0 + k] for i, k in enumerate(self.kept())])


# c -> (G, M, widths rule, Omega rule, tol, max_iter); BASELINE.json:configs[c]
CONFIGS = {
    0: dict(G=10, M=1000, widths="const:20", omega="llt+0.1", tol=1e-12, max_iter=0),
    1: dict(G=100, M=10000, widths="uniform:5:50", omega="llt+0.1", tol=1e-12, max_iter=0),
    2: dict(G=64, M=50000, widths="const:16", omega="rank:32", tol=1e-10, max_iter=0),
    3: dict(G=64, M=100000, widths="pattern:200", omega="llt+0.1", tol=1e-10, max_iter=0),
    4: dict(G=256, M=1000000, widths="const:32", omega="llt+0.1", tol=1e-10, max_iter=200),
}


def config_meta(c: int) -> dict:
    return dict(CONFIGS[c])


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed, stream]))


def omega_half(omega: np.ndarray) -> np.ndarray:
    """Symmetric PSD square root via the eigendecomposition, negative eigenvalues clamped to 0."""
    vals, vecs = np.linalg.eigh(omega)
    vals = np.clip(vals, 0.0, None)
    h = (vecs * np.sqrt(vals)) @ vecs.T
    return np.asfortranarray(0.5 * (h + h.T))


def make_omega(G: int, rule: str, seed: int) -> np.ndarray:
    r = _rng(seed, 2)
    if rule == "llt+0.1":
        L = np.tril(r.standard_normal((G, G)))
        om = L @ L.T + 0.1 * np.eye(G)
    elif rule.startswith("rank:"):
        k = int(rule.split(":")[1])
        L = r.standard_normal((G, k))
        om = L @ L.T
    else:
        raise ValueError(rule)
    om = 0.5 * (om + om.T)  # the Kronecker apply assumes symmetry (proj/src/operators.cpp:46)
    return np.asfortranarray(om)


def make_problem(c: int, M: Optional[int] = None, G: Optional[int] = None, N: Optional[int] = None,
                 seed: Optional[int] = None, with_data: bool = True) -> SurProblem:
    """Config c of BASELINE.json, optionally scaled down (M rows, G equations, N base params for c3)."""
    cfg = CONFIGS[c]
    G = int(G if G is not None else cfg["G"])
    M = int(M if M is not None else cfg["M"])
    seed = int(seed if seed is not None else 1000 + c)
    rule = cfg["widths"]
    omega = make_omega(G, cfg["omega"], seed)
    rz = _rng(seed, 3)
    if rule.startswith("pattern:"):
        # constrained multivariate model: X_i = kept columns of X0 (proj/src/experiments.cpp:453-489)
        N0 = int(N if N is not None else int(rule.split(":")[1]))
        rp = _rng(seed, 4)
        zero = rp.random((N0, G)) < 0.5          # Bernoulli(1/2) zero pattern per entry
        for i in range(G):                        # keep every equation identified
            if zero[:, i].all():
                zero[rp.integers(N0), i] = False
        B = _rng(seed, 1).standard_normal((N0, G))
        B[zero] = 0.0
        kept = [np.flatnonzero(~zero[:, i]) for i in range(G)]
        nb = np.array([len(k) for k in kept], dtype=np.int64)
        if not with_data:
            return SurProblem(f"c{c}", G, M, nb, None, None, omega, None, cfg["tol"], cfg["max_iter"])
        X0 = _rng(seed, 0).standard_normal((M, N0))
        X = np.asfortranarray(np.concatenate([X0[:, k] for k in kept], axis=1))
        beta = np.concatenate([B[k, i] for i, k in enumerate(kept)])
        mean = X0 @ B
    else:
        if rule.startswith("const:"):
            nb = np.full(G, int(rule.split(":")[1]), dtype=np.int64)
        else:
            _, lo, hi = rule.split(":")
            nb = _rng(seed, 4).integers(int(lo), int(hi) + 1, size=G).astype(np.int64)
        if not with_data:
            return SurProblem(f"c{c}", G, M, nb, None, None, omega, None, cfg["tol"], cfg["max_iter"])
        n = int(nb.sum())
        X = np.asfortranarray(_rng(seed, 0).standard_normal((n, M)).T)
        beta = _rng(seed, 1).standard_normal(n)
        mean = np.empty((M, G))
        p = 0
        for i in range(G):
            mean[:, i] = X[:, p:p + nb[i]] @ beta[p:p + nb[i]]
            p += nb[i]
    Z = rz.standard_normal((G, M)).T
    E = Z @ omega_half(omega)
    Y = np.asfortranarray(mean + E)
    return SurProblem(f"c{c}", G, M, nb, X, Y, omega, beta, cfg["tol"], cfg["max_iter"])


def random_sur(G: int, M: int, nb, seed: int, cond_omega: Optional[float] = None) -> SurProblem:
    """Small generic SUR problem (edge-case tests): Omega = L L' + 0.1 I, X, beta ~ N(0,1)."""
    nb = np.asarray(nb, dtype=np.int64)
    n = int(nb.sum())
    r = _rng(seed, 0)
    X = np.asfortranarray(r.standard_normal((M, n)))
    beta = r.standard_normal(n)
    L = np.tril(r.standard_normal((G, G)))
    omega = L @ L.T + 0.1 * np.eye(G)
    omega = np.asfortranarray(0.5 * (omega + omega.T))
    mean = np.empty((M, G))
    p = 0
    for i in range(G):
        mean[:, i] = X[:, p:p + nb[i]] @ beta[p:p + nb[i]]
        p += nb[i]
    Y = np.asfortranarray(mean + r.standard_normal((M, G)) @ omega_half(omega))
    return SurProblem(f"rand{seed}", G, M, nb, X, Y, omega, beta, 1e-12, 0)


def make_mv_problem(c: int = 3, M: Optional[int] = None, G: Optional[int] = None, N: Optional[int] = None,
                    seed: Optional[int] = None) -> MvProblem:
    """Config 3 as the multivariate model it is (BASELINE.json:configs[3]): the same draws as
    make_problem(3, ...), with the Bernoulli(1/2) zero pattern of B as exclusion restrictions."""
    cfg = CONFIGS[c]
    assert cfg["widths"].startswith("pattern:")
    G = int(G if G is not None else cfg["G"])
    M = int(M if M is not None else cfg["M"])
    seed = int(seed if seed is not None else 1000 + c)
    N0 = int(N if N is not None else int(cfg["widths"].split(":")[1]))
    omega = make_omega(G, cfg["omega"], seed)
    rp = _rng(seed, 4)
    zero = rp.random((N0, G)) < 0.5
    for i in range(G):
        if zero[:, i].all():
            zero[rp.integers(N0), i] = False
    B = _rng(seed, 1).standard_normal((N0, G))
    B[zero] = 0.0
    X0 = np.asfortranarray(_rng(seed, 0).standard_normal((M, N0)))
    Z = _rng(seed, 3).standard_normal((G, M)).T
    Y = np.asfortranarray(X0 @ B + Z @ omega_half(omega))
    restr = [np.flatnonzero(zero[:, i]).astype(np.int64) for i in range(G)]
    return MvProblem(f"c{c}-mv", G, M, N0, X0, Y, omega, restr, np.asarray(B.T.reshape(-1), dtype=np.float64),
                     cfg["tol"], cfg["max_iter"])


def random_mv(G: int, M0: int, N0: int, seed: int, frac: float = 0.5) -> MvProblem:
    """Small generic multivariate model with random exclusions (edge-case tests)."""
    r = _rng(seed, 0)
    Z0 = np.asfortranarray(r.standard_normal((M0, N0)))
    zero = r.random((N0, G)) < frac
    for i in range(G):
        if zero[:, i].all():
            zero[0, i] = False
    B = r.standard_normal((N0, G))
    B[zero] = 0.0
    L = np.tril(r.standard_normal((G, G)))
    omega = np.asfortranarray(0.5 * ((L @ L.T + 0.1 * np.eye(G)) + (L @ L.T + 0.1 * np.eye(G)).T))
    Y = np.asfortranarray(Z0 @ B + r.standard_normal((M0, G)) @ omega_half(omega))
    restr = [np.flatnonzero(zero[:, i]).astype(np.int64) for i in range(G)]
    return MvProblem(f"mv{seed}", G, M0, N0, Z0, Y, omega, restr, np.asarray(B.T.reshape(-1)), 1e-12, 0)
