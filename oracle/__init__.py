"""oracle -- TEST INFRASTRUCTURE ONLY (the parity checker; never the product).

ctypes bindings for
  * liboracle.so      -- the C restatement of the reference's SUR PCG-Aug path (gls_oracle.c), and
  * _ref/libglsref.so -- the UNMODIFIED reference gls_core compiled from /root/reference by
                         oracle/Makefile, driven through ref_shim.cpp's C wrappers.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import
this package.  See gls_oracle.c's header for what is restated from where.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libglsref.so")

TERMINATION = {0: "Converged", 1: "Breakdown", 2: "Stagnation", 3: "MaxIter", 4: "Direct"}
STATUS = {0: "ok", 1: "DimensionMismatch", 2: "RankDeficient", 3: "SingularD", 4: "SingularTriangular",
          5: "SingularCovariance",
          12: "NoMemory", 98: "std::exception", 99: "gls::Error"}


class Config(C.Structure):
    """gls::PcgConfig (proj/include/gls/pcg.hpp:12-30)."""
    _fields_ = [("tol_rel", C.c_double), ("max_iter", C.c_int64), ("breakdown_tol", C.c_double),
                ("stagnation_window", C.c_int64), ("growth_tol", C.c_double), ("growth_window", C.c_int64),
                ("record_z_every", C.c_int64)]


def make_config(tol_rel=1e-10, max_iter=0, breakdown_tol=1e-14, stagnation_window=5, growth_tol=1e4,
                growth_window=10, record_z_every=1) -> Config:
    return Config(tol_rel, max_iter, breakdown_tol, stagnation_window, growth_tol, growth_window, record_z_every)


class TraceRow(C.Structure):
    """gls::PcgTraceRow (proj/include/gls/pcg.hpp:32-39)."""
    _fields_ = [("iter", C.c_int64), ("c", C.c_double), ("aug_residual_norm", C.c_double),
                ("dual_feas_norm", C.c_double), ("rmse", C.c_double), ("elapsed_ns", C.c_int64)]


class Result(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("termination", C.c_int32), ("w1_projected", C.c_int32),
                ("breakdown_iteration", C.c_int64), ("residual_seminorm", C.c_double), ("n_rows", C.c_int64),
                ("sigma_scale", C.c_double)]


TRACE_DTYPE = np.dtype([("iter", np.int64), ("c", np.float64), ("aug_residual_norm", np.float64),
                        ("dual_feas_norm", np.float64), ("rmse", np.float64), ("elapsed_ns", np.int64)])


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"{STATUS.get(code, code)}: {what}")
        self.code = code
        self.kind = STATUS.get(code, str(code))


@dataclasses.dataclass
class SolveOut:
    b: np.ndarray
    w: np.ndarray
    iterations: int
    termination: str
    breakdown_iteration: Optional[int]
    residual_seminorm: float
    w1_projected: bool
    trace: np.ndarray
    sigma_scale: float
    counters: Optional[np.ndarray] = None   # reference CostCounters after the solve (kind="ref")


_P = C.POINTER(C.c_double)
_PI = C.POINTER(C.c_int64)


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.float64 and (a.flags.f_contiguous or a.flags.c_contiguous)
    return a.ctypes.data_as(_P)


def _load(path: str, kind: str):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle all ref` (or __graft_entry__.build())")
    lib = C.CDLL(path)
    if kind == "oracle":
        lib.orc_pcg_aug_sur.restype = C.c_int
        lib.orc_pcg_aug_sur.argtypes = [C.c_int, C.c_int64, _PI, _P, _P, _P, _P, _P, _P, C.POINTER(Config), _P,
                                        _P, _P, C.POINTER(TraceRow), C.c_int64, C.POINTER(Result),
                                        C.POINTER(C.c_int)]
        lib.orc_sur_apply.restype = C.c_int
        lib.orc_sur_apply.argtypes = [C.c_int, C.c_int64, _PI, _P, _P, C.c_int, _P, _P]
        lib.orc_sur_setup.restype = C.c_int
        lib.orc_sur_setup.argtypes = [C.c_int, C.c_int64, _PI, _P, _P, _P, _P, C.POINTER(C.c_int)]
        lib.orc_kron_apply.restype = None
        lib.orc_kron_apply.argtypes = [C.c_int, C.c_int64, _P, _P, _P]
        lib.orc_norm_probe.restype = C.c_double
        lib.orc_norm_probe.argtypes = [C.c_int, C.c_int64, _P, C.c_int64]
        lib.orc_qr_thin.restype = C.c_int
        lib.orc_qr_thin.argtypes = [C.c_int64, C.c_int64, _P, C.c_int64, C.c_double, _P, C.c_int64, _P]
        lib.orc_pcg_aug_mvrglm.restype = C.c_int
        lib.orc_pcg_aug_mvrglm.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _P, _P, _PI, _PI, _P, _P, _P, _P,
                                           C.POINTER(Config), _P, _P, _P, C.POINTER(TraceRow), C.c_int64,
                                           C.POINTER(Result), C.POINTER(C.c_int)]
        lib.orc_mvrglm_apply.restype = C.c_int
        lib.orc_mvrglm_apply.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _P, _PI, _PI, _P, _P, C.c_int, _P, _P]
        lib.orc_mvrglm_norm_probe.restype = C.c_double
        lib.orc_mvrglm_norm_probe.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _P, _PI, _PI]
        lib.orc_pcg_ne_sur.restype = C.c_int
        lib.orc_pcg_ne_sur.argtypes = [C.c_int, C.c_int64, _PI, _P, _P, _P, C.POINTER(Config), _P, _P, _P,
                                       C.POINTER(TraceRow), C.c_int64, C.POINTER(Result)]
        lib.orc_mv_reduce.restype = C.c_int
        lib.orc_mv_reduce.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _P, _P, _P]
        lib.orc_set_threads.restype = None
        lib.orc_set_threads.argtypes = [C.c_int]
        lib.orc_get_threads.restype = C.c_int
        lib.orc_get_threads.argtypes = []
    else:
        lib.ref_pcg_aug_sur.restype = C.c_int
        lib.ref_pcg_aug_sur.argtypes = [C.c_int, C.c_int64, _PI, _P, _P, _P, _P, _P, _P, C.POINTER(Config), _P,
                                        _P, _P, C.POINTER(TraceRow), C.c_int64, C.POINTER(Result),
                                        C.POINTER(C.c_uint64)]
        lib.ref_sur_apply.restype = C.c_int
        lib.ref_sur_apply.argtypes = [C.c_int, C.c_int64, _PI, _P, _P, C.c_int, _P, _P]
        lib.ref_kron_apply.restype = C.c_int
        lib.ref_kron_apply.argtypes = [C.c_int, C.c_int64, _P, _P, _P]
        lib.ref_norm_probe.restype = C.c_double
        lib.ref_norm_probe.argtypes = [C.c_int, C.c_int64, _P]
        lib.ref_qr_thin.restype = C.c_int
        lib.ref_qr_thin.argtypes = [C.c_int64, C.c_int64, _P, _P, _P]
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_pcg_aug_mvrglm.restype = C.c_int
        lib.ref_pcg_aug_mvrglm.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _P, _P, _PI, _PI, _P, _P, _P, _P,
                                           C.POINTER(Config), _P, _P, _P, C.POINTER(TraceRow), C.c_int64,
                                           C.POINTER(Result), C.POINTER(C.c_uint64)]
        lib.ref_mvrglm_apply.restype = C.c_int
        lib.ref_mvrglm_apply.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _PI, _PI, _P, _P, C.c_int, _P, _P]
        lib.ref_pcg_ne_sur.restype = C.c_int
        lib.ref_pcg_ne_sur.argtypes = [C.c_int, C.c_int64, _PI, _P, _P, _P, C.POINTER(Config), _P, _P, _P,
                                       C.POINTER(TraceRow), C.c_int64, C.POINTER(Result)]
        lib.ref_sur_reduce.restype = C.c_int
        lib.ref_sur_reduce.argtypes = [C.c_int, C.c_int64, _PI, _P, _P, C.c_double, C.POINTER(C.c_int64), _P, _P, _P]
        lib.ref_mv_reduce.restype = C.c_int
        lib.ref_mv_reduce.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _P, _P, _P]
    return lib


_libs = {}


def lib(kind: str = "oracle"):
    if kind not in _libs:
        _libs[kind] = _load(ORACLE_SO if kind == "oracle" else REF_SO, kind)
    return _libs[kind]


def set_threads(n: int) -> int:
    """Threads of the restatement's independent per-block / per-tile loops (OpenMP; results are bitwise the
    single-threaded ones).  Returns the count now in effect."""
    L = lib("oracle")
    L.orc_set_threads(int(n))
    return int(L.orc_get_threads())


def threads() -> int:
    return int(lib("oracle").orc_get_threads())


def have(kind: str) -> bool:
    return os.path.exists(ORACLE_SO if kind == "oracle" else REF_SO)


def solve(prob, kind: str = "oracle", cfg: Optional[Config] = None, w1=None, z1=None, trace: bool = True,
          beta_true: Optional[np.ndarray] = None) -> SolveOut:
    """pcg_aug(embed_sur(sur), *sur_preconditioner(sur[, scale]), w1, z1, cfg) on the CPU.

    kind="oracle": the restatement; kind="ref": the literal reference (dense embed; small sizes only).
    """
    L = lib(kind)
    if cfg is None:
        cfg = make_config(tol_rel=prob.tol_rel, max_iter=prob.max_iter)
    nb = np.ascontiguousarray(prob.nb, dtype=np.int64)
    m, n = prob.M * prob.G, int(nb.sum())
    max_iter = cfg.max_iter if cfg.max_iter else m - n + 1
    cap = max_iter + 1 if trace else 0
    rows = (TraceRow * max(cap, 1))()
    b = np.zeros(n)
    w = np.zeros(m)
    res = Result()
    scale = None if prob.scale is None else np.ascontiguousarray(prob.scale, dtype=np.float64)
    w1a = None if w1 is None else np.ascontiguousarray(w1, dtype=np.float64)
    z1a = None if z1 is None else np.ascontiguousarray(z1, dtype=np.float64)
    bt = None if beta_true is None else np.ascontiguousarray(beta_true, dtype=np.float64)
    args = [prob.G, prob.M, nb.ctypes.data_as(_PI), _dp(prob.X), _dp(prob.Y), _dp(prob.omega), _dp(scale), _dp(w1a),
            _dp(z1a), C.byref(cfg), _dp(bt), _dp(b), _dp(w), rows if trace else None, cap, C.byref(res)]
    if kind == "oracle":
        bad = C.c_int(-1)
        st = L.orc_pcg_aug_sur(*args, C.byref(bad))
        if st:
            raise OracleError(st, f"block {bad.value}")
    else:
        counters = np.zeros(6, dtype=np.uint64)
        st = L.ref_pcg_aug_sur(*args, counters.ctypes.data_as(C.POINTER(C.c_uint64)))
        if st:
            raise OracleError(st, L.ref_last_error().decode())
    tr = np.frombuffer(rows, dtype=TRACE_DTYPE, count=min(res.n_rows, cap)).copy() if trace else np.zeros(0, TRACE_DTYPE)
    return SolveOut(b=b, w=w, iterations=int(res.iterations), termination=TERMINATION[res.termination],
                    breakdown_iteration=None if res.breakdown_iteration < 0 else int(res.breakdown_iteration),
                    residual_seminorm=float(res.residual_seminorm), w1_projected=bool(res.w1_projected),
                    trace=tr, sigma_scale=float(res.sigma_scale),
                    counters=counters if kind != "oracle" else None)


def sur_apply(prob, kind_op: str, vec: np.ndarray, kind: str = "oracle") -> np.ndarray:
    """apply_pi / apply_xstar_t / apply_xstar of sur_preconditioner(sur[, scale])."""
    L = lib(kind)
    op = {"pi": 0, "xstar_t": 1, "xstar": 2}[kind_op]
    nb = np.ascontiguousarray(prob.nb, dtype=np.int64)
    m, n = prob.M * prob.G, int(nb.sum())
    out = np.zeros(n if op == 1 else m)
    v = np.ascontiguousarray(vec, dtype=np.float64)
    scale = None if prob.scale is None else np.ascontiguousarray(prob.scale, dtype=np.float64)
    fn = L.orc_sur_apply if kind == "oracle" else L.ref_sur_apply
    st = fn(prob.G, prob.M, nb.ctypes.data_as(_PI), _dp(prob.X), _dp(scale), op, _dp(v), _dp(out))
    if st:
        raise OracleError(st)
    return out


def kron_apply(omega: np.ndarray, x: np.ndarray, M: int, kind: str = "oracle") -> np.ndarray:
    L = lib(kind)
    G = omega.shape[0]
    om = np.asfortranarray(omega, dtype=np.float64)
    xx = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    out = np.zeros(M * G)
    if kind == "oracle":
        L.orc_kron_apply(G, M, _dp(om), _dp(xx), _dp(out))
    else:
        st = L.ref_kron_apply(G, M, _dp(om), _dp(xx), _dp(out))
        if st:
            raise OracleError(st)
    return out


def norm_probe(omega: np.ndarray, M: int, kind: str = "oracle") -> float:
    om = np.asfortranarray(omega, dtype=np.float64)
    if kind == "oracle":
        return lib("oracle").orc_norm_probe(om.shape[0], M, _dp(om), 12)
    return lib("ref").ref_norm_probe(om.shape[0], M, _dp(om))


def sur_setup(prob):
    """Q (M x n) and concatenated R of sur_preconditioner's per-block qr_thin."""
    nb = np.ascontiguousarray(prob.nb, dtype=np.int64)
    n = int(nb.sum())
    Q = np.zeros((prob.M, n), order="F")
    R = np.zeros(int((nb * nb).sum()))
    scale = None if prob.scale is None else np.ascontiguousarray(prob.scale, dtype=np.float64)
    bad = C.c_int(-1)
    st = lib("oracle").orc_sur_setup(prob.G, prob.M, nb.ctypes.data_as(_PI), _dp(prob.X), _dp(scale), _dp(Q), _dp(R),
                                     C.byref(bad))
    if st:
        raise OracleError(st, f"block {bad.value}")
    return Q, R


def diag(kind: str = "oracle", cap: int = 1 << 16):
    """Per-iteration margins of the last restatement solve (DIAGNOSTIC): d / (u.u sigma_scale) of the
    breakdown test and c_next / c_best of the growth test (proj/src/pcg.cpp:144-147,197-200)."""
    L = lib(kind)
    L.orc_diag.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64]
    L.orc_diag.restype = C.c_int64
    d = np.zeros(cap)
    g = np.zeros(cap)
    n = L.orc_diag(d.ctypes.data_as(C.POINTER(C.c_double)), g.ctypes.data_as(C.POINTER(C.c_double)),
                   cap)
    return d[:n], g[:n]


# ------------------------------------------------------------------ MVRGLM (structured.cpp:77-95,121-130,365-414)
def _f(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def solve_mv(prob, kind: str = "oracle", cfg: Optional[Config] = None, w1=None, z1=None, trace: bool = True,
             beta_true: Optional[np.ndarray] = None) -> SolveOut:
    """pcg_aug(embed_mvrglm(mv), *mvrglm_preconditioner(mv[, z_scale, c_scale]), w1, z1, cfg).

    kind="oracle": the restatement; kind="ref": the literal reference (dense embed; small sizes only).
    Vectors use the reference's embedded row order (observation rows per equation, then constraints)."""
    L = lib(kind)
    if cfg is None:
        cfg = make_config(tol_rel=prob.tol_rel, max_iter=prob.max_iter)
    roff, ridx = prob.csr()
    m, n = prob.m, prob.n
    max_iter = cfg.max_iter if cfg.max_iter else m - n + 1
    cap = max_iter + 1 if trace else 0
    rows = (TraceRow * max(cap, 1))()
    b = np.zeros(n)
    w = np.zeros(m)
    res = Result()
    Z0 = np.asfortranarray(prob.Z0, dtype=np.float64)
    Y = np.asfortranarray(prob.Y, dtype=np.float64)
    om = np.asfortranarray(prob.omega, dtype=np.float64)
    args = [prob.G, prob.M0, prob.N0, _dp(Z0), _dp(Y), _dp(om), roff.ctypes.data_as(_PI), ridx.ctypes.data_as(_PI),
            _dp(_f(prob.z_scale)), _dp(_f(prob.c_scale)), _dp(_f(w1)), _dp(_f(z1)), C.byref(cfg),
            _dp(_f(beta_true)), _dp(b), _dp(w), rows if trace else None, cap, C.byref(res)]
    counters = None
    if kind == "oracle":
        bad = C.c_int(-1)
        st = L.orc_pcg_aug_mvrglm(*args, C.byref(bad))
        if st:
            raise OracleError(st, f"block {bad.value}")
    else:
        counters = np.zeros(6, dtype=np.uint64)
        st = L.ref_pcg_aug_mvrglm(*args, counters.ctypes.data_as(C.POINTER(C.c_uint64)))
        if st:
            raise OracleError(st, L.ref_last_error().decode())
    tr = np.frombuffer(rows, dtype=TRACE_DTYPE, count=min(res.n_rows, cap)).copy() if trace else np.zeros(0, TRACE_DTYPE)
    return SolveOut(b=b, w=w, iterations=int(res.iterations), termination=TERMINATION[res.termination],
                    breakdown_iteration=None if res.breakdown_iteration < 0 else int(res.breakdown_iteration),
                    residual_seminorm=float(res.residual_seminorm), w1_projected=bool(res.w1_projected),
                    trace=tr, sigma_scale=float(res.sigma_scale), counters=counters)


MV_OPS = {"pi": 0, "xstar_t": 1, "xstar": 2, "sigma": 3, "x": 4, "xt": 5}


def mv_apply(prob, kind_op: str, vec: np.ndarray, kind: str = "oracle") -> np.ndarray:
    """mvrglm_preconditioner applies (and, oracle only, the embedded Sigma / X / X' applies)."""
    L = lib(kind)
    op = MV_OPS[kind_op]
    roff, ridx = prob.csr()
    out = np.zeros(prob.n if op in (1, 5) else prob.m)
    v = np.ascontiguousarray(vec, dtype=np.float64)
    Z0 = np.asfortranarray(prob.Z0, dtype=np.float64)
    if kind == "oracle":
        om = np.asfortranarray(prob.omega, dtype=np.float64)
        st = L.orc_mvrglm_apply(prob.G, prob.M0, prob.N0, _dp(Z0), _dp(om), roff.ctypes.data_as(_PI),
                                ridx.ctypes.data_as(_PI), _dp(_f(prob.z_scale)), _dp(_f(prob.c_scale)), op, _dp(v),
                                _dp(out))
    else:
        assert op <= 2
        st = L.ref_mvrglm_apply(prob.G, prob.M0, prob.N0, _dp(Z0), roff.ctypes.data_as(_PI),
                                ridx.ctypes.data_as(_PI), _dp(_f(prob.z_scale)), _dp(_f(prob.c_scale)), op, _dp(v),
                                _dp(out))
    if st:
        raise OracleError(st)
    return out


def mv_norm_probe(prob) -> float:
    roff, ridx = prob.csr()
    return lib("oracle").orc_mvrglm_norm_probe(prob.G, prob.M0, prob.N0, _dp(np.asfortranarray(prob.Z0)),
                                               _dp(np.asfortranarray(prob.omega)), roff.ctypes.data_as(_PI),
                                               ridx.ctypes.data_as(_PI))


def mv_reduce(prob, kind: str = "oracle"):
    """mv_reduce: (R0 (N0 x N0), Q0'Y (N0 x G)) of the thin QR Z0 = Q0 R0."""
    L = lib(kind)
    R = np.zeros((prob.N0, prob.N0), order="F")
    QtY = np.zeros((prob.N0, prob.G), order="F")
    fn = L.orc_mv_reduce if kind == "oracle" else L.ref_mv_reduce
    st = fn(prob.G, prob.M0, prob.N0, _dp(np.asfortranarray(prob.Z0)), _dp(np.asfortranarray(prob.Y)), _dp(R),
            _dp(QtY))
    if st:
        raise OracleError(st)
    return R, QtY


def sur_reduce_ref(prob, rank_tol: float = 1e-10, want_basis: bool = False):
    """The reference's own sur_reduce (structured.cpp:132-178) through oracle/_ref: (q, X_red (q x n),
    Y_red (q x G), basis (M x q) or None).  q == M means "not reduced" (X_red / Y_red are the inputs)."""
    L = lib("ref")
    nb = np.ascontiguousarray(prob.nb, dtype=np.int64)
    n = int(nb.sum())
    Xr = np.zeros(prob.M * n)
    Yr = np.zeros(prob.M * prob.G)
    B = np.zeros(prob.M * min(prob.M, n)) if want_basis else None
    q = C.c_int64(0)
    st = L.ref_sur_reduce(prob.G, prob.M, nb.ctypes.data_as(_PI), _dp(np.asfortranarray(prob.X)),
                          _dp(np.asfortranarray(prob.Y)), rank_tol, C.byref(q), _dp(Xr), _dp(Yr), _dp(B))
    if st:
        raise OracleError(st, L.ref_last_error().decode())
    q = int(q.value)
    if q >= prob.M:
        return q, np.asfortranarray(prob.X), np.asfortranarray(prob.Y), None
    return (q, Xr[:q * n].reshape(q, n, order="F"), Yr[:q * prob.G].reshape(q, prob.G, order="F"),
            B[:prob.M * q].reshape(prob.M, q, order="F") if want_basis else None)


def solve_ne(prob, kind: str = "oracle", cfg: Optional[Config] = None, trace: bool = True,
             beta_true: Optional[np.ndarray] = None) -> SolveOut:
    """pcg_normal_equations(embed_sur(sur), nullptr, cfg, true_beta) (pcg.cpp:364-511): the PCG-NE comparison
    solver.  kind="oracle": the SUR-structured restatement; kind="ref": the literal reference (dense m x m
    Cholesky of Sigma; small sizes only).  sigma_scale holds the oracle's g_scale (0 for the reference)."""
    L = lib(kind)
    if cfg is None:
        cfg = make_config(tol_rel=prob.tol_rel, max_iter=prob.max_iter)
    nb = np.ascontiguousarray(prob.nb, dtype=np.int64)
    m, n = prob.M * prob.G, int(nb.sum())
    max_iter = cfg.max_iter if cfg.max_iter else 2 * n
    cap = max_iter + 1 if trace else 0
    rows = (TraceRow * max(cap, 1))()
    b, w, res = np.zeros(n), np.zeros(m), Result()
    bt = None if beta_true is None else np.ascontiguousarray(beta_true, dtype=np.float64)
    args = [prob.G, prob.M, nb.ctypes.data_as(_PI), _dp(prob.X), _dp(prob.Y), _dp(prob.omega), C.byref(cfg), _dp(bt),
            _dp(b), _dp(w), rows if trace else None, cap, C.byref(res)]
    st = (L.orc_pcg_ne_sur if kind == "oracle" else L.ref_pcg_ne_sur)(*args)
    if st:
        raise OracleError(st, L.ref_last_error().decode() if kind != "oracle" else "")
    tr = np.frombuffer(rows, dtype=TRACE_DTYPE, count=min(res.n_rows, cap)).copy() if trace else np.zeros(0, TRACE_DTYPE)
    return SolveOut(b=b, w=w, iterations=int(res.iterations), termination=TERMINATION[res.termination],
                    breakdown_iteration=None if res.breakdown_iteration < 0 else int(res.breakdown_iteration),
                    residual_seminorm=float(res.residual_seminorm), w1_projected=False, trace=tr,
                    sigma_scale=float(res.sigma_scale))
