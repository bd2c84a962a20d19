"""Python mirror of the reference's SUR solver API, backed by the B200 library through its C-ABI.

Names, argument meaning and error behaviour follow the reference (/root/reference/proj/include/gls):

  make_sur(blocks, y, sigma0) -> SurModel                     structured.hpp:53-63, structured.cpp:97-105
  sur_preconditioner(sur[, block_scale]) -> preconditioner    structured.hpp:105-108, structured.cpp:416-486
      .rows() .params() .apply_pi .apply_xstar_t .apply_xstar .counters() .reset_apply_counters()
                                                              preconditioner.hpp:30-53, preconditioner.cpp:9-47
  cost_counters(op) -> CostReport                             preconditioner.hpp:56-64, preconditioner.cpp:37-47
  pcg_aug(sur, op, w1, z1, config, true_beta) -> AugSolveResult    pcg.hpp:80-83 (Glm = embed_sur(sur))
  operator_norm_probe(op_or_sur, iters=12)                    pcg.hpp:132
  PcgConfig / PcgTraceRow / PcgTrace / GlsSolution / Termination   pcg.hpp:12-51, glm.hpp:26-37
  GlsError and subclasses                                     errors.hpp:10-88

The difference from the reference is the one the SURVEY calls the dense-embedding wall: the reference
takes `Glm glm = embed_sur(sur)` (a dense (G M) x n X); here the solver takes the SurModel itself and
never forms it (SURVEY.md s7 "hard parts").
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L

_P = C.POINTER(C.c_double)
_PI64 = C.POINTER(C.c_int64)


# ------------------------------------------------------------------------------------------ errors
class GlsError(RuntimeError):
    """gls::Error (errors.hpp:10-14)."""


class DimensionMismatch(GlsError):
    pass


class RankDeficient(GlsError):
    pass


class SingularD(GlsError):
    pass


class SingularTriangular(GlsError):
    pass


class DeviceError(GlsError):
    """CUDA failure / no device / unsupported shape (not in the reference: the device side)."""


class SingularCovariance(GlsError):
    pass


_ERRORS = {1: DimensionMismatch, 2: RankDeficient, 3: SingularD, 4: SingularTriangular, 5: SingularCovariance}


def _check(code: int, lib=None):
    if code == 0:
        return
    lib = lib or L.load()
    msg = lib.glsgpu_last_error_message().decode()
    raise _ERRORS.get(code, DeviceError)(f"[{code}] {msg}")


def _dp(a):
    if a is None:
        return None
    return a.ctypes.data_as(_P)


# ------------------------------------------------------------------------------------------ types
class Termination(enum.IntEnum):
    """gls::Termination (glm.hpp:26)."""
    Converged = 0
    Breakdown = 1
    Stagnation = 2
    MaxIter = 3
    Direct = 4


@dataclasses.dataclass
class PcgConfig:
    """gls::PcgConfig (pcg.hpp:12-30) plus the device knobs of glsgpu_pcg_config."""
    tol_rel: float = 1e-10
    max_iter: int = 0
    breakdown_tol: float = 1e-14
    stagnation_window: int = 5
    growth_tol: float = 1e4
    growth_window: int = 10
    record_z_every: int = 1
    diag_every: int = 1        # trace diagnostics every k rows (1 = as the reference; 0 = row 0 + final; -1 = none)
    xv_mode: str = "x"         # "x": X v with the original X (reference); "qr": Q (R v) by recurrence
    graph_chunk: int = 0
    kernel_timing: bool = False
    kron_fma: bool = False     # FP64-bound Kronecker pass (128 < G <= 256) with fused multiply-adds
    sw_mode: int = 0           # 1: Sigma w formed where read instead of by recurrence (kron_fma, diag_every <= 0)
    fused_c: int = 0           # 1: Sigma pr inside pass C, Sigma u by recurrence, element-wise pass A (needs sw_mode 1)

    def to_c(self) -> L.PcgConfigC:
        return L.PcgConfigC(self.tol_rel, self.max_iter, self.breakdown_tol, self.stagnation_window, self.growth_tol,
                            self.growth_window, self.record_z_every, self.diag_every,
                            1 if self.xv_mode == "qr" else 0, self.graph_chunk, 1 if self.kernel_timing else 0,
                            1 if self.kron_fma else 0, int(self.sw_mode), int(self.fused_c))


TRACE_DTYPE = np.dtype([("iter", np.int64), ("c", np.float64), ("aug_residual_norm", np.float64),
                        ("dual_feas_norm", np.float64), ("rmse", np.float64), ("elapsed_ns", np.int64)])


@dataclasses.dataclass
class PcgTrace:
    rows: np.ndarray                      # TRACE_DTYPE records, len == iterations + 1
    termination: Termination
    breakdown_iteration: Optional[int]
    w1_projected: bool


@dataclasses.dataclass
class GlsSolution:
    b: np.ndarray
    w: Optional[np.ndarray]
    iterations: int
    termination: Termination
    residual_seminorm: float


@dataclasses.dataclass
class AugSolveResult:
    solution: GlsSolution
    trace: PcgTrace
    sigma_scale: float = float("nan")
    solve_ms: float = float("nan")


@dataclasses.dataclass
class CostCounters:
    factorizations: int
    factor_multiplies: int
    pi_applies: int
    xstar_t_applies: int
    xstar_applies: int
    apply_multiplies: int


@dataclasses.dataclass
class CostReport:
    factorizations: int
    factor_multiplies: int
    total_applies: int
    apply_multiplies: int
    multiplies_per_apply: float


@dataclasses.dataclass
class SurModel:
    """gls::SurModel (structured.hpp:53-61): X_i blocks (M x n_i), Y (M x G), sigma0 (G x G).

    Stored as the concatenation X = [X_0 | ... | X_{G-1}] (M x n, column-major) plus widths.
    """
    X: np.ndarray
    nb: np.ndarray
    y: np.ndarray
    sigma0: np.ndarray

    def obs(self) -> int:
        return int(self.y.shape[0])

    def equations(self) -> int:
        return int(len(self.nb))

    def total_params(self) -> int:
        return int(self.nb.sum())


def make_sur(blocks: Sequence[np.ndarray], y: np.ndarray, sigma0: np.ndarray) -> SurModel:
    """make_sur (structured.cpp:97-105): same checks, same messages."""
    if len(blocks) == 0:
        raise DimensionMismatch("make_sur: need at least one block")
    y = np.asfortranarray(y, dtype=np.float64)
    if y.ndim != 2 or y.shape[1] != len(blocks):
        raise DimensionMismatch("make_sur: Y/blocks mismatch")
    for b in blocks:
        if b.shape[0] != y.shape[0]:
            raise DimensionMismatch("make_sur: block row mismatch")
    sigma0 = np.asfortranarray(sigma0, dtype=np.float64)
    if sigma0.shape != (len(blocks), len(blocks)):
        raise DimensionMismatch("make_sur: Sigma0 must be G x G")
    nb = np.array([b.shape[1] for b in blocks], dtype=np.int64)
    X = np.asfortranarray(np.concatenate([np.asarray(b, dtype=np.float64) for b in blocks], axis=1)) \
        if int(nb.sum()) > 0 else np.zeros((y.shape[0], 0), order="F")
    return SurModel(X=X, nb=nb, y=y, sigma0=sigma0)


def sur_from_problem(prob) -> SurModel:
    """SurModel of a synth.SurProblem (already concatenated)."""
    return SurModel(X=np.asfortranarray(prob.X), nb=np.asarray(prob.nb, dtype=np.int64),
                    y=np.asfortranarray(prob.Y), sigma0=np.asfortranarray(prob.omega))


# ------------------------------------------------------------------------------------------ operator
class GpuSurPreconditioner:
    """The SUR indefinite preconditioner (SurPreconditioner, structured.cpp:416-453) resident on a B200.

    Construction factors every block on the device: CholeskyQR2 on the FP64 tensor cores, the Householder TSQR tree
    per block as its fallback (factor_info()).
    """

    def __init__(self, sur: SurModel, block_scale: Optional[np.ndarray] = None, device: int = 0):
        self._lib = L.load()
        self.sur = sur
        self._h = C.c_void_p()
        nb = np.ascontiguousarray(sur.nb, dtype=np.int64)
        self._nb = nb
        bad = C.c_int(-1)
        scale = None if block_scale is None else np.ascontiguousarray(block_scale, dtype=np.float64)
        if scale is not None and scale.shape != (len(nb),):
            raise DimensionMismatch("sur_preconditioner: need one scale per block")
        X = np.asfortranarray(sur.X, dtype=np.float64)
        Y = np.asfortranarray(sur.y, dtype=np.float64)
        om = np.asfortranarray(sur.sigma0, dtype=np.float64)
        code = self._lib.glsgpu_sur_create(len(nb), sur.obs(), nb.ctypes.data_as(_PI64), _dp(X), _dp(Y), _dp(om),
                                           _dp(scale), device, C.byref(self._h), C.byref(bad))
        self.bad_block = bad.value
        _check(code, self._lib)
        self.m = sur.obs() * len(nb)
        self.n = int(nb.sum())

    @classmethod
    def from_device(cls, G: int, M: int, nb, X_ptr: int, ldx: int, Y_ptr: int, ldy: int, omega: np.ndarray,
                    block_scale=None, device: int = 0) -> "GpuSurPreconditioner":
        """Operator over device-resident X / Y (bench path: no host copy of the big inputs)."""
        self = cls.__new__(cls)
        self._lib = L.load()
        self.sur = None
        self._h = C.c_void_p()
        self._nb = np.ascontiguousarray(nb, dtype=np.int64)
        bad = C.c_int(-1)
        om = np.asfortranarray(omega, dtype=np.float64)
        scale = None if block_scale is None else np.ascontiguousarray(block_scale, dtype=np.float64)
        code = self._lib.glsgpu_sur_create_device(G, M, self._nb.ctypes.data_as(_PI64), C.c_void_p(X_ptr), ldx,
                                                  C.c_void_p(Y_ptr), ldy, _dp(om), _dp(scale), device,
                                                  C.byref(self._h), C.byref(bad))
        self.bad_block = bad.value
        _check(code, self._lib)
        self.m = M * G
        self.n = int(self._nb.sum())
        return self

    @classmethod
    def from_device_sharded(cls, G: int, M_local: int, M_global: int, nb, X_ptr: int, ldx: int, Y_ptr: int, ldy: int,
                            omega: np.ndarray, nccl_id: bytes, rank: int, nranks: int, block_scale=None,
                            device: int = 0) -> "GpuSurPreconditioner":
        """Row-sharded operator: this rank owns M_local of the M_global rows of every block."""
        self = cls.__new__(cls)
        self._lib = L.load()
        self.sur = None
        self._h = C.c_void_p()
        self._nb = np.ascontiguousarray(nb, dtype=np.int64)
        bad = C.c_int(-1)
        om = np.asfortranarray(omega, dtype=np.float64)
        scale = None if block_scale is None else np.ascontiguousarray(block_scale, dtype=np.float64)
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        code = self._lib.glsgpu_sur_create_sharded(G, M_local, M_global, self._nb.ctypes.data_as(_PI64),
                                                   C.c_void_p(X_ptr), ldx, C.c_void_p(Y_ptr), ldy, _dp(om), _dp(scale),
                                                   device, idbuf, rank, nranks, C.byref(self._h), C.byref(bad))
        self.bad_block = bad.value
        _check(code, self._lib)
        self.m = M_local * G      # host vectors of a sharded handle are the rank's local rows
        self.n = int(self._nb.sum())
        return self

    @classmethod
    def from_host_sharded(cls, G: int, M_local: int, M_global: int, nb, X: np.ndarray, Y: np.ndarray, omega: np.ndarray,
                          nccl_id: bytes, rank: int, nranks: int, block_scale=None,
                          device: int = 0) -> "GpuSurPreconditioner":
        """Row-sharded operator from this rank's HOST rows (X: M_local x n, Y: M_local x G); the handle owns its
        device copies, so update / stage / update_staged serve it."""
        self = cls.__new__(cls)
        self._lib = L.load()
        self.sur = None
        self._h = C.c_void_p()
        self._nb = np.ascontiguousarray(nb, dtype=np.int64)
        bad = C.c_int(-1)
        om = np.asfortranarray(omega, dtype=np.float64)
        scale = None if block_scale is None else np.ascontiguousarray(block_scale, dtype=np.float64)
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        code = self._lib.glsgpu_sur_create_sharded_host(G, M_local, M_global, self._nb.ctypes.data_as(_PI64),
                                                        C.c_void_p(_host_ptr(X, (M_local, int(self._nb.sum())))),
                                                        C.c_void_p(_host_ptr(Y, (M_local, G))), _dp(om), _dp(scale),
                                                        device, idbuf, rank, nranks, C.byref(self._h), C.byref(bad))
        self.bad_block = bad.value
        _check(code, self._lib)
        self.m = M_local * G
        self.n = int(self._nb.sum())
        return self

    @classmethod
    def from_device_local_group(cls, group: "LocalGroup", rank: int, G: int, M_local: int, M_global: int, nb,
                                X_ptr: int, ldx: int, Y_ptr: int, ldy: int, omega: np.ndarray,
                                block_scale=None) -> "GpuSurPreconditioner":
        """TEST-ONLY: rank `rank` of an in-process rank group on one device (glsgpu_sur_create_sharded_local).
        Every rank must be created, and solved, from its own thread, concurrently."""
        self = cls.__new__(cls)
        self._lib = L.load()
        self.sur = None
        self._h = C.c_void_p()
        self._nb = np.ascontiguousarray(nb, dtype=np.int64)
        bad = C.c_int(-1)
        om = np.asfortranarray(omega, dtype=np.float64)
        scale = None if block_scale is None else np.ascontiguousarray(block_scale, dtype=np.float64)
        code = self._lib.glsgpu_sur_create_sharded_local(G, M_local, M_global, self._nb.ctypes.data_as(_PI64),
                                                         C.c_void_p(X_ptr), ldx, C.c_void_p(Y_ptr), ldy, _dp(om),
                                                         _dp(scale), group.handle, rank, C.byref(self._h), C.byref(bad))
        self.bad_block = bad.value
        _check(code, self._lib)
        self.m = M_local * G
        self.n = int(self._nb.sum())
        return self

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.glsgpu_sur_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def stream_ptr(self) -> int:
        return int(self._lib.glsgpu_sur_stream(self._h) or 0)

    def rows(self) -> int:
        return self.m

    def params(self) -> int:
        return self.n

    def _apply(self, fn, vec, nin, nout):
        v = np.ascontiguousarray(vec, dtype=np.float64).reshape(-1)
        if v.size != nin:
            name = {"glsgpu_apply_pi": "apply_pi", "glsgpu_apply_xstar_t": "apply_xstar_t",
                    "glsgpu_apply_xstar": "apply_xstar"}.get(fn, fn)
            raise DimensionMismatch(f"{name}: size mismatch")
        out = np.empty(nout)
        _check(getattr(self._lib, fn)(self._h, _dp(v), _dp(out)), self._lib)
        return out

    def apply_pi(self, xi):
        return self._apply("glsgpu_apply_pi", xi, self.m, self.m)

    def apply_xstar_t(self, xi):
        return self._apply("glsgpu_apply_xstar_t", xi, self.m, self.n)

    def apply_xstar(self, v):
        return self._apply("glsgpu_apply_xstar", v, self.n, self.m)

    def sigma_apply(self, x):
        return self._apply("glsgpu_sigma_apply", x, self.m, self.m)

    def counters(self) -> CostCounters:
        c = L.CountersC()
        _check(self._lib.glsgpu_counters(self._h, C.byref(c)), self._lib)
        return CostCounters(c.factorizations, c.factor_multiplies, c.pi_applies, c.xstar_t_applies, c.xstar_applies,
                            c.apply_multiplies)

    def reset_apply_counters(self):
        _check(self._lib.glsgpu_reset_apply_counters(self._h), self._lib)

    def factors(self):
        Q = np.zeros((self.m // len(self._nb), self.n), order="F")
        R = np.zeros(int((self._nb * self._nb).sum()))
        _check(self._lib.glsgpu_get_factors(self._h, _dp(Q), _dp(R)), self._lib)
        return Q, R

    def factor_info(self):
        """(method, fallbacks): method "cholqr2" (csrc/cqr.cuh) or "tsqr" for the current factors; fallbacks = how
        many factorisations of this operator failed CholeskyQR2's own test and were redone by the Householder TSQR."""
        m, f = C.c_int(0), C.c_int(0)
        _check(self._lib.glsgpu_factor_info(self._h, C.byref(m), C.byref(f)), self._lib)
        return ("cholqr2" if m.value == 1 else "tsqr"), f.value

    def update(self, X: np.ndarray, y: np.ndarray):
        """New data of the same shapes (glsgpu_sur_update): upload X (M x n) and Y (M x G), refactor; the device
        memory and the factorisation plan of this operator are reused."""
        Xf = np.asfortranarray(X, dtype=np.float64)
        Yf = np.asfortranarray(y, dtype=np.float64)
        if Xf.shape != (self.m // len(self._nb), self.n) or Yf.shape != (self.m // len(self._nb), len(self._nb)):
            raise DimensionMismatch("update: shapes differ from the operator's")
        bad = C.c_int(-1)
        _check(self._lib.glsgpu_sur_update(self._h, _dp(Xf), _dp(Yf), C.byref(bad)), self._lib)

    def stage(self, X, Y):
        """Queue the NEXT model's X (M x n) and Y (M x G) for upload (glsgpu_sur_stage): the copy overlaps the
        current solve (xv_mode QR).  X / Y are numpy or CPU-torch arrays in that (column-major) layout -- pinned
        memory for a truly asynchronous copy -- and must stay alive and unchanged until update_staged()."""
        Mloc = self.m // len(self._nb)
        xp = _host_ptr(X, (Mloc, self.n))
        yp = _host_ptr(Y, (Mloc, len(self._nb)))
        self._staged_refs = (X, Y)
        _check(self._lib.glsgpu_sur_stage(self._h, C.c_void_p(xp), C.c_void_p(yp)), self._lib)

    def update_staged(self):
        """Make the staged model current: wait for its upload, refactor (glsgpu_sur_update_staged)."""
        bad = C.c_int(-1)
        _check(self._lib.glsgpu_sur_update_staged(self._h, C.byref(bad)), self._lib)
        self._staged_refs = None

    def refactor(self):
        bad = C.c_int(-1)
        _check(self._lib.glsgpu_sur_refactor(self._h, C.byref(bad)), self._lib)

    def launch_count(self) -> int:
        v = C.c_int64(0)
        _check(self._lib.glsgpu_launch_count(self._h, C.byref(v)), self._lib)
        return int(v.value)

    def kernel_stats(self) -> List[dict]:
        arr = (L.KernelStatC * 16)()
        k = self._lib.glsgpu_kernel_stats(self._h, arr, 16)
        return [dict(name=arr[i].name.decode(), launches=int(arr[i].launches), total_ms=float(arr[i].total_ms),
                     bytes_per_launch=float(arr[i].bytes_per_launch)) for i in range(k)]


def sur_preconditioner(sur: SurModel, block_scale: Optional[np.ndarray] = None, device: int = 0) -> GpuSurPreconditioner:
    """sur_preconditioner (structured.cpp:479-486)."""
    return GpuSurPreconditioner(sur, block_scale, device)


def cost_counters(op: GpuSurPreconditioner) -> CostReport:
    """cost_counters (preconditioner.cpp:37-47)."""
    c = op.counters()
    total = c.pi_applies + c.xstar_t_applies + c.xstar_applies
    return CostReport(c.factorizations, c.factor_multiplies, total, c.apply_multiplies,
                      (c.apply_multiplies / total) if total else 0.0)


def operator_norm_probe(op: GpuSurPreconditioner, iters: int = 12) -> float:
    out = C.c_double()
    _check(op._lib.glsgpu_operator_norm_probe(op.handle, iters, C.byref(out)), op._lib)
    return out.value


def pcg_aug(sur_or_op, precond: Optional[GpuSurPreconditioner] = None, w1=None, z1=None,
            config: Optional[PcgConfig] = None, true_beta=None, want_w: bool = True,
            want_trace: bool = True) -> AugSolveResult:
    """pcg_aug (pcg.cpp:346-350 -> run_aug, Recovery variant) on the SUR model, on the device.

    `sur_or_op` is the SurModel (the reference passes embed_sur(sur)) or the MvRglm (embed_mvrglm(mv));
    `precond` its sur_preconditioner / mvrglm_preconditioner (built here when None).
    """
    if precond is not None:
        op = precond
    elif isinstance(sur_or_op, GpuSurPreconditioner):
        op = sur_or_op
    elif isinstance(sur_or_op, MvRglm):
        op = mvrglm_preconditioner(sur_or_op)  # pcg_aug(embed_mvrglm(mv), *mvrglm_preconditioner(mv))
    else:
        op = sur_preconditioner(sur_or_op)
    cfg = config or PcgConfig()
    m, n = op.m, op.n
    if w1 is not None and np.asarray(w1).size != m or z1 is not None and np.asarray(z1).size != n:
        raise DimensionMismatch("pcg_aug: bad initial iterate size")
    w1a = None if w1 is None else np.ascontiguousarray(w1, dtype=np.float64)
    z1a = None if z1 is None else np.ascontiguousarray(z1, dtype=np.float64)
    bt = None if true_beta is None else np.ascontiguousarray(true_beta, dtype=np.float64)
    max_iter = cfg.max_iter if cfg.max_iter else m - n + 1
    cap = (max_iter + 1) if want_trace else 0
    rows = (L.TraceRowC * max(cap, 1))()
    b = np.empty(n)
    w = np.empty(m) if want_w else None
    res = L.ResultC()
    cc = cfg.to_c()
    code = op._lib.glsgpu_sur_solve(op.handle, C.byref(cc), _dp(w1a), _dp(z1a), _dp(bt), _dp(b), _dp(w),
                                    rows if want_trace else None, cap, C.byref(res))
    _check(code, op._lib)
    k = min(res.n_rows, cap)
    tr = np.frombuffer(rows, dtype=TRACE_DTYPE, count=k).copy() if want_trace else np.zeros(0, TRACE_DTYPE)
    term = Termination(res.termination)
    sol = GlsSolution(b=b, w=w, iterations=int(res.iterations), termination=term,
                      residual_seminorm=float(res.residual_seminorm))
    trace = PcgTrace(rows=tr, termination=term,
                     breakdown_iteration=None if res.breakdown_iteration < 0 else int(res.breakdown_iteration),
                     w1_projected=bool(res.w1_projected))
    return AugSolveResult(solution=sol, trace=trace, sigma_scale=float(res.sigma_scale), solve_ms=float(res.solve_ms))


# ------------------------------------------------------------------------------------------ MVRGLM
@dataclasses.dataclass
class MvRglm:
    """gls::MvRglm (structured.hpp:33-43): Y = Z0 B + U, restrictions[i] = zero-forced rows of B[:, i]."""
    z0: np.ndarray
    y: np.ndarray
    omega0: np.ndarray
    restrictions: List[np.ndarray]

    def obs(self) -> int:
        return int(self.z0.shape[0])

    def params_per_eq(self) -> int:
        return int(self.z0.shape[1])

    def equations(self) -> int:
        return int(self.y.shape[1])

    def total_restrictions(self) -> int:
        return int(sum(len(r) for r in self.restrictions))

    def csr(self):
        roff = np.zeros(self.equations() + 1, dtype=np.int64)
        roff[1:] = np.cumsum([len(r) for r in self.restrictions])
        ridx = (np.concatenate([np.asarray(r, dtype=np.int64) for r in self.restrictions])
                if roff[-1] else np.zeros(1, dtype=np.int64))
        return roff, np.ascontiguousarray(ridx, dtype=np.int64)


@dataclasses.dataclass
class ReductionRecord:
    """gls::ReductionRecord (structured.hpp:67-72)."""
    original_rows: int
    reduced_rows: int
    rank: int


def make_mvrglm(z0: np.ndarray, y: np.ndarray, omega0: np.ndarray, restrictions) -> MvRglm:
    """make_mvrglm (structured.cpp:63-74): same checks, same messages."""
    z0 = np.asfortranarray(z0, dtype=np.float64)
    y = np.asfortranarray(y, dtype=np.float64)
    omega0 = np.asfortranarray(omega0, dtype=np.float64)
    if z0.shape[0] < z0.shape[1]:
        raise DimensionMismatch("make_mvrglm: Z0 must be tall")
    if y.shape[0] != z0.shape[0]:
        raise DimensionMismatch("make_mvrglm: Y/Z0 row mismatch")
    if omega0.shape != (y.shape[1], y.shape[1]):
        raise DimensionMismatch("make_mvrglm: Omega0 must be G x G")
    if len(restrictions) != y.shape[1]:
        raise DimensionMismatch("restrictions: need one list per equation")
    out = []
    for lst in restrictions:
        a = np.asarray(lst, dtype=np.int64).reshape(-1)
        if a.size and (a.min() < 0 or a.max() >= z0.shape[1]):
            raise DimensionMismatch("restrictions: index out of range")
        if a.size > 1 and np.any(np.diff(a) <= 0):
            raise DimensionMismatch("restrictions: indices must be strictly increasing")
        out.append(a)
    return MvRglm(z0=z0, y=y, omega0=omega0, restrictions=out)


def mv_from_problem(prob) -> MvRglm:
    return make_mvrglm(prob.Z0, prob.Y, prob.omega, prob.restrictions)


class GpuMvRglmPreconditioner(GpuSurPreconditioner):
    """MvRglmPreconditioner (structured.cpp:365-414) on the B200, with the embed_mvrglm operator
    (structured.cpp:77-95) behind the same handle: per-equation QR of the stacked [Z0 w_z; C_i w_c].
    Host m-vectors use the reference's embedded order (G M0 observation rows, then the k constraint rows)."""

    def __init__(self, mv: MvRglm, z_scale=None, c_scale=None, device: int = 0):
        self._lib = L.load()
        self.sur = None
        self.mv = mv
        self._h = C.c_void_p()
        G = mv.equations()
        self._nb = np.full(G, mv.params_per_eq(), dtype=np.int64)
        zs = None if z_scale is None else np.ascontiguousarray(z_scale, dtype=np.float64)
        cs = None if c_scale is None else np.ascontiguousarray(c_scale, dtype=np.float64)
        for v in (zs, cs):
            if v is not None and v.shape != (G,):
                raise DimensionMismatch("mvrglm_preconditioner: need one scale per equation")
        roff, ridx = mv.csr()
        bad = C.c_int(-1)
        code = self._lib.glsgpu_mvrglm_create(G, mv.obs(), mv.params_per_eq(), _dp(mv.z0), _dp(mv.y), _dp(mv.omega0),
                                              roff.ctypes.data_as(_PI64), ridx.ctypes.data_as(_PI64), _dp(zs), _dp(cs),
                                              device, C.byref(self._h), C.byref(bad))
        self.bad_block = bad.value
        _check(code, self._lib)
        m, n = C.c_int64(0), C.c_int64(0)
        _check(self._lib.glsgpu_model_dims(self._h, C.byref(m), C.byref(n)), self._lib)
        self.m, self.n = int(m.value), int(n.value)

    def factors(self):
        raise NotImplementedError("factors(): SUR handles only")


def mvrglm_preconditioner(mv: MvRglm, z_scale=None, c_scale=None, device: int = 0) -> GpuMvRglmPreconditioner:
    """mvrglm_preconditioner (structured.cpp:468-477); identity auxiliary when no scales are given."""
    return GpuMvRglmPreconditioner(mv, z_scale, c_scale, device)


def mv_reduce(mv: MvRglm, device: int = 0):
    """mv_reduce (structured.cpp:121-130) on the device: (reduced MvRglm with Z0 -> R0, Y -> Q0'Y, record).

    R0 is the reference's up to row signs (TSQR instead of one Householder sweep); the GLS estimate of the
    reduced model does not depend on them."""
    lib = L.load()
    G, M0, N0 = mv.equations(), mv.obs(), mv.params_per_eq()
    R = np.zeros((N0, N0), order="F")
    QtY = np.zeros((N0, G), order="F")
    _check(lib.glsgpu_mv_reduce(G, M0, N0, _dp(mv.z0), _dp(mv.y), _dp(R), _dp(QtY), device), lib)
    red = MvRglm(z0=R, y=QtY, omega0=mv.omega0, restrictions=list(mv.restrictions))
    return red, ReductionRecord(original_rows=M0, reduced_rows=N0, rank=N0)


def sur_reduce(sur: SurModel, rank_tol: float = 1e-10, device: int = 0, want_transform: bool = False):
    """sur_reduce (structured.cpp:132-178, the paper's Remark 1) on the device: every equation rotated onto
    an orthonormal basis of range([X_1 ... X_G]), q = its numerical rank.  Returns (reduced SurModel,
    ReductionRecord[, transform M x q]).  The basis equals the reference's up to an orthogonal q x q factor."""
    lib = L.load()
    G, M, n = sur.equations(), sur.obs(), sur.total_params()
    nb = np.ascontiguousarray(sur.nb, dtype=np.int64)
    cap = min(M, n)
    Xr = np.zeros(cap * n if cap < M else M * n)
    Yr = np.zeros(cap * G if cap < M else M * G)
    B = np.zeros(M * cap) if want_transform else None
    q = C.c_int64(0)
    _check(lib.glsgpu_sur_reduce(G, M, nb.ctypes.data_as(_PI64), _dp(np.asfortranarray(sur.X)),
                                 _dp(np.asfortranarray(sur.y)), rank_tol, device, C.byref(q), _dp(Xr), _dp(Yr),
                                 _dp(B) if B is not None and cap < M else None), lib)
    q = int(q.value)
    rec = ReductionRecord(original_rows=M, reduced_rows=q, rank=q if q < M else M)
    if q >= M:
        out = (sur, rec)
        return out + (np.eye(M),) if want_transform else out
    red = SurModel(X=np.asfortranarray(Xr[:q * n].reshape(q, n, order="F")), nb=nb.copy(),
                   y=np.asfortranarray(Yr[:q * G].reshape(q, G, order="F")), sigma0=sur.sigma0)
    if want_transform:
        return red, rec, B[:M * q].reshape(M, q, order="F")
    return red, rec


def _frobenius(a: np.ndarray) -> float:
    """DenseMatrix::frobenius_norm (dense_matrix.cpp:93-97): sequential sum of squares in storage order."""
    v = np.asarray(a, dtype=np.float64).reshape(-1, order="F")
    return float(np.sqrt(np.cumsum(v * v)[-1])) if v.size else 0.0


def auxiliary_scales(omega0: np.ndarray, rule: str, z0: Optional[np.ndarray] = None):
    """The harness's scaled-D choices (experiments.cpp:826-851): K1 = alpha I with alpha = max_i Omega_ii,
    K2 = diag(Omega).  Returns the SUR block scales, or with z0 (the reduced multivariate regressor) the
    (z_scale, c_scale) pair of mvrglm_preconditioner: the constraint rows' auxiliary variance is matched to
    the data scale |Z0|_F^2 / N0."""
    d = np.array([float(omega0[i, i]) for i in range(omega0.shape[0])])
    alpha = 0.0
    for v in d:  # std::max in the reference's loop order
        alpha = max(alpha, v)
    if rule == "k1":
        z = np.full(len(d), alpha)
    elif rule == "k2":
        z = d.copy()
    else:
        raise ValueError(rule)
    if z0 is None:
        return z
    f = _frobenius(z0)
    z_scale2 = f * f / float(z0.shape[1])
    return z, z / z_scale2


def pcg_normal_equations(sur_or_op, config: Optional[PcgConfig] = None, true_beta=None, want_w: bool = True,
                         want_trace: bool = True) -> AugSolveResult:
    """pcg_normal_equations(embed_sur(sur), nullptr, config, true_beta) (pcg.cpp:364-511) on the device: the
    PCG-NE comparison solver (identity preconditioner).  Raises SingularCovariance for a singular Omega."""
    op = sur_or_op if isinstance(sur_or_op, GpuSurPreconditioner) else sur_preconditioner(sur_or_op)
    cfg = config or PcgConfig()
    m, n = op.m, op.n
    max_iter = cfg.max_iter if cfg.max_iter else 2 * n
    cap = (max_iter + 1) if want_trace else 0
    rows = (L.TraceRowC * max(cap, 1))()
    b = np.empty(n)
    w = np.empty(m) if want_w else None
    bt = None if true_beta is None else np.ascontiguousarray(true_beta, dtype=np.float64)
    res = L.ResultC()
    cc = cfg.to_c()
    _check(op._lib.glsgpu_pcg_ne(op.handle, C.byref(cc), _dp(bt), _dp(b), _dp(w), rows if want_trace else None, cap,
                                 C.byref(res)), op._lib)
    k = min(res.n_rows, cap)
    tr = np.frombuffer(rows, dtype=TRACE_DTYPE, count=k).copy() if want_trace else np.zeros(0, TRACE_DTYPE)
    term = Termination(res.termination)
    sol = GlsSolution(b=b, w=w, iterations=int(res.iterations), termination=term,
                      residual_seminorm=float(res.residual_seminorm))
    trace = PcgTrace(rows=tr, termination=term,
                     breakdown_iteration=None if res.breakdown_iteration < 0 else int(res.breakdown_iteration),
                     w1_projected=False)
    return AugSolveResult(solution=sol, trace=trace, sigma_scale=float(res.sigma_scale), solve_ms=float(res.solve_ms))


def _host_ptr(a, shape) -> int:
    """Address of a column-major (shape) float64 host array: a Fortran-ordered numpy array, or a C-contiguous
    (cols, rows) numpy / CPU torch array (its transpose; pinned torch tensors give pinned pointers)."""
    rows, cols = shape
    if hasattr(a, "data_ptr"):  # torch tensor (cols, rows), row-major == rows x cols column-major
        if tuple(a.shape) != (cols, rows) or not a.is_contiguous() or a.is_cuda or str(a.dtype) != "torch.float64":
            raise DimensionMismatch(f"host tensor must be CPU float64 contiguous of shape {(cols, rows)}")
        return int(a.data_ptr())
    arr = np.asarray(a)
    if arr.dtype != np.float64:
        raise DimensionMismatch("host array must be float64")
    if arr.shape == (rows, cols) and arr.flags.f_contiguous:
        return int(arr.ctypes.data)
    if arr.shape == (cols, rows) and arr.flags.c_contiguous:
        return int(arr.ctypes.data)
    raise DimensionMismatch(f"host array must be ({rows}, {cols}) Fortran-ordered")


class LocalGroup:
    """TEST-ONLY in-process rank group on one device (glsgpu_local_group_create): the library's real sharded
    decomposition with device-to-device copies in place of NCCL, one host thread per rank."""

    def __init__(self, nranks: int, device: int = 0):
        self._lib = L.load()
        self.handle = C.c_void_p()
        _check(self._lib.glsgpu_local_group_create(nranks, device, C.byref(self.handle)), self._lib)
        self.nranks = nranks

    def close(self):
        if self.handle and self.handle.value:
            self._lib.glsgpu_local_group_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 creates it; the ranks share it over torch.distributed)."""
    lib = L.load()
    buf = C.create_string_buffer(128)
    _check(lib.glsgpu_nccl_unique_id(buf), lib)
    return buf.raw


def row_partition(M: int, nranks: int, rank: int, align: int = 32):
    """Contiguous row shard of rank r: [row0, row0 + rows), 32-row aligned boundaries (last takes the rest)."""
    base = (M // nranks) // align * align
    if base == 0:
        base = M // nranks
    row0 = rank * base
    rows = (M - row0) if rank == nranks - 1 else base
    return row0, rows


def device_count() -> int:
    lib = L.load()
    n = C.c_int(0)
    lib.glsgpu_device_count(C.byref(n))
    return n.value
