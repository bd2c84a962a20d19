"""Device-generated synthetic inputs of BASELINE.json's configs (the bench's inputs).

The full c4 model (G = 256, M = 1e6, n_i = 32: 65.5 GB of X) is drawn on the device by the library's
counter-based generator (``glsgpu_synth_normal``: Philox4x32-10 keyed by (seed, stream), one normal per
global matrix element), so any row shard of it is the same slice of the same global matrices
(``tests/test_gpu_parity.py::test_device_synth_is_shard_invariant``).  Omega, its PSD root and beta are
the host generator's (``synth.make_problem``): the same distributions as every other config.

Y = X beta + Z Omega^1/2 with Z from stream 3 (``glsgpu_synth_response``).
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from . import synth

__all__ = ["DeviceProblem", "device_problem"]


@dataclasses.dataclass
class DeviceProblem:
    name: str
    G: int
    M: int                   # global rows
    row0: int                # this rank's first row
    M_local: int             # this rank's rows
    nb: np.ndarray
    X: "object"              # torch (n, M_local) float64 on the device == M_local x n column-major
    Y: "object"              # torch (G, M_local) float64 on the device == M_local x G column-major
    omega: np.ndarray
    beta: np.ndarray
    tol_rel: float
    max_iter: int
    seed: int

    @property
    def n(self) -> int:
        return int(self.nb.sum())

    def to_host_problem(self) -> synth.SurProblem:
        """The same model on the host (D2H of X and Y; pageable numpy, Fortran views): the oracle's input."""
        X = self.X.cpu().numpy().T          # (M_local, n), Fortran order, no copy beyond the D2H
        Y = self.Y.cpu().numpy().T
        return synth.SurProblem(self.name, self.G, self.M_local, self.nb.copy(), X, Y, np.asfortranarray(self.omega),
                                self.beta.copy(), self.tol_rel, self.max_iter)


def device_problem(config: int = 4, M: int | None = None, G: int | None = None, world: int = 1, rank: int = 0,
                   device: int = 0) -> DeviceProblem:
    """Config `config` (SUR configs with constant or uniform widths) drawn on `device`; with world > 1 this
    rank's row shard (api.row_partition) of the same global model."""
    import torch

    from . import _lib as L
    from . import api

    meta = synth.config_meta(config)
    M = int(M or meta["M"])
    prob = synth.make_problem(config, M=M, G=G, with_data=False)
    if prob.name.startswith("c3"):
        raise ValueError("device_problem: config 3 (column-pattern model) is host-generated (synth.make_problem)")
    G = prob.G
    seed = 1000 + config
    nb = np.ascontiguousarray(prob.nb, dtype=np.int64)
    n = int(nb.sum())
    row0, Ml = api.row_partition(M, world, rank) if world > 1 else (0, M)
    lib = L.load()
    X = torch.empty((n, Ml), dtype=torch.float64, device=f"cuda:{device}")
    Y = torch.empty((G, Ml), dtype=torch.float64, device=f"cuda:{device}")
    rc = lib.glsgpu_synth_normal(C.c_void_p(X.data_ptr()), Ml, n, Ml, row0, M, seed, 0, device)
    if rc:
        raise api.DeviceError(lib.glsgpu_last_error_message().decode())
    beta = synth._rng(seed, 1).standard_normal(n)
    oh = synth.omega_half(prob.omega)
    rc = lib.glsgpu_synth_response(G, Ml, row0, M, nb.ctypes.data_as(C.POINTER(C.c_int64)), C.c_void_p(X.data_ptr()),
                                   Ml, beta.ctypes.data_as(C.POINTER(C.c_double)),
                                   oh.ctypes.data_as(C.POINTER(C.c_double)), seed, C.c_void_p(Y.data_ptr()), Ml,
                                   device)
    if rc:
        raise api.DeviceError(lib.glsgpu_last_error_message().decode())
    torch.cuda.synchronize(device)
    return DeviceProblem(f"c{config}", G, M, row0, Ml, nb, X, Y, np.asfortranarray(prob.omega), beta, meta["tol"],
                         meta["max_iter"], seed)
