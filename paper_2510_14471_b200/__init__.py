"""paper_2510_14471_b200 -- B200-native GLS-PCG (PCG-Aug) for SUR models (arXiv 2510.14471 hot path).

The product is the CUDA library libglsgpu.so (csrc/, C-ABI in include/glsgpu.h); this package is
its host-side mirror of the reference's C++ solver API (api.py) plus synthetic inputs (synth.py).
"""
from .api import (AugSolveResult, CostCounters, CostReport, DeviceError, DimensionMismatch, GlsError, GlsSolution,
                  GpuSurPreconditioner, PcgConfig, PcgTrace, RankDeficient, SingularD, SingularTriangular, SurModel,
                  Termination, cost_counters, device_count, make_sur, operator_norm_probe, pcg_aug, sur_from_problem,
                  sur_preconditioner)

__all__ = [
    "AugSolveResult", "CostCounters", "CostReport", "DeviceError", "DimensionMismatch", "GlsError", "GlsSolution",
    "GpuSurPreconditioner", "PcgConfig", "PcgTrace", "RankDeficient", "SingularD", "SingularTriangular", "SurModel",
    "Termination", "cost_counters", "device_count", "make_sur", "operator_norm_probe", "pcg_aug", "sur_from_problem",
    "sur_preconditioner",
]
