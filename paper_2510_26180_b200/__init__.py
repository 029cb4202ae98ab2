"""B200-native KLE-CGC hot path (arXiv 2510.26180): the fine propagator, the
diagonalised coarse-grid correction and the Hermite-gPC surrogate
evaluation as sm_100a CUDA kernels behind a C ABI (``include/kle_b200.h``),
with a host API mirroring the reference package ``pintuq``.
"""
from .core import (
    CoarseTrajectory,
    ConfigError,
    DeviceError,
    InitMode,
    IterationRecord,
    IterationTrace,
    MaxItersExceededError,
    NonConvergenceError,
    ParameterSample,
    PintuqError,
    RankDeficientError,
    RngStream,
    SingularShiftError,
    SnapshotError,
    SolverConfig,
    TimeGrid,
    make_time_grid,
)
from .models import (AllenCahn1D, Burgers1D, LinearModel, LogNormalKL1D, LogNormalKL2D, Model, ParameterMap,
                     get_model)

__version__ = "0.1.0"

__all__ = [
    "AllenCahn1D", "Burgers1D", "CoarseTrajectory", "ConfigError", "DeviceError", "InitMode", "IterationRecord", "IterationTrace",
    "LinearModel", "LogNormalKL1D", "LogNormalKL2D", "MaxItersExceededError", "Model", "NonConvergenceError",
    "ParameterMap", "ParameterSample", "PintuqError", "RankDeficientError", "RngStream",
    "SingularShiftError", "SnapshotError", "SolverConfig", "TimeGrid", "get_model", "make_time_grid",
]
