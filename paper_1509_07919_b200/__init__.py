"""B200-native SaP (split-and-parallelize) banded solver hot path (arXiv 1509.07919).

The compute path is libsap_gpu.so (hand-written sm_100a CUDA + C++ host
logic behind the C ABI in include/sap_gpu.h); this package is the Python
mirror of the reference's setup()/solve() interface over that ABI.
"""
from ._lib import LIB_PATH, load  # noqa: F401
from .solver import (  # noqa: F401
    CudaError,
    KrylovFailure,
    KrylovMethod,
    KrylovOptions,
    PartitionLayout,
    PrecondKind,
    PreconditionerError,
    SolveStats,
    Solver,
    StateError,
    make_partition_layout,
    max_feasible_partitions,
    random_banded,
)

__all__ = [
    "Solver", "KrylovOptions", "SolveStats", "PrecondKind", "KrylovMethod", "KrylovFailure", "PartitionLayout",
    "PreconditionerError", "StateError", "CudaError", "make_partition_layout", "max_feasible_partitions",
    "random_banded", "load", "LIB_PATH",
]
