"""B200-native QSVM quantum-kernel engine (arXiv 2405.02630, cuTN-QSVM hot path).

Public API (mirrors the reference's SPEC kernel_pipeline):

    from paper_2405_02630_b200 import FeatureMapConfig, compute_kernel_matrix, compute_cross_kernel
    K = compute_kernel_matrix(X_train, FeatureMapConfig(784)).entries       # N x N, fp64
    Kx = compute_cross_kernel(X_test, X_train, FeatureMapConfig(784)).entries
    K, Kx = compute_kernel_matrices(X_train, X_test, FeatureMapConfig(784))  # one pass, both

Compute runs only in libqk.so (hand-written sm_100a CUDA, C ABI in include/qk.h).
"""
from .config import FeatureMapConfig
from .engine import contract_batch
from .errors import (CapacityError, ConfigError, ConvergenceError, DataFormatError, DeviceError,
                     NativeLibraryError, RebindError, ShardMergeError, SliceInfeasibleError,
                     StructuralError, TnkernelError)
from .kernel_pipeline import (KernelMatrix, compute_cross_kernel, compute_kernel_matrices,
                              compute_kernel_matrix, compute_kernel_shard, enumerate_pairs,
                              shard_merge, shard_range, symmetrize)
from .planner import SweepPlan, plan_for

__all__ = [
    "FeatureMapConfig", "KernelMatrix", "SweepPlan", "plan_for", "compute_kernel_matrix",
    "compute_cross_kernel", "compute_kernel_matrices", "compute_kernel_shard", "contract_batch",
    "enumerate_pairs", "symmetrize", "shard_merge", "shard_range", "TnkernelError",
    "ConfigError", "DataFormatError", "CapacityError", "StructuralError", "RebindError",
    "ShardMergeError", "SliceInfeasibleError", "ConvergenceError", "NativeLibraryError",
    "DeviceError",
]
