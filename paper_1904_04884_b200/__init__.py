"""B200-native RIHVR hot path: fused-lasso FISTA holographic volume reconstruction.

Drop-in for ``holotrack.solver.fista`` (arXiv:1904.04884 reference package):
hand-written sm_100a CUDA kernels behind the C ABI in ``include/holo_b200.h``
(``libholo_b200.so``), with a Python mirror of the reference's solver API.
"""

from .optics import ComplexField2D, TransferLadder, VolumeGeometry, adjoint, forward
from .prox import RegularizerWeights, prox_fl, prox_l1, prox_tv_2d
from .solver import DivergenceError, SolveReport, SolverConfig, estimate_operator_norm, fista
from .sparsevol import SparsePlane, SparseVolume, from_dense

__all__ = [
    "ComplexField2D", "VolumeGeometry", "TransferLadder", "forward", "adjoint",
    "RegularizerWeights", "prox_fl", "prox_l1", "prox_tv_2d",
    "SolverConfig", "SolveReport", "DivergenceError", "fista", "estimate_operator_norm",
    "SparsePlane", "SparseVolume", "from_dense",
]
