"""Fused-lasso proximal operators on the GPU (prox.py:15-165 of the reference).

``prox_fl``/``prox_tv_2d``/``prox_l1`` take plane stacks (..., ny, nx) of any
shape and run the fused prox kernel (FGP-TV with the per-plane guard, then
the complex soft threshold) through ``holo_op_prox_fl``.  Computation is
float32 on the device; results come back as float64/complex128 arrays like
the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["RegularizerWeights", "prox_l1", "prox_tv_2d", "prox_fl"]


@dataclass(frozen=True)
class RegularizerWeights:
    """Fused-lasso weights (prox.py:26-35)."""

    lambda_l1: float
    lambda_tv: float

    def __post_init__(self):
        if self.lambda_l1 < 0 or self.lambda_tv < 0:
            raise ValueError(f"regularizer weights must be nonnegative, got {self}")


def _run(v, tau_l1, tau_tv, inner):
    from .engine import prox_session
    v = np.asarray(v)
    if v.ndim < 2:
        raise ValueError("prox operators take (..., ny, nx) planes")
    shape = v.shape
    stack = v.reshape(-1, shape[-2], shape[-1])
    out = prox_session().prox_fl(stack, tau_l1, tau_tv, inner)
    return out.reshape(shape)


def prox_fl(v, tau_l1: float, tau_tv: float, inner_iters: int = 5):
    """soft-threshold(prox_tv(Re) + i prox_tv(Im)) (prox.py:151-165)."""
    if tau_l1 < 0 or tau_tv < 0:
        raise ValueError("tau must be nonnegative")
    if inner_iters < 1:
        raise ValueError(f"inner_iters must be >= 1, got {inner_iters}")
    v = np.asarray(v)
    out = _run(v, tau_l1, tau_tv, inner_iters)
    return out if np.iscomplexobj(v) else out.real


def prox_tv_2d(v, tau: float, inner_iters: int = 5):
    """FGP TV prox of real planes with the never-worse guard (prox.py:104-148)."""
    if tau < 0:
        raise ValueError(f"tau must be nonnegative, got {tau}")
    if inner_iters < 1:
        raise ValueError(f"inner_iters must be >= 1, got {inner_iters}")
    v = np.asarray(v, dtype=np.float64)
    if tau == 0:
        return v.copy()
    return _run(v, 0.0, tau, inner_iters).real


def prox_l1(v, tau: float):
    """Complex soft threshold, |v| <= tau -> 0 (prox.py:83-96)."""
    if tau < 0:
        raise ValueError(f"tau must be nonnegative, got {tau}")
    v = np.asarray(v)
    if tau == 0:
        return v.copy()
    out = _run(v if v.ndim >= 2 else v.reshape(1, -1), tau, 0.0, 1).reshape(v.shape)
    return out if np.iscomplexobj(v) else out.real
