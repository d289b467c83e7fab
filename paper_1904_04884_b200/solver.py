"""Drop-in ``fista`` for the reference's ``holotrack.solver`` (solver.py:38-379).

Same signature, config, report and error behaviour; the solve itself is one
call into ``libholo_b200.so`` (``holo_solve``), which runs the whole FISTA
loop device-resident on a B200 and hands back the COO volume.

Differences a caller can observe (documented in DESIGN.md):
  * arithmetic is float32 on the device with float64 scalars, whatever
    ``cfg.dtype`` says (the north-star parity bar is rel-L2 <= 1e-4 in fp32);
  * ``dense_plane_budget`` is accepted and ignored: the whole volume is
    resident in HBM (it only bounded host memory in the reference);
  * ``real_nonnegative=True`` packs two real planes into one complex stack
    plane (Re / Im) and runs the complex kernels on half as many planes with
    the cosine weights c_2k + i c_2k+1 -- the same operator as the reference's
    half-spectrum rfft layout; its step estimate replays the
    reference's power iteration (same ``default_rng(0)`` start vector,
    generated on the host) on the GPU.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .optics import ComplexField2D, VolumeGeometry
from .prox import RegularizerWeights
from .sparsevol import SparseVolume

__all__ = ["SolverConfig", "SolveReport", "DivergenceError", "fista", "estimate_operator_norm", "DIVERGENCE_FACTOR"]

DIVERGENCE_FACTOR = 1e6  # solver.py:35


@dataclass
class SolverConfig:
    """solver.py:38-68, same fields, defaults and validation."""

    weights: RegularizerWeights = field(default_factory=lambda: RegularizerWeights(0.5, 0.2))
    max_iters: int = 100
    tv_inner_iters: int = 5
    step_policy: str = "backtracking"
    step_size: float | None = None
    bt_shrink: float = 0.5
    stop_tol: float = 0.0
    log_objective: bool = True
    real_nonnegative: bool = False
    dtype: str = "float64"
    dense_plane_budget: int = 16

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        if self.step_size is not None and self.step_size <= 0:
            raise ValueError(f"step_size must be positive, got {self.step_size}")
        if not 0.0 < self.bt_shrink < 1.0:
            raise ValueError(f"bt_shrink must be in (0, 1), got {self.bt_shrink}")
        if self.step_policy not in ("backtracking", "fixed"):
            raise ValueError(f"unknown step_policy {self.step_policy!r}")
        if self.tv_inner_iters < 1:
            raise ValueError(f"tv_inner_iters must be >= 1, got {self.tv_inner_iters}")
        if self.dtype not in ("float64", "float32"):
            raise ValueError(f"dtype must be float64 or float32, got {self.dtype!r}")
        if self.dense_plane_budget < 1:
            raise ValueError("dense_plane_budget must be >= 1")
        if self.stop_tol < 0:
            raise ValueError("stop_tol must be nonnegative")


@dataclass
class SolveReport:
    """solver.py:71-85."""

    objective: list
    iterations: int
    final_sparsity: float
    wall_time: float
    step_size: float
    restarts: int = 0
    diverged: bool = False

    def history_table(self) -> str:
        lines = ["iteration\tobjective"]
        lines += [f"{i}\t{v:.10g}" for i, v in enumerate(self.objective)]
        return "\n".join(lines) + "\n"


class DivergenceError(RuntimeError):
    """solver.py:88-91: raised with the partial report attached."""

    def __init__(self, message: str, report: SolveReport):
        super().__init__(message)
        self.report = report


def native_config(cfg: SolverConfig, step_size: float | None = None) -> nat.SolverConfig:
    """SolverConfig -> the C struct of include/holo_b200.h."""
    w = cfg.weights
    step = cfg.step_size if cfg.step_size is not None else step_size
    return nat.SolverConfig(
        lambda_l1=float(w.lambda_l1), lambda_tv=float(w.lambda_tv), max_iters=int(cfg.max_iters),
        tv_inner_iters=int(cfg.tv_inner_iters), step_policy=nat.POLICY[cfg.step_policy],
        step_size=float(step) if step is not None else -1.0, bt_shrink=float(cfg.bt_shrink),
        stop_tol=float(cfg.stop_tol), log_objective=int(bool(cfg.log_objective)),
        real_nonnegative=int(bool(cfg.real_nonnegative)))


def power_start(geom, seed: int = 0, real: bool = False) -> np.ndarray:
    """The reference's unit-norm start vector (solver.py:231-237): default_rng(seed) normals."""
    rng = np.random.default_rng(seed)
    shape = (geom.nz,) + tuple(geom.plane_shape)
    if real:
        v = rng.standard_normal(shape)
    else:
        v = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    return v / np.linalg.norm(v)


def estimate_operator_norm(geom, iters: int = 10, seed: int = 0, real: bool = False, dtype: str = "float64") -> float:
    """||A||^2 estimate (solver.py:225-247).

    Complex engine: A A^H = nz * (band-limit projector), so the reference's
    power iteration converges to nz after one step (it returns nz to
    ~1e-15); the closed form is returned.  Real engine: the 10-step power
    iteration does NOT converge, so the reference's estimate is
    replayed on the GPU from the identical start vector.
    """
    del dtype
    from .engine import session
    eng = session(geom)
    if not real:
        return eng.operator_norm(False)
    return eng.power_iteration(power_start(geom, seed, True), iters, real=True)


def _check_b(b, geom):
    vals = b.values if hasattr(b, "values") else np.asarray(b)
    if tuple(vals.shape) != tuple(geom.plane_shape):
        raise ValueError(f"hologram shape {vals.shape} does not match geometry {geom.plane_shape}")
    return np.ascontiguousarray(np.real(vals), dtype=np.float64)


def fista(b: ComplexField2D, geom: VolumeGeometry, cfg: SolverConfig):
    """Reconstruct a sparse volume from the hologram residual b (solver.py:254-379).

    Returns (SparseVolume, SolveReport); raises DivergenceError when the
    objective exceeds 1e6 times its initial value and ValueError on a shape
    mismatch or an unsupported plane shape.
    """
    from .engine import session

    t0 = time.perf_counter()
    bb = _check_b(b, geom)
    step = None
    if cfg.real_nonnegative and cfg.step_size is None:
        s2 = estimate_operator_norm(geom, real=True, dtype=cfg.dtype)
        step = 1.0 / (2.0 * s2) if s2 > 0 else 1.0
    ncfg = native_config(cfg, step)
    eng = session(geom)
    code, rep, hist = eng.solve(bb, ncfg)
    per, rows, cols, vals = eng.export_coo()
    vol = SparseVolume.from_coo(geom, per, rows, cols, vals)
    report = SolveReport(
        objective=list(hist) if (cfg.log_objective or code == nat.HOLO_ERR_DIVERGED) else [],
        iterations=int(rep.iterations), final_sparsity=float(rep.final_sparsity),
        wall_time=time.perf_counter() - t0, step_size=float(rep.step_size), restarts=int(rep.restarts),
        diverged=bool(rep.diverged))
    if code == nat.HOLO_ERR_DIVERGED:
        raise DivergenceError(f"objective diverged at iteration {rep.iterations - 1}", report)
    return vol, report
