"""Sparsity-aware forward (north_star; the reference's forward_sparse skips
all-zero chunks and planes, solver.py:110-124, :115 and :119).

The engine marks a stack plane of the prox output dead when its sum |x_new| is
exactly zero (k_prox_reduce) and the forward row and column passes then
neither read nor transform it.  Skipping must be exact: the same solve with
the skipping switched off (HOLO_NO_PLANE_SKIP=1 at engine creation) gives the
same volume and objective history bit for bit, and both match the oracle."""
import os

import numpy as np
import pytest

from conftest import rel_l2
from oracle import holo_oracle as O

pytestmark = pytest.mark.gpu

GEOM = (128, 128, 16, 10e-6, 100e-6, 2e-3, 632e-9)


def _hologram(seed=1):
    g = O.Geometry(*GEOM)
    pts = O.make_scene(3, g, 40e-6, seed=seed, margin_planes=2)
    return O.invert_residual(O.render_hologram(pts, g, 40e-6))


def _solve(b, lam_l1, lam_tv, iters, inner, skip, real=False, geom=GEOM):
    from paper_1904_04884_b200 import RegularizerWeights, SolverConfig, VolumeGeometry
    from paper_1904_04884_b200.engine import HoloEngine
    from paper_1904_04884_b200.solver import native_config

    g = VolumeGeometry(*geom)
    old = os.environ.pop("HOLO_NO_PLANE_SKIP", None)
    if not skip:
        os.environ["HOLO_NO_PLANE_SKIP"] = "1"
    try:
        eng = HoloEngine(g)  # the switch is read when the handle is created
    finally:
        os.environ.pop("HOLO_NO_PLANE_SKIP", None)
        if old is not None:
            os.environ["HOLO_NO_PLANE_SKIP"] = old
    cfg = native_config(SolverConfig(weights=RegularizerWeights(lam_l1, lam_tv), max_iters=iters,
                                     tv_inner_iters=inner, step_size=1.0 / (2 * geom[2]),
                                     real_nonnegative=real))
    code, rep, hist = eng.solve(np.ascontiguousarray(b, dtype=np.float64), cfg)
    assert code == 0
    x = eng.solution_dense().cpu().numpy()
    eng.close()
    return x, rep, np.asarray(hist)


@pytest.mark.parametrize("lam_l1,inner", [(3.0, 5), (3.5, 5), (3.0, 20)])
def test_skipping_is_exact_and_matches_oracle(lam_l1, inner):
    b = _hologram()
    x1, r1, h1 = _solve(b, lam_l1, 0.2, 8, inner, skip=True)
    x0, r0, h0 = _solve(b, lam_l1, 0.2, 8, inner, skip=False)
    assert r1.skipped_planes > 0 and r0.skipped_planes == 0
    assert np.array_equal(h1, h0)
    assert np.array_equal(x1, x0)
    assert (r1.iterations, r1.restarts, r1.attempts) == (r0.iterations, r0.restarts, r0.attempts)
    ref = O.fista_solve(b, O.Geometry(*GEOM), lam_l1=lam_l1, lam_tv=0.2, max_iters=8, inner=inner,
                        step_size=1.0 / 32)
    dead_ref = [k for k in range(GEOM[2]) if not np.any(ref.x[k])]
    dead_gpu = [k for k in range(GEOM[2]) if not np.any(x1[k])]
    assert dead_gpu == dead_ref and len(dead_ref) > 0
    assert rel_l2(x1, ref.x) <= 1e-4, rel_l2(x1, ref.x)
    assert np.allclose(h1, ref.history, rtol=2e-5, atol=1e-9)


def test_all_planes_dead():
    # lambda_L1 above every |v|: the first prox zeroes the volume and every
    # later forward skips all planes (x stays 0, like the reference)
    b = _hologram()
    x, rep, hist = _solve(b, 50.0, 0.2, 4, 5, skip=True)
    assert not np.any(x)
    assert rep.skipped_planes == rep.attempts * GEOM[2]
    ref = O.fista_solve(b, O.Geometry(*GEOM), lam_l1=50.0, lam_tv=0.2, max_iters=4, inner=5, step_size=1.0 / 32)
    assert not np.any(ref.x)
    assert np.allclose(hist, ref.history, rtol=2e-5, atol=1e-9)


def test_real_engine_skipping_is_exact():
    # packed real engine: a stack plane holds two real planes and is dead when
    # both are (here planes 2+3 and 6+7 end up zero)
    b = _hologram(seed=1)
    x1, r1, h1 = _solve(b, 1.2, 0.2, 6, 5, skip=True, real=True)
    x0, r0, h0 = _solve(b, 1.2, 0.2, 6, 5, skip=False, real=True)
    assert r1.skipped_planes > 0 and r0.skipped_planes == 0
    assert np.array_equal(h1, h0)
    assert np.array_equal(x1, x0)
    ref = O.fista_solve(b, O.Geometry(*GEOM), lam_l1=1.2, lam_tv=0.2, max_iters=6, inner=5, step_size=1.0 / 32,
                        real=True)
    assert rel_l2(x1, ref.x) <= 1e-4, rel_l2(x1, ref.x)
    assert np.allclose(h1, ref.history, rtol=2e-5, atol=1e-9)


def test_skipping_on_general_plane_sides():
    """The mixed-radix passes (gfft.cu, sides that are not powers of two) skip
    dead planes exactly like the fused passes."""
    geom = (120, 96, 16, 10e-6, 100e-6, 2e-3, 632e-9)
    g = O.Geometry(*geom)
    pts = O.make_scene(3, g, 40e-6, seed=1, margin_planes=2)
    b = O.invert_residual(O.render_hologram(pts, g, 40e-6))
    x1, r1, h1 = _solve(b, 3.0, 0.2, 8, 5, skip=True, geom=geom)
    x0, r0, h0 = _solve(b, 3.0, 0.2, 8, 5, skip=False, geom=geom)
    assert r1.skipped_planes > 0 and r0.skipped_planes == 0
    assert np.array_equal(h1, h0) and np.array_equal(x1, x0)
    ref = O.fista_solve(b, g, lam_l1=3.0, lam_tv=0.2, max_iters=8, inner=5, step_size=1.0 / 32)
    assert [k for k in range(16) if not np.any(x1[k])] == [k for k in range(16) if not np.any(ref.x[k])]
    assert rel_l2(x1, ref.x) <= 1e-4
