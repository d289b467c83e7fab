"""The interior-first region order of the engine's main prox launch
(prox_strip.cu `ordered_work`, the T = 5 FAST kernel) changes only the order in
which a CTA visits regions: every region is computed by the same code with the
same inputs and writes its own tiles and partial-sum slots, so fista() must
give bit-identical volumes and histories with the order switched off
(HOLO_PROX_NOORD, read at every launch).  Plane shapes cover square and
non-square interiors, a plane too short to have interior regions (ordered
launch not taken) and several planes per stack (the per-plane interior /
edge-ring enumeration)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(128, 128), (256, 128), (128, 512), (512, 256), (64, 256)]  # (ny, nx)


def _solve(ny, nx, nz, seed):
    from paper_1904_04884_b200 import ComplexField2D, RegularizerWeights, SolverConfig, VolumeGeometry, fista
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    b = np.random.default_rng(seed).standard_normal((ny, nx))
    cfg = SolverConfig(weights=RegularizerWeights(0.05, 0.2), max_iters=3, tv_inner_iters=5)
    vol, rep = fista(ComplexField2D(b, g.pitch, g.wavelength), g, cfg)
    return vol.to_dense(), np.array(rep.objective)


@pytest.mark.parametrize("shape", SHAPES)
def test_region_order_is_bit_identical(shape):
    ny, nx = shape
    x0, h0 = _solve(ny, nx, 3, 7)
    os.environ["HOLO_PROX_NOORD"] = "1"
    try:
        x1, h1 = _solve(ny, nx, 3, 7)
    finally:
        del os.environ["HOLO_PROX_NOORD"]
    assert np.count_nonzero(x0) > 0
    assert np.array_equal(x0, x1)
    assert np.array_equal(h0, h1)
