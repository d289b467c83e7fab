"""Plane sides that are not powers of two (the reference's numpy FFTs take any
size, optics.py:119-122, solver.py:117-132): the mixed-radix passes of
csrc/gfft.cu against numpy and the fp64 oracle (pinned to the reference by
test_oracle.py), operators and end-to-end fista() in both engines."""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import holo_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nx,ny", [(96, 80), (100, 100), (210, 126), (1280, 24), (24, 1080), (122, 61), (1000, 8),
                                   (99, 35), (1021, 8), (134, 67),
                                   (96, 64), (64, 96), (100, 64)])  # one fused side (see Plan::generic_x / _y)
def test_fft2_general_sizes(nx, ny):
    from paper_1904_04884_b200 import VolumeGeometry
    from paper_1904_04884_b200.engine import HoloEngine
    eng = HoloEngine(VolumeGeometry(nx, ny, 1, 1e-5, 1e-5, 5e-3, 632e-9))
    rng = np.random.default_rng(nx * 31 + ny)
    x = rng.standard_normal((2, ny, nx)) + 1j * rng.standard_normal((2, ny, nx))
    f = eng.fft2(x)
    tol = 3e-6 if max(nx, ny) <= 2048 and all(_largest_prime(n) <= 7 for n in (nx, ny)) else 2e-5  # direct DFTs
    assert rel_l2(f, np.fft.fft2(x)) < tol
    assert rel_l2(eng.fft2(f, inverse=True), x) < tol
    eng.close()


def _largest_prime(n):
    best, p = 1, 2
    while n > 1:
        while n % p == 0:
            best, n = p, n // p
        p += 1
    return best


@pytest.mark.parametrize("nx,ny,nz", [(100, 60, 5), (96, 200, 3), (1280, 40, 2),
                                      (1280, 64, 2), (64, 1080, 2)])  # mixed-radix rows + fused TMA columns, and back
def test_forward_adjoint_general_sizes_vs_oracle(nx, ny, nz):
    from paper_1904_04884_b200 import VolumeGeometry
    from paper_1904_04884_b200.engine import HoloEngine
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    og = O.Geometry.of(g)
    eng = HoloEngine(g)
    rng = np.random.default_rng(nx + ny + nz)
    x = (rng.standard_normal((nz, ny, nx)) + 1j * rng.standard_normal((nz, ny, nx))) * (rng.random((nz, ny, nx)) < 0.1)
    assert rel_l2(eng.forward(x), O.sensor_forward(x, og)) < 1e-5
    r = rng.standard_normal((ny, nx))
    assert rel_l2(eng.adjoint(r), O.back_project(r, og)) < 1e-5
    eng.close()


@pytest.mark.parametrize("shape,inner,real", [((100, 120, 4), 5, False),   # strip prox on a 100-wide plane
                                              ((96, 80, 3), 13, False),    # multi-pass strip walk
                                              ((40, 24, 3), 5, False),     # generic prox (planes < 64)
                                              ((100, 72, 3), 5, True),     # packed real engine, odd nz
                                              ((99, 70, 3), 5, False),     # odd nx: generic tile prox
                                              ((75, 66, 3), 13, True),     # odd nx, real engine, T = 13
                                              ((134, 67, 2), 5, False),    # prime factors 67 (direct DFT lines)
                                              ((96, 64, 3), 5, False),     # mixed-radix rows, fused columns
                                              ((64, 96, 4), 13, True),     # fused rows, mixed-radix columns, real
                                              ((1000, 1000, 2), 5, False)])  # a 1000x1000 camera frame
def test_fista_general_sizes_vs_oracle(shape, inner, real):
    from paper_1904_04884_b200 import ComplexField2D, RegularizerWeights, SolverConfig, VolumeGeometry, fista
    nx, ny, nz = shape
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    og = O.Geometry.of(g)
    pts = O.make_scene(6, og, 30e-6, seed=nx + ny + nz + inner)
    b = O.invert_residual(O.add_noise(O.render_hologram(pts, og, 30e-6), 0.01, seed=1))
    iters = 5 if nx >= 1000 else 12
    step = 1.0 / (2.0 * O.power_norm(og, real=True)) if real else None
    ref = O.fista_solve(b, og, lam_l1=0.05, lam_tv=0.1, max_iters=iters, inner=inner, real=real, step_size=step)
    vol, rep = fista(ComplexField2D(b, g.pitch, g.wavelength), g,
                     SolverConfig(weights=RegularizerWeights(0.05, 0.1), max_iters=iters, tv_inner_iters=inner,
                                  real_nonnegative=real, step_size=step))
    assert rep.iterations == ref.iterations and rep.restarts == ref.restarts
    assert np.allclose(rep.objective, ref.history, rtol=2e-5, atol=1e-9)
    assert rel_l2(vol.to_dense(), ref.x) <= 1e-4


@pytest.mark.parametrize("nranks,real", [(2, False), (3, True)])
def test_rank_group_general_sizes(nranks, real):
    """z-sharded engine (in-process rank group, peer-memory plane sum over a
    P that is not a power of two) on a 100x72 geometry: identical decisions
    and the unsharded volume."""
    import threading
    from paper_1904_04884_b200 import RegularizerWeights, VolumeGeometry, estimate_operator_norm
    from paper_1904_04884_b200.engine import HoloEngine
    from paper_1904_04884_b200.solver import SolverConfig, native_config
    g = VolumeGeometry(100, 72, 6, 10e-6, 10e-6, 5e-3, 632e-9)
    og = O.Geometry.of(g)
    pts = O.make_scene(6, og, 30e-6, seed=5)
    b = np.ascontiguousarray(O.invert_residual(O.add_noise(O.render_hologram(pts, og, 30e-6), 0.01, seed=1)))
    step = 1.0 / (2.0 * estimate_operator_norm(g, real=True)) if real else None
    cfg = native_config(SolverConfig(weights=RegularizerWeights(0.05, 0.1), max_iters=12, tv_inner_iters=5,
                                     real_nonnegative=real, step_size=step))
    group = HoloEngine.local_group(g, nranks)
    out, errs = [None] * nranks, []

    def run(r):
        try:
            out[r] = group[r].solve(b, cfg)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    plain = HoloEngine(g)
    _, rp, hp = plain.solve(b, cfg)
    for _, rs, hs in out:
        assert (rs.iterations, rs.restarts) == (rp.iterations, rp.restarts)
        assert np.allclose(hs, hp, rtol=1e-5)
    xs = np.concatenate([e.solution_dense().cpu().numpy() for e in group])
    assert rel_l2(xs, plain.solution_dense().cpu().numpy()) < 1e-5
    for e in group:
        e.close()
    plain.close()
