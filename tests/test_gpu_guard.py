"""The per-plane TV guard (reference prox.py:138-147) on the PRODUCTION prox:
the 64x64 register-strip kernel (single pass, T <= 8) and the multi-pass
strip walk (T > 8), on planes large enough to have interior and edge
regions, and the engine's fix-up inside fista() (engine.cu guard branch:
gradient recompute, forced prox rerun, forward redo).

Inputs that make the guard fire: a plateau (a box of ones in zeros).  FGP
stopped after T steps moves the box edges by about tau and creates new
small steps beside them, which costs more than the TV it removes, so
tau TV(out) + |out - v|^2 / 2 > tau TV(v) and the reference returns v for
that part.  Relative margins 10-27 % (tests below check the oracle fires)."""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import holo_oracle as O

# T -> tau_TV at which the plateau's guard margin is largest (single pass:
# 1 and 5; multi-pass 7+6 and 7+7+6 steps)
TAU_FOR_T = {1: 0.1, 5: 0.5, 13: 1.0, 20: 2.0}


def box(n, r0, r1, c0, c1):
    v = np.zeros((n, n))
    v[r0:r1, c0:c1] = 1.0
    return v


def guard_stack(n=256, seed=0):
    """Three complex planes: the guard fires on Re of plane 0 (interior box),
    on Im of plane 1 (box on the top-left plane corner: edge regions), and on
    neither part of plane 2 (noise, smoothed by the prox)."""
    rng = np.random.default_rng(seed)
    noise = lambda: 0.3 * rng.standard_normal((n, n))  # noqa: E731
    v = np.empty((3, n, n), dtype=np.complex128)
    v[0] = box(n, 80, 176, 64, 192) + 1j * noise()
    v[1] = noise() + 1j * box(n, 0, 72, 0, 100)
    v[2] = noise() + 1j * noise()
    return v


def oracle_fired(v, tau, T):
    """(plane, part) -> the reference guard returned its input."""
    out = np.empty((v.shape[0], 2), dtype=bool)
    for k in range(v.shape[0]):
        for j, part in enumerate((v[k].real, v[k].imag)):
            out[k, j] = np.array_equal(O.fgp_tv(part, tau, T), part)
    return out


EXPECTED = np.array([[True, False], [False, True], [False, False]])


@pytest.mark.parametrize("T", sorted(TAU_FOR_T))
def test_guard_construction_fires_in_oracle(T):
    """CPU pin of the construction: the oracle (pinned to the reference's
    guard golden by test_oracle.py) fires exactly on the box parts."""
    v = guard_stack(128)
    v[0] = box(128, 40, 88, 32, 96) + 1j * v[0].imag
    v[1] = v[1].real + 1j * box(128, 0, 36, 0, 50)
    assert np.array_equal(oracle_fired(v, TAU_FOR_T[T], T), EXPECTED)


@pytest.mark.gpu
@pytest.mark.parametrize("T", sorted(TAU_FOR_T))
def test_strip_prox_guard_fixup_vs_oracle(T):
    """holo_op_prox_fl on 256x256 planes routes through k_prox_strip (single
    pass for T <= 8, the strip walk's first/middle/last passes beyond): the
    guard statistics, the per-plane decision and the forced rerun that
    takes the identity for the failing part match the reference."""
    from paper_1904_04884_b200 import prox as P
    tau_tv, tau_l1 = TAU_FOR_T[T], 0.05
    v = guard_stack(256)
    fired = oracle_fired(v, tau_tv, T)
    assert np.array_equal(fired, EXPECTED)
    ref = O.fused_prox(v, tau_l1, tau_tv, T)
    out = P.prox_fl(v, tau_l1, tau_tv, T)
    assert rel_l2(out, ref) <= 1e-5, rel_l2(out, ref)
    # without the guard's select the fired planes would differ by percents
    unguarded = O.fused_prox(v, tau_l1, tau_tv, T, guard=False)
    for k in range(3):
        assert rel_l2(out[k], ref[k]) <= 1e-5
        if fired[k].any():
            assert rel_l2(out[k], unguarded[k]) > 1e-3
        else:
            assert rel_l2(out[k], unguarded[k]) <= 1e-5


def _guard_geometry(n, nz):
    """z0 = 0 and pitch >> wavelength: H_0 = 1 on every frequency, so A^H b
    on plane 0 is b itself and the first prox input is exactly b (the step
    is 1 / (2 nz) = 1/2 with nz = 1)."""
    from paper_1904_04884_b200 import VolumeGeometry
    return VolumeGeometry(n, n, nz, 10e-6, 10e-6, 0.0, 632e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("T", [5, 20])
def test_fista_guard_fixup_engine_vs_oracle(T):
    """fista() whose first prox input is a plateau: the guard fires inside
    the solve (report.guard_fixups > 0), the engine recomputes the gradient,
    reruns the prox with the force bits and redoes the forward; iterations,
    restarts, objective history and volume match the fp64 oracle."""
    from paper_1904_04884_b200 import ComplexField2D, RegularizerWeights, SolverConfig, fista
    from paper_1904_04884_b200.engine import HoloEngine
    from paper_1904_04884_b200.solver import native_config
    n = 256
    g = _guard_geometry(n, 1)
    tau = TAU_FOR_T[T]
    lam_tv = 2.0 * tau  # tau = step * lambda_TV, step = 1/2
    b = box(n, 60, 140, 90, 200) - 0.5 * box(n, 170, 230, 20, 90)
    scfg = SolverConfig(weights=RegularizerWeights(0.02, lam_tv), max_iters=6, tv_inner_iters=T)
    og = O.Geometry.of(g)
    ref = O.fista_solve(b, og, lam_l1=0.02, lam_tv=lam_tv, max_iters=6, inner=T)
    # the construction: the reference's first prox fires on Re (Im is 0)
    assert np.array_equal(O.fgp_tv(b, tau, T), b)
    eng = HoloEngine(g)
    code, rep, hist = eng.solve(b, native_config(scfg))
    assert rep.guard_fixups > 0
    eng.close()
    vol, rep2 = fista(ComplexField2D(b, g.pitch, g.wavelength), g, scfg)
    assert rep2.iterations == ref.iterations and rep2.restarts == ref.restarts
    assert abs(rep2.step_size - ref.step) <= 1e-12 * ref.step
    assert np.allclose(rep2.objective, ref.history, rtol=2e-5, atol=1e-9)
    assert rel_l2(vol.to_dense(), ref.x) <= 1e-4, rel_l2(vol.to_dense(), ref.x)
