"""CPU: pin oracle/holo_oracle.py to the golden vectors produced by the reference
(tests/golden/make_golden.py).  Tolerances are fp64 round-off level."""
import numpy as np
import pytest

from conftest import FISTA_CASES, dense_from_golden, fista_kwargs, geom_of, golden, rel_l2
from oracle import holo_oracle as O


@pytest.mark.parametrize("name", ["ops_a", "ops_evan"])
def test_operators_match_reference(name):
    d = golden(name)
    g = geom_of(d["geom"])
    assert rel_l2(O.transfer_stack(g, 0, g.nz), d["transfer"]) < 1e-13
    assert rel_l2(O.transfer_stack(g, 0, g.nz, conj=True), d["transfer_conj"]) < 1e-13
    assert rel_l2(O.sensor_forward(d["x"], g, chunk=4), d["forward"]) < 1e-12
    assert rel_l2(O.sensor_forward(d["x"], g), d["forward_optics"]) < 1e-12
    bp = O.back_project(d["r"], g)
    assert rel_l2(bp, d["adjoint"]) < 1e-12
    assert rel_l2(2.0 * bp, d["gradient"]) < 1e-12


def test_real_engine_operators_match_reference():
    d = golden("ops_real")
    g = geom_of(d["geom"])
    assert rel_l2(O.real_forward(d["x"], g), d["forward"]) < 1e-12
    assert rel_l2(2.0 * O.real_back_project(d["r"], g), d["gradient"]) < 1e-12
    assert abs(O.power_norm(g, real=True) - float(d["sigma2"])) < 1e-9 * float(d["sigma2"])
    # the real engine is the complex engine restricted to real volumes
    assert rel_l2(O.sensor_forward(d["x"].astype(complex), g), d["forward"]) < 1e-12
    assert rel_l2(O.back_project(d["r"], g).real, 0.5 * d["gradient"]) < 1e-12


def test_power_iteration_matches_reference():
    d = golden("ops_a")
    g = geom_of(d["geom"])
    s2 = O.power_norm(g)
    assert abs(s2 - float(d["sigma2"])) < 1e-10 * g.nz
    assert abs(s2 - g.nz) < 1e-9 * g.nz  # A A^H = nz * projector


def test_prox_matches_reference():
    d = golden("prox")
    v = d["v"]
    for key in d:
        if key.startswith("fl_T"):
            _, t, tl, tt = key.split("_")
            out = O.fused_prox(v, float(tl), float(tt), int(t[1:]))
            assert np.max(np.abs(out - d[key])) < 1e-12, key
    for T in (1, 5):
        out = O.fgp_tv(d["real"], 0.4, T)
        assert np.max(np.abs(out - d[f"tv_real_T{T}"])) < 1e-12
    tvn = [O.tv_norm(v[i].real) for i in range(3)] + [O.tv_norm(v[i].imag) for i in range(3)]
    assert np.allclose(tvn, d["tv_norm"], rtol=1e-13)
    assert np.max(np.abs(O.soft_threshold(v, 0.25) - d["l1_025"])) < 1e-14
    # guard: FGP output rejected for exactly the planes the reference rejected
    out = O.fused_prox(d["guard_v"], 0.05, 0.34, 1)
    assert np.max(np.abs(out - d["guard_out"])) < 1e-14
    assert d["guard_fired"].any() and not d["guard_fired"].all()


def test_spec_pins():
    # prox_l1(+-2, 0.5) = +-1.5; const plane unchanged by TV
    assert np.allclose(O.soft_threshold(np.array([2.0, -2.0]), 0.5), [1.5, -1.5])
    c = np.full((6, 7), 0.3)
    assert np.array_equal(O.fgp_tv(c, 0.7, 5), c)
    assert O.tv_norm(np.array([[0.0, 1.0]])) == 1.0
    # H(0, 0, z = lam) = 1; evanescent -> 0
    lam = 632e-9
    h = O.transfer(4, 4, 10e-6, lam, lam)
    assert abs(h[0, 0] - 1.0) < 1e-12
    hev = O.transfer(4, 4, lam / 1.5 / 2, lam, 1e-3)  # pitch so that lam * f_nyq = 1.5
    assert hev[0, 2] == 0


@pytest.mark.parametrize("name", [c for c in FISTA_CASES if c != "fista_c1"])
def test_fista_matches_reference(name):
    d = golden(name)
    g = geom_of(d["geom"])
    res = O.fista_solve(d["b"], g, **fista_kwargs(d))
    assert res.diverged == bool(d["diverged"])
    assert res.iterations == int(d["iterations"])
    assert res.restarts == int(d["restarts"])
    assert abs(res.step - float(d["step"])) <= 1e-14 * abs(float(d["step"]))
    assert np.allclose(res.history, d["history"], rtol=1e-9, atol=0)
    if not res.diverged:
        assert rel_l2(res.x, dense_from_golden(d)) < 1e-9
        assert res.nnz == len(d["v"])


def test_detection_matches_reference():
    d = golden("fista_128")
    x = dense_from_golden(d)
    g = geom_of(d["geom"])
    dets = O.detect_particles(x, 2 / 256, 5)
    ref = d["detections"]
    assert dets.shape == ref.shape
    assert np.allclose(dets, ref, atol=1e-9)


@pytest.mark.slow
def test_fista_c1_matches_reference():
    d = golden("fista_c1")
    g = geom_of(d["geom"])
    res = O.fista_solve(d["b"], g, **fista_kwargs(d))
    assert np.allclose(res.history, d["history"], rtol=1e-9)
    assert rel_l2(res.x, dense_from_golden(d)) < 1e-9


def test_synthetic_inputs_match_reference():
    # the oracle's scene/render/noise restatement reproduces the reference's b
    d = golden("fista_64")
    g = geom_of(d["geom"])
    pts = O.make_scene(8, g, 20e-6, seed=11, margin_planes=2)
    assert np.allclose(pts, d["truth"], rtol=0, atol=0)
    b = O.invert_residual(O.add_noise(O.render_hologram(pts, g, 20e-6), 0.02, seed=18))
    assert np.max(np.abs(b - d["b"])) < 1e-12
