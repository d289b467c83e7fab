"""GPU parity of the operator kernels against the reference goldens and the oracle.
Tolerances are float32-level (the device computes in fp32 with fp64 scalars)."""
import numpy as np
import pytest

from conftest import geom_of, golden, rel_l2
from oracle import holo_oracle as O

pytestmark = pytest.mark.gpu


def _geom(d):
    from paper_1904_04884_b200 import VolumeGeometry
    nx, ny, nz, pitch, dz, z0, lam = d["geom"]
    return VolumeGeometry(int(nx), int(ny), int(nz), pitch, dz, z0, lam)


@pytest.fixture(scope="module")
def eng_a():
    from paper_1904_04884_b200.engine import HoloEngine
    d = golden("ops_a")
    return HoloEngine(_geom(d)), d


@pytest.mark.parametrize("name", ["ops_a", "ops_evan"])
def test_transfer_forward_adjoint(name):
    from paper_1904_04884_b200.engine import HoloEngine
    d = golden(name)
    eng = HoloEngine(_geom(d))
    g = geom_of(d["geom"])
    h = eng.transfer(0, g.nz)
    assert np.max(np.abs(h - d["transfer"])) < 2e-6
    assert np.max(np.abs(eng.transfer(0, g.nz, conj=True) - d["transfer_conj"])) < 2e-6
    assert rel_l2(eng.forward(d["x"]), d["forward"]) < 2e-6
    assert rel_l2(eng.adjoint(d["r"]), d["adjoint"]) < 2e-6
    assert rel_l2(eng.adjoint(d["r"], scale=2.0), d["gradient"]) < 2e-6
    eng.close()


@pytest.mark.parametrize("ny,nx,nz", [(2048, 64, 40),   # TMA-staged forward columns (2 per CTA), 2 plane groups
                                      (4096, 32, 3),    # direct-load forward columns, 1024-thread adjoint
                                      (1024, 64, 70)])  # Horner / recurrence across 32-plane groups
def test_forward_adjoint_tall_columns_vs_oracle(ny, nx, nz):
    """Forward (Horner z-accumulation per plane group) and adjoint (transfer
    recurrence, staged bulk stores) for the column lengths of C3/C4 and
    beyond, against the fp64 oracle."""
    from paper_1904_04884_b200 import VolumeGeometry
    from paper_1904_04884_b200.engine import HoloEngine
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    og = O.Geometry.of(g)
    eng = HoloEngine(g)
    rng = np.random.default_rng(ny + nz)
    x = (rng.standard_normal((nz, ny, nx)) + 1j * rng.standard_normal((nz, ny, nx))) * (rng.random((nz, ny, nx)) < 0.1)
    assert rel_l2(eng.forward(x), O.sensor_forward(x, og)) < 1e-5
    r = rng.standard_normal((ny, nx))
    assert rel_l2(eng.adjoint(r), O.back_project(r, og)) < 1e-5
    eng.close()


@pytest.mark.parametrize("n", [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
def test_fft2_all_sizes(n):
    from paper_1904_04884_b200 import VolumeGeometry
    from paper_1904_04884_b200.engine import HoloEngine
    ny = n if n <= 1024 else 16
    eng = HoloEngine(VolumeGeometry(n, ny, 1, 1e-5, 1e-5, 5e-3, 632e-9))
    rng = np.random.default_rng(n)
    x = rng.standard_normal((2, ny, n)) + 1j * rng.standard_normal((2, ny, n))
    f = eng.fft2(x)
    assert rel_l2(f, np.fft.fft2(x)) < 3e-6
    b = eng.fft2(f, inverse=True)
    assert rel_l2(b, x) < 3e-6
    eng.close()
    # column transforms of tall planes
    eng = HoloEngine(VolumeGeometry(16, n, 1, 1e-5, 1e-5, 5e-3, 632e-9))
    x = rng.standard_normal((1, n, 16)) + 1j * rng.standard_normal((1, n, 16))
    assert rel_l2(eng.fft2(x), np.fft.fft2(x)) < 3e-6
    eng.close()


def test_adjointness_full_width():
    """<A x, r> = Re<x, A^H r> at the C3 plane size."""
    from paper_1904_04884_b200 import VolumeGeometry
    from paper_1904_04884_b200.engine import HoloEngine
    g = VolumeGeometry(1024, 1024, 4, 10e-6, 10e-6, 5e-3, 632e-9)
    eng = HoloEngine(g)
    rng = np.random.default_rng(3)
    for _ in range(3):
        x = (rng.standard_normal((4, 1024, 1024)) + 1j * rng.standard_normal((4, 1024, 1024))) * (
            rng.random((4, 1024, 1024)) < 0.01)
        r = rng.standard_normal((1024, 1024))
        lhs = float(np.sum(eng.forward(x) * r))
        rhs = float(np.real(np.vdot(eng.adjoint(r), x)))
        assert abs(lhs - rhs) <= 1e-5 * max(abs(lhs), 1.0)
    # and against the fp64 oracle on the same input
    og = O.Geometry.of(g)
    assert rel_l2(eng.forward(x), O.sensor_forward(x, og)) < 5e-6
    eng.close()


def test_long_plane_stacks_vs_oracle():
    """Forward and adjoint over 2.5 transfer-recurrence lengths of planes (the column
    passes carry H_k from plane to plane by one complex multiply, re-anchored
    exactly every 32 planes) against the fp64 oracle."""
    from paper_1904_04884_b200 import VolumeGeometry
    from paper_1904_04884_b200.engine import HoloEngine
    g = VolumeGeometry(128, 128, 80, 10e-6, 10e-6, 5e-3, 632e-9)
    eng = HoloEngine(g)
    og = O.Geometry.of(g)
    rng = np.random.default_rng(11)
    x = (rng.standard_normal((80, 128, 128)) + 1j * rng.standard_normal((80, 128, 128))) * (
        rng.random((80, 128, 128)) < 0.05)
    r = rng.standard_normal((128, 128))
    assert rel_l2(eng.forward(x), O.sensor_forward(x, og)) < 5e-6
    adj = eng.adjoint(r)
    ref = O.back_project(r, og)
    assert rel_l2(adj, ref) < 5e-6
    # per-plane error stays flat across the recurrence (no drift with k)
    per = [rel_l2(adj[k], ref[k]) for k in range(80)]
    assert max(per) < 5e-6
    eng.close()


def test_prox_matches_reference():
    from paper_1904_04884_b200 import prox_fl, prox_l1, prox_tv_2d
    d = golden("prox")
    v = d["v"]
    for key in d:
        if key.startswith("fl_T"):
            _, t, tl, tt = key.split("_")
            out = prox_fl(v, float(tl), float(tt), int(t[1:]))
            err = np.max(np.abs(out - d[key])) / max(np.max(np.abs(d[key])), 1e-30)
            assert err < 1e-5, (key, err)
    for T in (1, 5):
        out = prox_tv_2d(d["real"], 0.4, T)
        assert np.max(np.abs(out - d[f"tv_real_T{T}"])) < 1e-5
    assert np.max(np.abs(prox_l1(v, 0.25) - d["l1_025"])) < 1e-6
    # guard: same planes rejected as in the reference
    out = prox_fl(d["guard_v"], 0.05, 0.34, 1)
    assert np.max(np.abs(out - d["guard_out"])) < 1e-5


def test_prox_spec_pins():
    from paper_1904_04884_b200 import prox_fl, prox_l1, prox_tv_2d
    assert np.allclose(prox_l1(np.array([[2.0, -2.0, 0.0]]), 0.5), [[1.5, -1.5, 0.0]])
    c = np.full((3, 40, 33), 0.3)
    assert np.allclose(prox_tv_2d(c, 0.7, 5), c, atol=1e-7)
    rng = np.random.default_rng(1)
    v = rng.standard_normal((2, 50, 70)) + 1j * rng.standard_normal((2, 50, 70))
    # tau_l1 above the max modulus -> zero plane
    assert np.count_nonzero(prox_fl(v, 100.0, 0.3, 5)) == 0
    # big planes, deep halos: oracle parity over many tiles, T = 5 and 20
    for T in (5, 20):
        vb = (rng.standard_normal((2, 300, 260)) + 1j * rng.standard_normal((2, 300, 260))) * 0.2
        out = prox_fl(vb, 0.05, 0.1, T)
        ref = O.fused_prox(vb, 0.05, 0.1, T)
        assert np.max(np.abs(out - ref)) < 2e-5, T


@pytest.mark.parametrize("n,nz", [(1024, 512),   # the full C3 volume
                                  (2048, 40)])   # C4 planes (2048-point rows: radix-64 pass), 40 of its 1000
def test_c3_volume_adjointness_and_far_planes(n, nz):
    """At the full C3 volume (1024^2 x 512, device-resident, through the C ABI)
    and on C4-sized planes: <A x, r> = Re<x, A^H r> with A summing every plane
    (SPEC.md:70, :83), and the deepest planes -- up to 15 transfer-recurrence
    re-anchors in -- against the fp64 oracle run on a one-plane geometry at
    that plane's depth."""
    import ctypes
    import torch
    from paper_1904_04884_b200 import VolumeGeometry
    from paper_1904_04884_b200.engine import HoloEngine
    nx = ny = n
    dz, z0 = 10e-6, 5e-3
    eng = HoloEngine(VolumeGeometry(nx, ny, nz, 10e-6, dz, z0, 632e-9))
    dev = torch.device("cuda", eng.device)
    s = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    gen = torch.Generator(device=dev).manual_seed(5)
    x = torch.randn(nz, ny, nx, dtype=torch.complex64, device=dev, generator=gen)
    x *= torch.rand(nz, ny, nx, device=dev, generator=gen) < 0.01
    r = torch.randn(ny, nx, dtype=torch.float32, device=dev, generator=gen)
    ax = torch.empty(ny, nx, dtype=torch.float32, device=dev)
    adj = torch.empty_like(x)
    assert eng.lib.holo_op_forward(eng.h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(ax.data_ptr()), s) == 0
    assert eng.lib.holo_op_adjoint(eng.h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(adj.data_ptr()),
                                   ctypes.c_double(1.0), s) == 0
    torch.cuda.synchronize(dev)
    lhs = float((ax.double() * r.double()).sum())
    rhs = 0.0
    for k in range(0, nz, 64):  # fp64 inner product in plane chunks
        xa, aa = torch.view_as_real(x[k:k + 64]).double(), torch.view_as_real(adj[k:k + 64]).double()
        rhs += float((xa * aa).sum())
    scale = float(ax.double().norm() * r.double().norm())
    assert abs(lhs - rhs) <= 1e-7 * scale, (lhs, rhs, scale)
    rn = r.double().cpu().numpy()
    for k in (nz - 1, nz // 2 + 7):
        og = O.Geometry(nx, ny, 1, 10e-6, dz, z0 + k * dz, 632e-9)
        assert rel_l2(adj[k].cpu().numpy(), O.back_project(rn, og)[0]) < 5e-6, k
    # forward of a volume holding only the deepest plane
    xk = x[nz - 1].clone()
    x.zero_()
    x[nz - 1] = xk
    assert eng.lib.holo_op_forward(eng.h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(ax.data_ptr()), s) == 0
    torch.cuda.synchronize(dev)
    og = O.Geometry(nx, ny, 1, 10e-6, dz, z0 + (nz - 1) * dz, 632e-9)
    ref = O.sensor_forward(xk.cpu().numpy().astype(np.complex128)[None], og)
    assert rel_l2(ax.cpu().numpy().astype(np.float64), ref) < 5e-6
    eng.close()
