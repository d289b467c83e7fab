"""CPU: the host-side mirror of the reference API (types, validation, error
behaviour before any device work)."""
import numpy as np
import pytest

from paper_1904_04884_b200 import (ComplexField2D, RegularizerWeights, SolverConfig, SparsePlane, SparseVolume,
                                   VolumeGeometry, fista, from_dense)
from paper_1904_04884_b200.solver import native_config


def test_solver_config_validation_mirrors_reference():
    SolverConfig()
    for bad in (dict(max_iters=0), dict(step_size=-1.0), dict(bt_shrink=1.0), dict(step_policy="x"),
                dict(tv_inner_iters=0), dict(dtype="float16"), dict(dense_plane_budget=0), dict(stop_tol=-1)):
        with pytest.raises(ValueError):
            SolverConfig(**bad)
    with pytest.raises(ValueError):
        RegularizerWeights(-1.0, 0.0)


def test_geometry_and_field_validation():
    with pytest.raises(ValueError):
        VolumeGeometry(0, 4, 4, 1e-5, 1e-5, 0, 6e-7)
    with pytest.raises(ValueError):
        VolumeGeometry(4, 4, 4, 1e-5, 1e-5, -1, 6e-7)
    with pytest.raises(ValueError):
        ComplexField2D(np.array([[np.nan]]), 1e-5, 6e-7)
    g = VolumeGeometry(64, 32, 4, 1e-5, 1e-5, 5e-3, 632e-9)
    assert g.plane_shape == (32, 64) and g.n_voxels == 64 * 32 * 4 and g.plane_z(2) == 5e-3 + 2e-5


def test_native_config_mapping():
    c = native_config(SolverConfig(weights=RegularizerWeights(0.3, 0.1), step_policy="fixed", step_size=0.25))
    assert (c.lambda_l1, c.lambda_tv, c.step_policy, c.step_size) == (0.3, 0.1, 1, 0.25)
    assert native_config(SolverConfig()).step_size == -1.0
    assert native_config(SolverConfig(real_nonnegative=True), 0.25).real_nonnegative == 1
    assert native_config(SolverConfig(real_nonnegative=True), 0.25).step_size == 0.25


def test_fista_shape_mismatch_raises_before_device_work():
    g = VolumeGeometry(64, 64, 4, 1e-5, 1e-5, 5e-3, 632e-9)
    with pytest.raises(ValueError):
        fista(ComplexField2D(np.zeros((32, 64)), 1e-5, 632e-9), g, SolverConfig())


def test_sparse_containers():
    rng = np.random.default_rng(0)
    p = (rng.standard_normal((5, 7)) * (rng.random((5, 7)) < 0.3)).astype(np.complex128)
    sp = from_dense(p)
    sp.validate()
    assert np.array_equal(sp.to_dense(), p)
    g = VolumeGeometry(7, 5, 2, 1e-5, 1e-5, 5e-3, 632e-9)
    vol = SparseVolume.from_coo(g, [sp.nnz, 0], sp.rows, sp.cols, sp.values)
    assert vol.nnz == sp.nnz and vol.planes[1].nnz == 0
    assert np.array_equal(vol.to_dense()[0], p)
    assert isinstance(SparseVolume.zeros(g).planes[0], SparsePlane)


def test_axpy_exact_merge():
    """axpy = alpha x + y with the reference's entry-set semantics (sparsevol.py:146-176):
    (row, col) order, coincident entries summed, exact cancellations dropped."""
    from paper_1904_04884_b200.sparsevol import axpy
    rng = np.random.default_rng(5)
    g = VolumeGeometry(9, 6, 3, 1e-5, 1e-5, 5e-3, 632e-9)
    a = (rng.standard_normal((3, 6, 9)) + 1j * rng.standard_normal((3, 6, 9))) * (rng.random((3, 6, 9)) < 0.3)
    b = (rng.standard_normal((3, 6, 9)) + 1j * rng.standard_normal((3, 6, 9))) * (rng.random((3, 6, 9)) < 0.3)
    b[0, 1, 2] = -(1.5 - 0.5j) * 2.0  # exact cancellation against alpha * a
    a[0, 1, 2] = 2.0
    alpha = 1.5 - 0.5j
    x, y = SparseVolume.from_dense_stack(a, g), SparseVolume.from_dense_stack(b, g)
    z = axpy(alpha, x, y)
    want = alpha * a + b
    assert np.array_equal(z.to_dense(), want)
    for zp, wp in zip(z.planes, want):
        zp.validate()
        assert zp.nnz == int(np.count_nonzero(wp))  # the cancelled entry is gone
    assert axpy(0, x, y).nnz == y.nnz
    with pytest.raises(ValueError):
        axpy(1.0, x, SparseVolume.zeros(VolumeGeometry(9, 6, 4, 1e-5, 1e-5, 5e-3, 632e-9)))
