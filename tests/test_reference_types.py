"""The drop-in claim of INTEGRATION.md section 1: holotrack's own objects
(`ComplexField2D`, `VolumeGeometry`, `SolverConfig`, `RegularizerWeights`) go
into this package's `fista()` unchanged, and its outputs go into holotrack's
own consumers (`segment.extract_particles`, `sparsevol.save_volume`).

holotrack is imported from the driver's install of the unmodified reference
(`baseline/_ref`, which travels to the GPU box) or, in the build container,
from the read-only mount; the tests skip when neither exists."""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, dense_from_golden, golden, rel_l2


def _holotrack():
    for base in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isfile(os.path.join(base, "holotrack", "solver.py")):
            if base not in sys.path:
                sys.path.insert(0, base)
            sys.dont_write_bytecode = True  # the mount is read-only
            import holotrack.optics as optics
            import holotrack.prox as prox
            import holotrack.segment as segment
            import holotrack.solver as solver
            import holotrack.sparsevol as sparsevol
            return optics, prox, solver, segment, sparsevol
    pytest.skip("holotrack (the reference package) is not importable here")


def _ref_inputs(d, **cfg):
    optics, prox, solver, _, _ = _holotrack()
    nx, ny, nz, pitch, dz, z0, lam = d["geom"]
    g = optics.VolumeGeometry(int(nx), int(ny), int(nz), float(pitch), float(dz), float(z0), float(lam))
    b = optics.ComplexField2D(d["b"], float(pitch), float(lam))
    c = solver.SolverConfig(weights=prox.RegularizerWeights(*map(float, d["lam"])), max_iters=int(d["iters"]),
                            tv_inner_iters=int(d["inner"]), **cfg)
    return b, g, c


def test_reference_objects_map_to_the_native_config():
    from paper_1904_04884_b200.solver import _check_b, native_config
    d = golden("fista_64")
    b, g, c = _ref_inputs(d, step_policy="fixed", step_size=0.01, stop_tol=1e-6)
    n = native_config(c)
    assert (n.lambda_l1, n.lambda_tv) == tuple(map(float, d["lam"]))
    assert (n.max_iters, n.tv_inner_iters, n.step_policy, n.step_size) == (int(d["iters"]), int(d["inner"]), 1, 0.01)
    assert n.stop_tol == 1e-6 and n.real_nonnegative == 0
    bb = _check_b(b, g)
    assert bb.dtype == np.float64 and bb.shape == (g.ny, g.nx)
    assert np.array_equal(bb, np.real(d["b"]))


def test_reference_objects_shape_mismatch_is_a_value_error():
    from paper_1904_04884_b200 import fista
    optics, _, _, _, _ = _holotrack()
    d = golden("fista_64")
    b, g, c = _ref_inputs(d)
    wrong = optics.VolumeGeometry(g.nx * 2, g.ny, g.nz, g.pitch, g.dz, g.z0, g.wavelength)
    with pytest.raises(ValueError):
        fista(b, wrong, c)


@pytest.mark.gpu
def test_fista_takes_and_feeds_reference_objects(tmp_path):
    """fista() on holotrack's own input objects matches the reference's golden
    output; the returned volume goes through holotrack's extract_particles
    and save_volume."""
    from paper_1904_04884_b200 import fista
    _, _, _, segment, sparsevol = _holotrack()
    d = golden("fista_c1")
    b, g, c = _ref_inputs(d)
    vol, rep = fista(b, g, c)
    assert rep.iterations == int(d["iterations"]) and rep.restarts == int(d["restarts"])
    assert rel_l2(vol.to_dense(), dense_from_golden(d)) <= 1e-4
    dets = segment.extract_particles(vol, 2 / 256, 5)
    assert len(dets) == len(d["detections"]) > 0
    got = np.array([[p.x_vox, p.y_vox, p.z_vox] for p in dets])
    assert np.max(np.abs(got - d["detections"][:, :3])) < 0.5
    path = tmp_path / "vol.rihv"
    sparsevol.save_volume(path, vol)
    back = sparsevol.load_volume(path)
    assert back.nnz == vol.nnz
