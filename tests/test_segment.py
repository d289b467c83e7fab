"""Output side: RIHV container (CPU) and GPU particle extraction."""
import os

import numpy as np
import pytest

from conftest import dense_from_golden, golden


def _vol(name):
    from paper_1904_04884_b200 import SparseVolume, VolumeGeometry
    d = golden(name)
    nx, ny, nz, pitch, dz, z0, lam = d["geom"]
    g = VolumeGeometry(int(nx), int(ny), int(nz), pitch, dz, z0, lam)
    return SparseVolume.from_dense_stack(dense_from_golden(d), g)


def test_rihv_bytes_match_reference(tmp_path):
    from paper_1904_04884_b200.sparsevol import load_volume, save_volume
    ref = golden("segment")["rihv"].tobytes()
    vol = _vol("fista_128")
    path = tmp_path / "v.rihv"
    save_volume(path, vol)
    assert path.read_bytes() == ref
    back = load_volume(path)
    assert back.nnz == vol.nnz and back.geom == vol.geom
    assert np.allclose(back.to_dense(), vol.to_dense().astype(np.complex64), atol=0)
    (tmp_path / "bad.rihv").write_bytes(b"XXXX" + ref[4:])
    with pytest.raises(ValueError):
        load_volume(tmp_path / "bad.rihv")


@pytest.mark.gpu
@pytest.mark.parametrize("name,min_vox", [("fista_128", 5), ("fista_c1", 5)])
def test_extract_particles_matches_reference(name, min_vox):
    from paper_1904_04884_b200.segment import extract_particles
    d = golden(name)
    dets = extract_particles(_vol(name), 2 / 256, min_vox)
    ref = d["detections"]
    got = np.array([[p.x_vox, p.y_vox, p.z_vox, p.volume] for p in dets]).reshape(-1, 4)
    assert got.shape == ref.shape
    assert np.allclose(got, ref, atol=1e-9)


@pytest.mark.gpu
def test_extract_particles_with_orientation():
    from paper_1904_04884_b200.segment import extract_particles
    ref = golden("segment")["dets"]
    dets = extract_particles(_vol("fista_128"), 2 / 256, 2, with_orientation=True)
    assert len(dets) == len(ref)
    for p, r in zip(dets, ref):
        assert p.blob_id == int(r[0]) and p.volume == int(r[7])
        assert np.allclose([p.x_vox, p.y_vox, p.z_vox, p.x, p.y, p.z, p.peak_intensity], r[[1, 2, 3, 4, 5, 6, 8]],
                           rtol=1e-12, atol=1e-12)
        if np.isnan(r[9]):
            assert p.axis is None
        else:
            assert np.allclose(p.axis, r[9:12], atol=1e-9) and abs(p.elongation - r[12]) < 1e-9 * r[12]
