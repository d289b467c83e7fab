"""Input side: scenes, noise (CPU, same draws as the reference)
and the GPU render / background removal against the reference's outputs."""
import numpy as np
import pytest

from conftest import golden


def _geom(d):
    from paper_1904_04884_b200 import VolumeGeometry
    nx, ny, nz, pitch, dz, z0, lam = d["geom"]
    return VolumeGeometry(int(nx), int(ny), int(nz), pitch, dz, z0, lam)


def test_scene_and_noise_match_reference():
    from paper_1904_04884_b200 import synth
    d = golden("render")
    g = _geom(d)
    sc = synth.generate_scene(12, g, 20e-6, seed=21, margin_planes=2)
    assert np.array_equal(sc.positions(), d["scene"])
    assert np.array_equal(synth.add_noise(d["img_disk"], 0.02, seed=5), d["noisy"])
    assert synth.shadow_density(1.8e12, 1e-3, 10e-6) == pytest.approx(0.18, abs=1e-15)  # SPEC acceptance 6


def test_masks_match_reference_definition():
    from paper_1904_04884_b200 import synth
    d = golden("render")
    g = _geom(d)
    for p in synth.generate_scene(12, g, 20e-6, seed=21, margin_planes=2).particles:
        r, c, a = synth.particle_mask(p, g)
        xs = (np.arange(g.nx) * g.pitch - p.x)[None, :]
        ys = (np.arange(g.ny) * g.pitch - p.y)[:, None]
        full = ((xs ** 2 + ys ** 2) <= (p.diameter / 2) ** 2)
        got = np.zeros_like(full)
        got[r, c] = True
        assert np.array_equal(got, full)


@pytest.mark.gpu
def test_gpu_render_matches_reference():
    from paper_1904_04884_b200 import synth
    d = golden("render")
    g = _geom(d)
    sc = synth.generate_scene(12, g, 20e-6, seed=21, margin_planes=2)
    img = synth.render_hologram(sc)
    assert np.max(np.abs(img - d["img_disk"])) < 2e-6
    rods = []
    for row in d["rods"]:
        o = None if np.isnan(row[5]) else row[5:8]
        ln = None if np.isnan(row[8]) else row[8]
        rods.append(synth.Particle(x=row[0], y=row[1], z=row[2], diameter=row[3], opacity=row[4],
                                   orientation=o, length=ln))
    with pytest.warns(UserWarning):
        img2 = synth.render_hologram(synth.Scene(rods, g))
    assert np.max(np.abs(img2 - d["img_rod"])) < 2e-6


@pytest.mark.gpu
def test_gpu_background_matches_reference():
    from paper_1904_04884_b200 import synth
    d = golden("render")
    out = synth.preprocess_background(d["stack"], 5)
    assert np.max(np.abs(out - d["background"])) < 1e-12
