"""The batch reconstruct caller against the reference CLI's own
output on the same two frames (tests/golden/pipeline.npz)."""
import os

import numpy as np
import pytest

from conftest import golden


def _table(text):
    lines = [ln for ln in str(text).splitlines() if ln.strip()]
    return lines[0].split("\t"), np.array([[float(x) for x in ln.split("\t")] for ln in lines[1:]])


def _write_frames(tmp_path, d):
    from paper_1904_04884_b200.pipeline import save_image
    for t, img in enumerate(d["frames"]):
        save_image(tmp_path / f"hologram_{t:04d}.f32", img.astype(np.float64))
    cfg = tmp_path / "cfg.yaml"
    cfg.write_text(str(d["config"]))
    return cfg


def test_io_and_settings(tmp_path):
    from paper_1904_04884_b200.pipeline import PipelineSettings, load_image
    d = golden("pipeline")
    cfg = _write_frames(tmp_path, d)
    assert np.array_equal(load_image(tmp_path / "hologram_0001.f32"), d["frames"][1].astype(np.float64))
    st = PipelineSettings.from_yaml(cfg)
    assert st.geom().plane_shape == (64, 64) and st.solver_config().max_iters == 15
    assert st.segmentation["min_vox"] == 2 and st.segmentation["with_orientation"] is True


@pytest.mark.gpu
def test_reconstruct_cli_matches_reference(tmp_path):
    from paper_1904_04884_b200.cli import main
    d = golden("pipeline")
    cfg = _write_frames(tmp_path, d)
    assert main(["reconstruct", "--config", str(cfg), "--output", str(tmp_path)]) == 0
    hdr, got = _table((tmp_path / "particles.tsv").read_text())
    rhdr, ref = _table(d["particles"])
    assert hdr == rhdr and got.shape == ref.shape
    assert np.array_equal(got[:, [0, 1, 8]], ref[:, [0, 1, 8]])  # frame, blob, volume
    assert np.max(np.abs(got[:, 2:5] - ref[:, 2:5])) < 0.05    # centroids (voxels)
    for t in range(2):
        _, o = _table((tmp_path / f"objective_{t:04d}.tsv").read_text())
        _, r = _table(d[f"objective{t}"])
        assert np.allclose(o, r, rtol=2e-5)
        assert os.path.getsize(tmp_path / f"volume_{t:04d}.rihv") > 0
