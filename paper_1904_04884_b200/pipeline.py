"""Batch reconstruction pipeline: the caller of the hot path.

Mirrors ``holotrack reconstruct`` (cli.py:138-190): load frames, form
residuals (preprocess.py), estimate the step once, run ``fista`` per frame,
segment, and write ``volume_XXXX.rihv``, ``objective_XXXX.tsv`` and
``particles.tsv``.  Instead of a process pool per frame (cli.py:166-168), one
device-resident engine is reused for every frame on a GPU; under torchrun
each rank takes frames rank::world (independent replicas, no collective on
the data path) and rank 0 writes the merged particle table.
"""

from __future__ import annotations

import glob
import math
import os
from dataclasses import dataclass, field

import numpy as np

from .optics import ComplexField2D, VolumeGeometry
from .prox import RegularizerWeights
from .segment import extract_particles
from .solver import SolverConfig, estimate_operator_norm, fista
from .sparsevol import save_volume
from .synth import invert_residual, preprocess_background

PARTICLE_COLUMNS = ["frame", "blob", "x_vox", "y_vox", "z_vox", "x", "y", "z",
                    "volume", "peak_intensity", "px", "py", "pz", "elongation"]  # cli.py:27-30


# ---------------------------------------------------------------- io ---------
def load_image(path) -> np.ndarray:
    """Raw little-endian f32 with a '.dims' sidecar ('ny nx'), or PNG/TIFF in [0, 1] (io.py:25-49)."""
    path = os.fspath(path)
    ext = os.path.splitext(path)[1].lower()
    if ext in (".png", ".tif", ".tiff"):
        from PIL import Image
        with Image.open(path) as im:
            arr = np.asarray(im)
        if arr.ndim == 3:
            arr = arr[..., 0]
        if arr.dtype.kind in "iu":
            return arr.astype(np.float64) / float(np.iinfo(arr.dtype).max)
        return arr.astype(np.float64)
    dims = path + ".dims"
    if not os.path.exists(dims):
        raise FileNotFoundError(f"raw image {path} needs a sidecar {dims} with 'ny nx'")
    with open(dims) as f:
        ny, nx = (int(t) for t in f.read().split()[:2])
    data = np.fromfile(path, dtype="<f4")
    if data.size != ny * nx:
        raise ValueError(f"{path}: expected {ny * nx} float32 values, found {data.size}")
    return data.reshape(ny, nx).astype(np.float64)


def save_image(path, image):
    """Raw f32 + '.dims' (io.py:52-63, raw branch)."""
    image = np.asarray(image, dtype=np.float64)
    image.astype("<f4").tofile(path)
    with open(os.fspath(path) + ".dims", "w") as f:
        f.write(f"{image.shape[0]} {image.shape[1]}\n")


def _fmt(v) -> str:
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return f"{float(v):.10g}"
    return str(v)


def write_table(path, columns, rows):
    """Tab-separated table with a header line (io.py:74-79)."""
    with open(path, "w") as f:
        f.write("\t".join(columns) + "\n")
        for row in rows:
            f.write("\t".join(_fmt(v) for v in row) + "\n")


# ------------------------------------------------------------- config --------
@dataclass
class PipelineSettings:
    """The config.py sections the reconstruct path reads (defaults of config.py:35-107)."""

    geometry: dict = field(default_factory=lambda: dict(nx=512, ny=512, nz=700, pitch=10e-6, dz=10e-6, z0=5e-3,
                                                         wavelength=632e-9))
    solver: dict = field(default_factory=dict)
    preprocessing: dict = field(default_factory=lambda: dict(mode="invert", window=151))
    segmentation: dict = field(default_factory=lambda: dict(rel_tol=2 / 256, min_vox=5, with_orientation=False))
    paths: dict = field(default_factory=lambda: dict(input="", output="out"))

    @classmethod
    def from_yaml(cls, path):
        import yaml
        with open(path) as f:
            raw = yaml.safe_load(f) or {}
        s = cls()
        for sec in ("geometry", "solver", "preprocessing", "segmentation", "paths"):
            getattr(s, sec).update(raw.get(sec, {}) or {})
        return s

    def geom(self) -> VolumeGeometry:
        g = self.geometry
        return VolumeGeometry(int(g["nx"]), int(g["ny"]), int(g["nz"]), float(g["pitch"]), float(g["dz"]),
                              float(g["z0"]), float(g["wavelength"]))

    def solver_config(self, step_size=None) -> SolverConfig:
        s = dict(lambda_l1=0.5, lambda_tv=0.2, max_iters=100, tv_inner_iters=5, step_policy="backtracking",
                 step_size=None, bt_shrink=0.5, stop_tol=0.0, real_nonnegative=False, dtype="float64",
                 dense_plane_budget=16)
        s.update({k: v for k, v in self.solver.items() if k in s})
        if self.solver.get("method", "fista") != "fista":
            raise ValueError("only the fista method is on the B200 path")
        return SolverConfig(weights=RegularizerWeights(float(s["lambda_l1"]), float(s["lambda_tv"])),
                            max_iters=int(s["max_iters"]), tv_inner_iters=int(s["tv_inner_iters"]),
                            step_policy=s["step_policy"],
                            step_size=s["step_size"] if s["step_size"] is not None else step_size,
                            bt_shrink=float(s["bt_shrink"]), stop_tol=float(s["stop_tol"]),
                            real_nonnegative=bool(s["real_nonnegative"]), dtype=s["dtype"],
                            dense_plane_budget=int(s["dense_plane_budget"]))


# ----------------------------------------------------------- pipeline -------
def residuals(images, mode="invert", window=151):
    """cli.py:105-117."""
    if mode == "none":
        return [np.asarray(i, dtype=np.float64) for i in images]
    if mode == "invert":
        return [invert_residual(i) for i in images]
    stack = np.stack(images)
    w = min(window, len(images) - (1 - len(images) % 2))
    if w < 3:
        raise ValueError("background preprocessing needs at least 3 frames")
    cleaned = preprocess_background(stack, w)
    return [-cleaned[t] for t in range(len(images))]  # opaque objects give negative residuals


def reconstruct_frames(images, settings: PipelineSettings, frames=None):
    """fista + extract_particles for each frame; returns [(frame, vol, dets, history)]."""
    geom = settings.geom()
    res = residuals(images, settings.preprocessing.get("mode", "invert"),
                    int(settings.preprocessing.get("window", 151)))
    base = settings.solver_config()
    step = base.step_size
    if step is None:  # estimated once for all frames (cli.py:157-162)
        step = 1.0 / (2.0 * estimate_operator_norm(geom, real=base.real_nonnegative, dtype=base.dtype))
    cfg = settings.solver_config(step)
    seg = settings.segmentation
    out = []
    for t in (range(len(images)) if frames is None else frames):
        vol, rep = fista(ComplexField2D(res[t], geom.pitch, geom.wavelength), geom, cfg)
        dets = extract_particles(vol, float(seg.get("rel_tol", 2 / 256)), int(seg.get("min_vox", 5)),
                                 bool(seg.get("with_orientation", False)))
        out.append((t, vol, dets, rep.objective))
    return out


def particle_rows(results):
    rows = []
    for frame, _vol, dets, _hist in results:
        for d in dets:
            ax = d.axis if d.axis is not None else (math.nan,) * 3
            el = d.elongation if d.elongation is not None else math.nan
            rows.append((frame, d.blob_id, d.x_vox, d.y_vox, d.z_vox, d.x, d.y, d.z, d.volume, d.peak_intensity,
                         ax[0], ax[1], ax[2], el))
    return rows


def run_reconstruct(settings: PipelineSettings, input_glob: str | None = None, out_dir: str | None = None) -> int:
    out_dir = out_dir or settings.paths.get("output", "out")
    pattern = input_glob or settings.paths.get("input") or os.path.join(out_dir, "hologram_*.f32")
    files = sorted(glob.glob(pattern))
    if not files:
        raise FileNotFoundError(f"no input holograms match {pattern!r}")
    images = [load_image(p) for p in files]
    geom = settings.geom()
    for p, img in zip(files, images):
        if img.shape != geom.plane_shape:
            raise ValueError(f"{p}: image shape {img.shape} does not match geometry {geom.plane_shape}")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    mine = list(range(rank, len(files), world))
    results = reconstruct_frames(images, settings, mine)
    rows = particle_rows(results)
    if world > 1:
        import torch.distributed as dist
        gathered = [None] * world
        dist.all_gather_object(gathered, rows)
        rows = sorted((r for part in gathered for r in part), key=lambda r: (r[0], r[1]))
    os.makedirs(out_dir, exist_ok=True)
    for frame, vol, _dets, hist in results:
        save_volume(os.path.join(out_dir, f"volume_{frame:04d}.rihv"), vol)
        if hist is not None:
            write_table(os.path.join(out_dir, f"objective_{frame:04d}.tsv"), ["iteration", "objective"],
                        list(enumerate(hist)))
    if rank == 0:
        write_table(os.path.join(out_dir, "particles.tsv"), PARTICLE_COLUMNS, rows)
    return len(files)
