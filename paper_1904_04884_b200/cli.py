"""Command line for the B200 path: ``synthesize`` (GPU render) and ``reconstruct``
(batch fista + segmentation), file formats of the reference CLI (cli.py).

    python -m paper_1904_04884_b200.cli synthesize --config cfg.yaml --output out
    python -m paper_1904_04884_b200.cli reconstruct --config cfg.yaml --output out
    torchrun --nproc-per-node 8 -m paper_1904_04884_b200.cli reconstruct ...   # frames across GPUs
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np


def cmd_synthesize(args) -> int:
    from .pipeline import PipelineSettings, save_image, write_table
    from .synth import add_noise, generate_scene, render_hologram
    import yaml
    st = PipelineSettings.from_yaml(args.config) if args.config else PipelineSettings()
    raw = {}
    if args.config:
        with open(args.config) as f:
            raw = (yaml.safe_load(f) or {}).get("synthesis", {}) or {}
    n = int(raw.get("particles", 50))
    d = float(raw.get("diameter", 20e-6))
    frames = int(raw.get("frames", 1))
    sigma = float(raw.get("noise_sigma", 0.0))
    margin = int(raw.get("margin_planes", 0))
    seed = args.seed if args.seed is not None else 0
    out = args.output or st.paths.get("output", "out")
    os.makedirs(out, exist_ok=True)
    g = st.geom()
    truth = []
    for t in range(frames):
        sc = generate_scene(n, g, d, seed=seed + t, margin_planes=margin)
        img = add_noise(render_hologram(sc), sigma, seed=seed + 1000 + t)
        save_image(os.path.join(out, f"hologram_{t:04d}.f32"), img)
        truth += [(t, i, p.x, p.y, p.z, np.nan, np.nan, np.nan) for i, p in enumerate(sc.particles)]
    write_table(os.path.join(out, "truth.tsv"), ["frame", "particle", "x", "y", "z", "px", "py", "pz"], truth)
    print(f"synthesized {frames} frame(s) into {out}")
    return 0


def cmd_reconstruct(args) -> int:
    from .pipeline import PipelineSettings, run_reconstruct
    st = PipelineSettings.from_yaml(args.config) if args.config else PipelineSettings()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("gloo")
    try:
        n = run_reconstruct(st, args.input, args.output)
    except (OSError, ValueError) as exc:
        print(f"reconstruct failed: {exc}", file=sys.stderr)
        return 1
    print(f"reconstructed {n} frame(s)")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1904_04884_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("synthesize", "reconstruct"):
        p = sub.add_parser(name)
        p.add_argument("--config")
        p.add_argument("--output")
        p.add_argument("--seed", type=int)
        if name == "reconstruct":
            p.add_argument("--input", help="glob of input frames (default: <output>/hologram_*.f32)")
    a = ap.parse_args(argv)
    return {"synthesize": cmd_synthesize, "reconstruct": cmd_reconstruct}[a.cmd](a)


if __name__ == "__main__":
    raise SystemExit(main())
