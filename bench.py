"""Benchmark: voxel-iterations/s of the fused-lasso FISTA reconstruction
(BASELINE.json metric) on the 1024x1024x512 high-concentration field (C3).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c3]

One step = one complete fista() solve of the config (100 FISTA iterations on
a synthetic hologram whose inputs are already resident in HBM).  N>1 runs are
launched by torchrun (`--gpus N` without torchrun relaunches itself under
it); the volume is z-sharded over the ranks (weak scaling would fix
planes/GPU; here the C3 volume is fixed, so scaling is "strong").
The reference arm (--impl reference) times the reference's own CPU solver
(holotrack from baseline/_ref; the oracle port if that install is absent)
on every host core, on a bounded sample of the same workload and hologram.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PITCH, DZ, Z0, LAM = 10e-6, 10e-6, 5e-3, 632e-9
CONFIGS = {
    # name: (nx, ny, nz, iters, shadow density, seed, lam_l1, lam_tv, inner, diameter)
    "c1": (256, 256, 64, 50, None, 0, 0.5, 0.2, 5, 20e-6),
    "c2": (1024, 1024, 256, 100, 0.05, 1, 0.5, 0.2, 5, 20e-6),
    "c3": (1024, 1024, 512, 100, 0.2, 2, 0.5, 0.2, 5, 20e-6),
    "c4": (2048, 2048, 1000, 100, 0.05, 3, 0.5, 0.2, 5, 20e-6),  # 134 GB of state on one B200 (8 GPUs in BASELINE)
    "c5": (1024, 1024, 512, 100, 0.05, 4, 0.05, 1.0, 20, 20e-6),  # rods (microfibers), length 10 d
    # a 1280x1024 camera frame (not a BASELINE config): C3's volume depth and weights,
    # mixed-radix rows (csrc/gfft.cu) with the fused column passes
    "cam": (1280, 1024, 512, 100, 0.2, 5, 0.5, 0.2, 5, 20e-6),
}
METRIC = "voxel-iterations/sec (1024²×512 fused-lasso FISTA) at 1/2/4/8 B200; % HBM roofline"
BYTES_PER_VOXEL_ITER = 72  # SURVEY.md 8(d) algorithmic bytes per voxel-iteration
# algorithmic HBM bytes per local voxel for one launch of each kernel class
KERNEL_BYTES = {"prox": 32, "adj_cols": 8, "adj_rows": 16, "fwd_rows": 16, "fwd_cols": 8}


def n_particles(cfg):
    nx, _, _, _, sd, _, _, _, inner, d = cfg
    if sd is None:
        return 50
    ny = cfg[1]
    area = d ** 2 if cfg is not CONFIGS.get("c5") else 7.9 * d ** 2  # mean projected rod area ~ pi/4 * 10 d^2
    return int(round(sd * nx * ny * PITCH ** 2 / area))


def make_hologram(cfg, device=None):
    """Synthetic C-config hologram: seeded scene, GPU render (holo_render_spectrum +
    library FFT, fp64 accumulation), noise sigma 0.02, b = 1 - I/mean(I)
    (synth.py:74-191, preprocess.py:41-53).  Input generation, not timed."""
    from paper_1904_04884_b200 import VolumeGeometry
    from paper_1904_04884_b200.synth import add_noise, generate_scene, invert_residual, render_hologram
    nx, ny, nz, _, _, seed, *_rest = cfg
    g = VolumeGeometry(nx, ny, nz, PITCH, DZ, Z0, LAM)
    sc = generate_scene(n_particles(cfg), g, cfg[9], seed=seed, margin_planes=2)
    if cfg is CONFIGS["c5"]:  # microfibers: random unit orientation, length 10 d
        rng = np.random.default_rng(seed + 100)
        for p in sc.particles:
            o = rng.standard_normal(3)
            p.orientation, p.length = o / np.linalg.norm(o), 10 * cfg[9]
    return invert_residual(add_noise(render_hologram(sc), 0.02, seed=seed + 7))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_traffic(kernel, voxels):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, scaled from
    the committed ncu --set full capture of one launch (profiles/r02_traffic.json,
    else r01; written by tools/ncu_traffic.py); None if that kernel was not captured."""
    for name in ("r02_traffic.json", "r01_traffic.json"):  # latest capture first
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                rec = json.load(f).get(kernel)
        except (OSError, ValueError):
            continue
        if rec is not None:
            return rec["dram_bytes_per_voxel"] * voxels
    return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# ------------------------------------------------------------- CPU arms ----
#
# The CPU legs time the reference itself when the driver's offline install of
# the unmodified package is present (baseline/_ref/holotrack, the
# `pip install --no-deps --target baseline/_ref /root/reference/pkg` of
# DESIGN.md section 6), else the oracle port (pinned to the reference by
# tests/test_oracle.py).  Sample: the config's full lateral size, the
# first REF_PLANES planes, REF_ITERS iterations from x = 0 (the second is a
# steady-state iteration: momentum on, y != 0, every plane forward-projected),
# initial step 1/(2 nz) so the infeasible power iteration is skipped; the
# per-voxel cost is independent of nz.

REF_PLANES, REF_ITERS = 4, 2


def reference_module():
    """holotrack.solver from baseline/_ref (driver install), or None."""
    for base in (os.path.join(ROOT, "baseline", "_ref"), os.path.join(ROOT, "baseline", "_ref", "pkg", "src")):
        if os.path.isfile(os.path.join(base, "holotrack", "solver.py")):
            if base not in sys.path:
                sys.path.insert(0, base)
            import holotrack.solver as hs
            return hs
    return None


def _cpu_sample(args):
    """One bounded CPU solve of the sample; returns (voxel-iterations, seconds,
    dense volume or None, history)."""
    b, nx, ny, nzs, iters, lam_l1, lam_tv, inner, want_x = args
    hs = reference_module()
    step = 1.0 / (2.0 * nzs)
    if hs is not None:  # the unmodified reference, through its public API
        from holotrack.optics import ComplexField2D, VolumeGeometry
        from holotrack.prox import RegularizerWeights
        g = VolumeGeometry(nx, ny, nzs, PITCH, DZ, Z0, LAM)
        cfg = hs.SolverConfig(weights=RegularizerWeights(lam_l1, lam_tv), max_iters=iters, tv_inner_iters=inner,
                              step_size=step)
        t0 = time.perf_counter()
        vol, rep = hs.fista(ComplexField2D(b, PITCH, LAM), g, cfg)
        dt = time.perf_counter() - t0
        return nx * ny * nzs * rep.iterations, dt, (vol.to_dense() if want_x else None), list(rep.objective)
    from oracle.holo_oracle import Geometry, fista_solve
    g = Geometry(nx, ny, nzs, PITCH, DZ, Z0, LAM)
    t0 = time.perf_counter()
    res = fista_solve(b, g, lam_l1=lam_l1, lam_tv=lam_tv, max_iters=iters, inner=inner, step_size=step)
    dt = time.perf_counter() - t0
    return nx * ny * nzs * res.iterations, dt, (res.x if want_x else None), list(res.history)


def cpu_kind():
    return "reference" if reference_module() is not None else "port"


def cpu_sample_spec(cfg, planes=REF_PLANES, iters=REF_ITERS):
    nx, ny, nz, _, _, _, l1, tv, inner, _ = cfg
    who = "holotrack.solver.fista (baseline/_ref)" if cpu_kind() == "reference" else "oracle port"
    return planes, iters, f"{who}: {nx}x{ny}x{planes} planes x {iters} FISTA iterations from x=0 " \
                          f"(initial step 1/(2*{planes})), the bench hologram, lambda=({l1},{tv}), T={inner}; " \
                          f"per-voxel cost is nz-independent"


def cpu_baseline(cfg, b):
    """1-core CPU leg on rank 0; also returns the sample's volume/history for
    the GPU-vs-CPU parity check."""
    planes, iters, desc = cpu_sample_spec(cfg)
    nx, ny, _, _, _, _, l1, tv, inner, _ = cfg
    vox, dt, x, hist = _cpu_sample((b, nx, ny, planes, iters, l1, tv, inner, True))
    return {"value": vox / dt, "unit": "voxel-iter/s", "cores": 1, "kind": cpu_kind(),
            "sample": desc + f"; {dt:.1f} s on 1 core"}, x, hist


def sample_parity(cfg, b, x_cpu, hist_cpu, dev):
    """The GPU path (public fista()) on the CPU leg's sample: same hologram,
    geometry, step and iterations; volume rel-L2 and history agreement."""
    from paper_1904_04884_b200 import ComplexField2D, RegularizerWeights, SolverConfig, VolumeGeometry, fista
    nx, ny, _, _, _, _, l1, tv, inner, _ = cfg
    planes, iters, _ = cpu_sample_spec(cfg)
    g = VolumeGeometry(nx, ny, planes, PITCH, DZ, Z0, LAM)
    scfg = SolverConfig(weights=RegularizerWeights(l1, tv), max_iters=iters, tv_inner_iters=inner,
                        step_size=1.0 / (2.0 * planes))
    vol, rep = fista(ComplexField2D(b, PITCH, LAM), g, scfg)
    x = vol.to_dense()
    rel = float(np.linalg.norm(x - x_cpu) / max(np.linalg.norm(x_cpu), 1e-300))
    hrel = float(max(abs(a - c) / max(abs(c), 1e-300) for a, c in zip(rep.objective, hist_cpu))) \
        if len(hist_cpu) else 0.0
    return {"rel_l2": rel, "history_max_rel": hrel, "iterations_equal": rep.iterations == len(hist_cpu),
            "against": cpu_kind(), "bar": "rel_l2 <= 1e-4 (north_star)"}


def run_reference(a, cfg_name):
    """--impl reference: the reference's own CPU implementation on every host
    core, one independent solve per core per step (like holotrack's
    `reconstruct --workers`), on the GPU arm's hologram."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    cfg = CONFIGS[cfg_name]
    nx, ny, nz, iters_full, _, seed, l1, tv, inner, d = cfg
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    planes, iters, desc = cpu_sample_spec(cfg)
    # workers are forked before this process touches CUDA (GPU input render below)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        b = reference_hologram(cfg)
        job = (b, nx, ny, planes, iters, l1, tv, inner, False)
        for _ in range(a.warmup):
            pool.map(_cpu_sample, [job] * cores)
        times = []
        for _ in range(a.steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_sample, [job] * cores)
            times.append(time.perf_counter() - t0)
    vox = sum(r[0] for r in res)
    step_s = statistics.mean(times)
    value = vox / step_s
    line = {"metric": METRIC, "value": value, "unit": "voxel-iter/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg_name}: {nx}x{ny}x{nz}, {iters_full} iterations (sampled)",
                       "sample": desc}, "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "voxel-iter/s", "cores": cores, "kind": cpu_kind(),
                             "sample": desc + f"; {cores} concurrent solves (one per core)"},
            "e2e": {"value": value, "unit": "voxel-iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def reference_hologram(cfg):
    """The GPU arm's hologram (make_hologram: same scene, render, noise); on a
    host without a GPU only the small C1 scene can be rendered, by the oracle."""
    try:
        import torch
        gpu = torch.cuda.is_available()
    except ImportError:
        gpu = False
    if gpu:
        return make_hologram(cfg)
    if cfg is not CONFIGS["c1"]:
        raise SystemExit("the reference arm needs a GPU to render this config's hologram")
    from oracle.holo_oracle import Geometry, add_noise, invert_residual, make_scene, render_hologram
    nx, ny, nz, _, _, seed, _, _, _, d = cfg
    g = Geometry(nx, ny, nz, PITCH, DZ, Z0, LAM)
    pts = make_scene(n_particles(cfg), g, d, seed=seed, margin_planes=2)
    return invert_residual(add_noise(render_hologram(pts, g, d), 0.02, seed=seed + 7))


def self_launch(a):
    """`bench.py --gpus N` without torchrun: relaunch under torchrun, one rank
    per GPU (NCCL_DEBUG=INFO so the communicator lines show the N ranks)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------- GPU arm -----

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--iters", type=int, default=0, help="override FISTA iterations (0 = config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()
    # (HOLO_SELF_LAUNCH=1: also for one GPU, e.g. with HOLO_NCCL_SINGLE_RANK=1 to run the
    # torchrun + NCCL plumbing of the sharded engine on a single-GPU box)
    if (a.gpus > 1 or os.environ.get("HOLO_SELF_LAUNCH") == "1") and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(a))
    if a.impl == "reference":
        run_reference(a, a.config)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # HOLO_NCCL_SINGLE_RANK=1 runs the sharded (NCCL) path even with one rank
    sharded = world > 1 or os.environ.get("HOLO_NCCL_SINGLE_RANK") == "1"
    if sharded:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1904_04884_b200 import _native as nat
    from paper_1904_04884_b200 import ComplexField2D, RegularizerWeights, SolverConfig, VolumeGeometry, fista
    from paper_1904_04884_b200.engine import HoloEngine
    from paper_1904_04884_b200.solver import native_config

    cfg = CONFIGS[a.config]
    nx, ny, nz, iters, _, seed, l1, tv, inner, d = cfg
    if a.iters:
        iters = a.iters
    geom = VolumeGeometry(nx, ny, nz, PITCH, DZ, Z0, LAM)
    # identical synthetic hologram on every rank (seeded), generated on the GPU
    b = make_hologram(cfg, dev) if rank == 0 or world == 1 else None
    if sharded:
        bt = torch.as_tensor(b if b is not None else np.zeros((ny, nx)), dtype=torch.float64, device=dev)
        dist.broadcast(bt, 0)
        b = bt.cpu().numpy()
    scfg = SolverConfig(weights=RegularizerWeights(l1, tv), max_iters=iters, tv_inner_iters=inner)
    ncfg = native_config(scfg)
    lib = nat.load()
    if sharded:
        nid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            nat.check(lib.holo_nccl_unique_id(buf))
            nid = torch.tensor(list(buf.raw), dtype=torch.uint8, device=dev)
        dist.broadcast(nid, 0)
        eng = HoloEngine(geom, local, shard=(rank, world, bytes(nid.cpu().tolist())))
        if world > 1 and os.environ.get("HOLO_PEER_ALLREDUCE") == "1":
            # forward plane sum over NVLink peer memory instead of the NCCL allreduce
            def gather(blob):
                out = [None] * world
                dist.all_gather_object(out, blob)
                return out
            eng.enable_peer_reduction(gather)
    else:
        eng = HoloEngine(geom, local)
    b_dev = torch.as_tensor(b, dtype=torch.float64, device=dev).contiguous()
    stream = torch.cuda.current_stream(dev)

    def one_solve():
        code, rep, hist = eng.solve(b_dev, ncfg, stream=stream.cuda_stream)
        return rep

    for _ in range(a.warmup):
        rep = one_solve()

    def read_prof():
        n = ctypes.c_int32()
        names = ctypes.create_string_buffer(32 * 16)
        kms = (ctypes.c_double * 16)()
        kcnt = (ctypes.c_int64 * 16)()
        lib.holo_profile_read(eng.h, ctypes.byref(n), names, kms, kcnt)
        out = {}
        for i in range(n.value):
            nm = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
            out[nm] = {"ms": kms[i], "launches": int(kcnt[i]), "index": i}
        return out

    # per-kernel-class breakdown from one profiled solve outside the timed
    # region (events around every launch cost ~1 % of a solve); inside the
    # timed region only the dominant class is timed live, for the roofline
    lib.holo_profile_classes(eng.h, 0xFFFFFFFF)
    lib.holo_profile_enable(eng.h, 1)
    one_solve()
    prof = read_prof()
    dom = max((k for k in prof if k in KERNEL_BYTES), key=lambda k: prof[k]["ms"])
    lib.holo_profile_classes(eng.h, 1 << prof[dom]["index"])
    lib.holo_profile_enable(eng.h, 1)
    launches0 = lib.holo_launch_count()
    if sharded:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    vox_iters = 0
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            rep = one_solve()
            vox_iters += nx * ny * nz * rep.iterations
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if sharded:
        dist.barrier()
    launches = lib.holo_launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    if sharded:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    timed = read_prof()[dom]  # the dominant class, recorded live during the timed region
    lib.holo_profile_enable(eng.h, 0)
    lib.holo_profile_classes(eng.h, 0xFFFFFFFF)

    value = vox_iters / (ms / 1e3)
    hbm, peak_kind = peaks()
    local_vox = nx * ny * eng.nz_local
    per_launch_s = timed["ms"] / 1e3 / max(timed["launches"], 1)
    achieved = KERNEL_BYTES[dom] * local_vox / per_launch_s / 1e9
    traffic = measured_traffic(dom, local_vox)
    total_kernel_ms = sum(v["ms"] for v in prof.values())
    step_roof = value / world * BYTES_PER_VOXEL_ITER / 1e9

    # end to end with host buffers: N=1 through the public fista() (pinned b in,
    # SparseVolume out); z-sharded through each rank's engine (holo_solve from
    # the host hologram, then the rank's COO export to host), max over ranks
    e2e = None
    if not a.no_e2e and sharded:
        b_host = np.ascontiguousarray(b, dtype=np.float64)
        eng.solve(b_host, ncfg)  # warm the host path
        eng.export_coo()
        e2e_steps = max(1, min(a.steps, 2))
        dist.barrier()
        t0 = time.perf_counter()
        e_vox, d2h = 0, 0
        for _ in range(e2e_steps):
            _, rep_e, _ = eng.solve(b_host, ncfg)
            per, rows, cols, vals = eng.export_coo()
            e_vox += nx * ny * nz * rep_e.iterations
            d2h = rows.nbytes + cols.nbytes + vals.nbytes + per.nbytes + 8 * rep_e.iterations
        e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(e_s, op=dist.ReduceOp.MAX)
        d2h_t = torch.tensor([float(d2h)], dtype=torch.float64, device=dev)
        dist.all_reduce(d2h_t)
        e2e = {"value": e_vox / float(e_s.item()), "unit": "voxel-iter/s",
               "h2d_bytes_per_step": 8 * nx * ny * world, "d2h_bytes_per_step": int(d2h_t.item()),
               "steps": e2e_steps, "path": "per-rank holo_solve (host b) + holo_export_coo_host"}
    if not a.no_e2e and world == 1 and not sharded:
        eng.close()  # the public path builds its own engine (C4: 134 GB each)
        pinned = torch.empty((ny, nx), dtype=torch.float64, pin_memory=True)
        pinned.copy_(torch.as_tensor(b))
        field = ComplexField2D.__new__(ComplexField2D)  # wrap the pinned buffer without a copy
        field.values, field.pitch, field.wavelength = pinned.numpy(), PITCH, LAM
        e2e_steps = max(1, min(a.steps, 2))
        fista(field, geom, scfg)  # warm the public path
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        e_vox, nnz = 0, 0
        for _ in range(e2e_steps):
            vol, rep_e = fista(field, geom, scfg)
            e_vox += nx * ny * nz * rep_e.iterations
            nnz = vol.nnz
        e_s = time.perf_counter() - t0
        e2e = {"value": e_vox / e_s, "unit": "voxel-iter/s", "h2d_bytes_per_step": 8 * nx * ny,
               "d2h_bytes_per_step": 24 * nnz + 8 * nz + 8 * iters, "steps": e2e_steps}

    cpu = parity = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu, x_cpu, hist_cpu = cpu_baseline(cfg, b)
        parity = sample_parity(cfg, b, x_cpu, hist_cpu, dev)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "voxel-iter/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{a.config}: {nx}x{ny}x{nz} fused-lasso FISTA, {iters} iterations, "
                                   f"{n_particles(cfg)} particles d=20um, lambda=({l1},{tv}), T={inner}",
                       "l2": f"inputs larger than L2 (state 3 x {nx * ny * nz * 8 / 1e9:.1f} GB complex64)", "parallelism": f"z-shard x{world}"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
                         "alg_bytes_per_voxel": KERNEL_BYTES[dom]},
            "step_roofline": {"bytes_per_voxel_iter": BYTES_PER_VOXEL_ITER, "achieved": step_roof, "peak": hbm,
                              "frac": step_roof / hbm, "frac_of_spec_8tbs": step_roof / 8000.0,
                              # compulsory floor (x, x_prev read, x_new write) and the
                              # radix-2 flop model F = 10 log2(P) + 48 T + 100 against the spec FP32 peak
                              "floor_bytes_per_voxel_iter": 24,
                              "floor_frac": value / world * 24 / 1e9 / hbm,
                              "flop_per_voxel_iter": 10 * math.log2(nx * ny) + 48 * inner + 100,
                              "fp32_tflops": value / world * (10 * math.log2(nx * ny) + 48 * inner + 100) / 1e12,
                              "fp32_peak_tflops": 74.4,
                              "fp32_frac": value / world * (10 * math.log2(nx * ny) + 48 * inner + 100) / 74.4e12},
            # one profiled solve after the warm-up (per-solve ms by kernel class)
            "kernels_ms": {k: round(v["ms"], 3) for k, v in prof.items()},
            "kernel_share": {k: round(v["ms"] / total_kernel_ms, 4) for k, v in prof.items()} if total_kernel_ms else {},
            "kernels_profiled": "one extra solve before the timed region; only the roofline kernel is timed "
                                "inside it",
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "solve": {"iterations": rep.iterations, "restarts": rep.restarts, "nnz": rep.nnz,
                      "final_sparsity": rep.final_sparsity, "attempts": rep.attempts,
                      "skipped_planes": rep.skipped_planes},
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
