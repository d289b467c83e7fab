"""Generate the golden vectors in tests/golden/ from the REFERENCE package.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-c1]

Every fixture stores the exact inputs handed to the reference and the outputs
the reference produced.  tests/test_oracle.py pins oracle/holo_oracle.py to
these, and the GPU parity tests compare the CUDA path against them.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from holotrack import optics, prox, segment, solver, sparsevol, synth  # noqa: E402
from holotrack.optics import ComplexField2D, VolumeGeometry  # noqa: E402
from holotrack.prox import RegularizerWeights  # noqa: E402

PITCH, DZ, Z0, LAM = 10e-6, 10e-6, 5e-3, 632e-9


def geom_arr(g):
    return np.array([g.nx, g.ny, g.nz, g.pitch, g.dz, g.z0, g.wavelength], dtype=np.float64)


def coo(vol):
    ks, rs, cs, vals = [], [], [], []
    for k, p in enumerate(vol.planes):
        ks.append(np.full(p.nnz, k, dtype=np.int32))
        rs.append(p.rows)
        cs.append(p.cols)
        vals.append(p.values)
    return (np.concatenate(ks), np.concatenate(rs).astype(np.int32), np.concatenate(cs).astype(np.int32),
            np.concatenate(vals).astype(np.complex128))


def save(name, **arrs):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def hologram(g, n, diameter, seed, noise=0.02, margin=2):
    scene = synth.generate_scene(n, g, diameter, seed=seed, margin_planes=margin)
    img = synth.add_noise(synth.render_hologram(scene), noise, seed=seed + 7)
    from holotrack.preprocess import invert_residual
    return invert_residual(img), scene.positions()


def op_fixture(name, g, seed):
    rng = np.random.default_rng(seed)
    shp = (g.nz, g.ny, g.nx)
    dense = (rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) * (rng.random(shp) < 0.05)
    vol = sparsevol.SparseVolume.from_dense_stack(dense, g)
    r = rng.standard_normal(g.plane_shape)
    eng = solver._ComplexEngine(g, "float64")
    fwd = eng.forward_sparse(vol.planes, 4)
    fwd_opt = optics.forward(vol, g).values.real
    adj = optics.adjoint(ComplexField2D(r, g.pitch, g.wavelength), g)
    grad = np.concatenate([gc for _, _, gc in eng.gradient_chunks(r, 4)])
    ladder = optics.TransferLadder(g)
    save(name, geom=geom_arr(g), x=dense, r=r, forward=fwd, forward_optics=fwd_opt, adjoint=adj,
         gradient=grad, transfer=ladder.stack(0, g.nz), transfer_conj=ladder.stack(0, g.nz, conj=True),
         sigma2=np.array(solver.estimate_operator_norm(g)))


def prox_fixture():
    rng = np.random.default_rng(5)
    v = (rng.standard_normal((3, 40, 24)) + 1j * rng.standard_normal((3, 40, 24))) * 0.3
    v[1] = np.round(v[1] * 2) / 2  # piecewise-constant plane
    real = rng.standard_normal((2, 17, 33))
    cases = {}
    for T in (1, 5, 20):
        for tl, tt in ((0.1, 0.3), (0.0, 0.3), (0.2, 0.0), (0.05, 2.0)):
            cases[f"fl_T{T}_{tl}_{tt}"] = prox.prox_fl(v, tl, tt, T)
    tv_real = {f"tv_real_T{T}": prox.prox_tv_2d(real, 0.4, T) for T in (1, 5)}
    tvn = np.array([prox.tv_norm_2d(v[i].real) for i in range(3)] + [prox.tv_norm_2d(v[i].imag) for i in range(3)])
    l1 = prox.prox_l1(v, 0.25)
    # guard: FGP output worse than its input.  It only fires on thin planes
    # (found by search); plane 0 real part fires at tau=0.34, T=1.
    gv = np.array([[[2.0, 1.0, -1.0, -1.0]], [[0.5, -1.0, 2.0, 0.0]], [[1.0, 1.0, 0.0, -2.0]]])
    gv = gv + 1j * np.array([[[0.0, 1.0, 0.5, 2.0]], [[2.0, 1.0, -1.0, -1.0]], [[0.25, 0.0, 0.0, 1.0]]])
    fired = np.array([[np.array_equal(prox.prox_tv_2d(part[i], 0.34, 1), part[i]) for i in range(3)]
                      for part in (gv.real, gv.imag)])
    print("guard fired (re/im x plane):", fired.tolist())
    extra = dict(guard_v=gv, guard_out=prox.prox_fl(gv, 0.05, 0.34, 1), guard_fired=fired)
    save("prox", v=v, real=real, tv_norm=tvn, l1_025=l1, **cases, **tv_real, **extra)


def fista_fixture(name, g, b, truth=None, lam=(0.5, 0.2), iters=20, inner=5, policy="backtracking",
                  step=None, stop_tol=0.0, detect=True, real=False):
    cfg = solver.SolverConfig(weights=RegularizerWeights(*lam), max_iters=iters, tv_inner_iters=inner,
                              step_policy=policy, step_size=step, stop_tol=stop_tol, real_nonnegative=real)
    t0 = time.time()
    diverged = False
    try:
        vol, rep = solver.fista(ComplexField2D(b, g.pitch, g.wavelength), g, cfg)
    except solver.DivergenceError as e:
        diverged = True
        rep = e.report
        vol = sparsevol.SparseVolume.zeros(g)
    dt = time.time() - t0
    k, r, c, v = coo(vol)
    extra = {}
    if detect and not diverged:
        dets = segment.extract_particles(vol, 2 / 256, 5)
        extra["detections"] = np.array([[d.x_vox, d.y_vox, d.z_vox, d.volume] for d in dets]).reshape(-1, 4)
    if truth is not None:
        extra["truth"] = truth
    save(name, geom=geom_arr(g), b=b, lam=np.array(lam), iters=np.array(iters), inner=np.array(inner),
         policy=np.array(policy), step_in=np.array(-1.0 if step is None else step), stop_tol=np.array(stop_tol),
         k=k, r=r, c=c, v=v, history=np.array(rep.objective), iterations=np.array(rep.iterations),
         step=np.array(rep.step_size), restarts=np.array(rep.restarts), diverged=np.array(diverged),
         final_sparsity=np.array(rep.final_sparsity), ref_seconds=np.array(dt), real=np.array(real), **extra)
    print(f"  {name}: {dt:.1f}s  iters={rep.iterations} restarts={rep.restarts} nnz={vol.nnz} "
          f"div={diverged} dets={len(extra.get('detections', []))}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c1", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    only = set(a.only.split(",")) if a.only else None

    def want(n):
        return only is None or n in only

    if want("ops"):
        op_fixture("ops_a", VolumeGeometry(64, 32, 6, PITCH, DZ, Z0, LAM), 1)
        op_fixture("ops_evan", VolumeGeometry(32, 32, 4, 0.45e-6, 1e-6, 20e-6, LAM), 2)
    if want("prox"):
        prox_fixture()
    g64 = VolumeGeometry(64, 64, 16, PITCH, DZ, Z0, LAM)
    if want("small"):
        b64, t64 = hologram(g64, 8, 20e-6, 11)
        fista_fixture("fista_64", g64, b64, t64, iters=20)
        fista_fixture("fista_64_tvheavy", g64, b64, lam=(0.05, 0.5), iters=12, inner=20)
        fista_fixture("fista_64_stall", g64, b64, lam=(0.05, 2.0), iters=12, inner=20)
        fista_fixture("fista_64_backtrack", g64, b64, iters=10, step=4.0 / (2 * 16))
        fista_fixture("fista_64_fixed_stop", g64, b64, iters=40, policy="fixed", step=1.0 / 32, stop_tol=2e-3)
        fista_fixture("fista_64_diverge", g64, b64, lam=(0.0, 0.0), iters=30, policy="fixed", step=100.0)
        fista_fixture("fista_64_zero", g64, np.zeros((64, 64)), iters=5)
        g128 = VolumeGeometry(128, 128, 32, PITCH, DZ, Z0, LAM)
        b128, t128 = hologram(g128, 20, 20e-6, 12)
        fista_fixture("fista_128", g128, b128, t128, iters=30)
    if want("real"):
        b64, t64 = hologram(g64, 8, 20e-6, 11)
        fista_fixture("fista_64_real", g64, b64, iters=15, real=True)
        fista_fixture("fista_64_real_tv", g64, b64, lam=(0.05, 0.5), iters=10, inner=20, real=True)
        g128 = VolumeGeometry(128, 128, 32, PITCH, DZ, Z0, LAM)
        b128, t128 = hologram(g128, 20, 20e-6, 12)
        fista_fixture("fista_128_real", g128, b128, t128, iters=20, real=True)
        gr = VolumeGeometry(64, 32, 6, PITCH, DZ, Z0, LAM)
        rng = np.random.default_rng(4)
        shp = (gr.nz, gr.ny, gr.nx)
        dense = rng.standard_normal(shp) * (rng.random(shp) < 0.05)
        vol = sparsevol.SparseVolume.from_dense_stack(dense, gr)
        r = rng.standard_normal(gr.plane_shape)
        eng = solver._RealEngine(gr, "float64")
        save("ops_real", geom=geom_arr(gr), x=dense, r=r, forward=eng.forward_sparse(vol.planes, 4),
             gradient=np.concatenate([gc for _, _, gc in eng.gradient_chunks(r, 4)]),
             sigma2=np.array(solver.estimate_operator_norm(gr, real=True)),
             sigma2_g64=np.array(solver.estimate_operator_norm(g64, real=True)))
    if want("render"):
        # input side: nonlinear renders (disks, rods, a sub-pixel particle) and background removal
        g = VolumeGeometry(64, 32, 16, PITCH, DZ, Z0, LAM)
        sc = synth.generate_scene(12, g, 20e-6, seed=21, margin_planes=2)
        img_disk = synth.render_hologram(sc)
        rng = np.random.default_rng(22)
        rods = []
        for _ in range(5):
            o = rng.standard_normal(3)
            o /= np.linalg.norm(o)
            rods.append(synth.Particle(x=rng.uniform(0, g.nx * g.pitch), y=rng.uniform(0, g.ny * g.pitch),
                                       z=rng.uniform(g.z0, g.z0 + g.nz * g.dz), diameter=20e-6,
                                       orientation=o, length=200e-6, opacity=0.8))
        rods.append(synth.Particle(x=101e-6, y=203e-6, z=g.z0 + 3e-5, diameter=5e-6))
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            img_rod = synth.render_hologram(synth.Scene(rods, g))
        rod_arr = np.array([[p.x, p.y, p.z, p.diameter, p.opacity,
                             *(p.orientation if p.orientation is not None else [np.nan] * 3),
                             p.length if p.length is not None else np.nan] for p in rods])
        stack = rng.random((9, 8, 10)) + 0.5
        from holotrack.preprocess import preprocess_background
        save("render", geom=geom_arr(g), scene=sc.positions(), img_disk=img_disk, rods=rod_arr, img_rod=img_rod,
             noisy=synth.add_noise(img_disk, 0.02, seed=5), stack=stack, background=preprocess_background(stack, 5))
    if want("pipeline"):
        # the reference CLI end to end: 2 frames, invert residuals, step once, fista, segment, tables
        import tempfile
        from holotrack import cli as hcli
        import yaml
        g = VolumeGeometry(64, 64, 16, PITCH, DZ, Z0, LAM)
        cfgd = {"geometry": dict(nx=64, ny=64, nz=16, pitch=PITCH, dz=DZ, z0=Z0, wavelength=LAM),
                "solver": dict(max_iters=15), "segmentation": dict(min_vox=2, with_orientation=True),
                "preprocessing": dict(mode="invert")}
        with tempfile.TemporaryDirectory() as td:
            frames = []
            for t in range(2):
                sc = synth.generate_scene(6, g, 20e-6, seed=30 + t, margin_planes=2)
                img = synth.add_noise(synth.render_hologram(sc), 0.02, seed=40 + t)
                frames.append(img.astype("<f4"))
                from holotrack import io as hio
                hio.save_image(os.path.join(td, f"hologram_{t:04d}.f32"), img)
            cpath = os.path.join(td, "cfg.yaml")
            cfgd["paths"] = dict(output=td)
            with open(cpath, "w") as f:
                yaml.safe_dump(cfgd, f)
            assert hcli.main(["reconstruct", "--config", cpath]) == 0
            parts = open(os.path.join(td, "particles.tsv")).read()
            objs = [open(os.path.join(td, f"objective_{t:04d}.tsv")).read() for t in range(2)]
            vols = [np.frombuffer(open(os.path.join(td, f"volume_{t:04d}.rihv"), "rb").read(), np.uint8)
                    for t in range(2)]
        save("pipeline", frames=np.stack(frames), config=np.array(yaml.safe_dump(cfgd)), particles=np.array(parts),
             objective0=np.array(objs[0]), objective1=np.array(objs[1]), rihv0=vols[0], rihv1=vols[1])
    if want("segment"):
        # output side: RIHV container bytes and detections with orientation
        d = np.load(os.path.join(HERE, "fista_128.npz"))
        g = VolumeGeometry(*[int(x) for x in d["geom"][:3]], *d["geom"][3:])
        dense = np.zeros((g.nz, g.ny, g.nx), dtype=np.complex128)
        dense[d["k"], d["r"], d["c"]] = d["v"]
        vol = sparsevol.SparseVolume.from_dense_stack(dense, g)
        dets = segment.extract_particles(vol, 2 / 256, 2, with_orientation=True)
        rows = []
        for det in dets:
            ax = det.axis if det.axis is not None else np.full(3, np.nan)
            el = det.elongation if det.elongation is not None else np.nan
            rows.append([det.blob_id, det.x_vox, det.y_vox, det.z_vox, det.x, det.y, det.z, det.volume,
                         det.peak_intensity, *ax, el])
        path = os.path.join("/tmp", "golden_128.rihv")
        sparsevol.save_volume(path, vol)
        blob = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        save("segment", dets=np.array(rows), rihv=blob, rel_tol=np.array(2 / 256), min_vox=np.array(2))
    if want("c1") and not a.skip_c1:
        gc1 = VolumeGeometry(256, 256, 64, PITCH, DZ, Z0, LAM)
        bc1, tc1 = hologram(gc1, 50, 20e-6, 0)
        fista_fixture("fista_c1", gc1, bc1, tc1, iters=50)


if __name__ == "__main__":
    main()
