"""CPU, world_size 2 (gloo): the z-sharded decomposition the engine uses.

Each rank owns planes [r*nz/N, (r+1)*nz/N) (engine.cu Engine::init), forms its
partial spectrum, and one allreduce(sum) of the spectrum plus one of the fp64
scalars (ip, dx2, |x|_1, TV) gives every rank the unsharded values, so every
rank takes the same backtracking / restart decisions.  Modelled here with the
fp64 oracle per rank and torch.distributed over gloo; compared with the
unsharded oracle on the same input."""
import os
import socket

import numpy as np
import pytest

from conftest import golden, geom_of

pytestmark = pytest.mark.skipif(os.environ.get("HOLO_NO_DIST") == "1", reason="disabled")


def plane_range(nz, rank, n):
    return nz * rank // n, nz * (rank + 1) // n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_fista(rank, world, port, q):
    import math

    import torch
    import torch.distributed as dist

    from oracle import holo_oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = golden("fista_64")
    g = geom_of(d["geom"])
    kb, ke = plane_range(g.nz, rank, world)
    bb = d["b"]
    lam1, lamtv, inner, iters = 0.5, 0.2, 5, 6
    step = 1.0 / (2.0 * g.nz)
    hs_conj = O.transfer_stack(g, kb, ke, conj=True)
    hs = O.transfer_stack(g, kb, ke)

    def allreduce(a):
        t = torch.as_tensor(np.ascontiguousarray(a))
        if t.is_complex():
            t = torch.view_as_real(t).contiguous()
            dist.all_reduce(t)
            return torch.view_as_complex(t).numpy()
        dist.all_reduce(t)
        return t.numpy()

    def spectrum(xl):
        s = np.zeros(g.shape, dtype=np.complex128)
        for i in range(ke - kb):
            s += np.fft.fft2(xl[i]) * hs_conj[i]
        return allreduce(s)

    def residual(spec):
        r = np.fft.ifft2(spec).real - bb
        return r, float(np.sum(r * r))

    x = np.zeros((ke - kb,) + g.shape, dtype=np.complex128)
    x_old = x.copy()
    sx = sxo = np.zeros(g.shape, dtype=np.complex128)
    t = 1.0
    last = float(np.sum(bb * bb))
    hist = []
    for it in range(iters):
        tn = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
        beta = (t - 1.0) / tn
        y = (1 + beta) * x - beta * x_old
        sy = (1 + beta) * sx - beta * sxo  # forward of y by linearity (no extra FFTs)
        r, f_y = residual(sy)
        rs = np.fft.fft2(r)
        grad = 2.0 * np.fft.ifft2(hs * rs[None], axes=(-2, -1))
        new = O.fused_prox(y - step * grad, step * lam1, step * lamtv, inner)
        dxv = new - y
        sc = allreduce(np.array([float(np.sum((grad.conj() * dxv).real)), float(np.sum(np.abs(dxv) ** 2)),
                                 float(np.sum(np.abs(new))),
                                 sum(O.tv_norm(p.real) + O.tv_norm(p.imag) for p in new)]))
        s_new = spectrum(new)
        _, f_new = residual(s_new)
        assert f_new <= f_y + sc[0] + sc[1] / (2 * step) + 1e-9 * abs(f_y)  # accepted, same on all ranks
        obj = f_new + lam1 * sc[2] + lamtv * sc[3]
        assert obj <= last  # no restart in this case (reference: 0 restarts)
        x_old, x, sxo, sx, t = x, new, sx, s_new, tn
        hist.append(obj)
        last = obj
    full = [None] * world
    dist.all_gather_object(full, (kb, ke, x))
    if rank == 0:
        q.put((hist, full))
    dist.destroy_process_group()


def test_sharded_fista_matches_unsharded():
    import torch.multiprocessing as mp

    from oracle import holo_oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_fista, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    hist, parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = golden("fista_64")
    g = geom_of(d["geom"])
    ref = O.fista_solve(d["b"], g, max_iters=6, step_size=1.0 / (2.0 * g.nz))
    x = np.zeros_like(ref.x)
    for kb, ke, xl in parts:
        x[kb:ke] = xl
    assert np.allclose(hist, ref.history, rtol=1e-10)
    assert np.linalg.norm(x - ref.x) <= 1e-10 * np.linalg.norm(ref.x)


def test_plane_ranges_partition():
    for nz in (1, 7, 16, 512, 1000):
        for n in (1, 2, 3, 4, 8):
            rs = [plane_range(nz, r, n) for r in range(n)]
            assert rs[0][0] == 0 and rs[-1][1] == nz
            assert all(rs[i][1] == rs[i + 1][0] for i in range(n - 1))


# ---- peer-memory spectrum reduction (csrc/peer.cu): host-side algorithm ----

def _peer_reduce_model(rank, world, port, q, P, groups, seed):
    """Rank r models holo_peer_*: k_peer_scatter sums its plane groups (fp32,
    group order) and sends element i to owner i // L, slot r; k_peer_gather
    sums the owner's slots in rank order (fp32) and all-gathers.  The exchange
    is all_gather over gloo (what the IPC stores deliver)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_1904_04884_b200 import _native as nat

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = nat.load().holo_peer_slice(P, world)
    rng = np.random.default_rng(seed + rank)
    spart = (rng.standard_normal((groups, P)) + 1j * rng.standard_normal((groups, P))).astype(np.complex64)
    part = spart[0].copy()
    for g in range(1, groups):
        part = (part + spart[g]).astype(np.complex64)
    # scatter: my partial of every owner's slice, padded to world * L
    padded = np.zeros(world * L, np.complex64)
    padded[:P] = part
    mine = [None] * world
    dist.all_gather_object(mine, padded.reshape(world, L))  # row o of rank j = rank j's partial of slice o
    inbox = np.stack([mine[j][rank] for j in range(world)])  # [slot j][L], as k_peer_scatter writes it
    red = inbox[0].copy()
    for j in range(1, world):
        red = (red + inbox[j]).astype(np.complex64)
    slices = [None] * world
    dist.all_gather_object(slices, red)
    result = np.concatenate(slices)[:P]
    q.put((rank, part, result))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,P,groups", [(2, 4096, 3), (3, 1000, 2), (4, 65536, 5)])
def test_peer_reduction_model(world, P, groups):
    """Slice ownership covers every element once, the rank-order fp32 sums are
    deterministic, and every rank ends with the same spectrum = sum over ranks
    of sum over groups."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_reduce_model, args=(r, world, port, q, P, groups, 11)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict((r, (part, res)) for r, part, res in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = [out[r][0] for r in range(world)]
    expect = parts[0].copy()
    for r in range(1, world):
        expect = (expect + parts[r]).astype(np.complex64)
    for r in range(world):
        assert np.array_equal(out[r][1], expect)  # bitwise: rank-order fp32 sums


def test_peer_slices_cover_the_plane():
    from paper_1904_04884_b200 import _native as nat
    lib = nat.load()
    for P in (64, 1000, 65536, 1 << 20, 1 << 22):
        for n in range(1, 9):
            L = lib.holo_peer_slice(P, n)
            assert L % 64 == 0 and n * L >= P and (n * L - P) < 64 * n + L
            owners = np.minimum(np.arange(P) // L, n - 1)
            assert owners.max() < n and np.all(np.arange(P) // L < n)


# ---- the reconstruct pipeline's frame replicas (pipeline.run_reconstruct) ----
# Each rank takes frames rank::world and rank 0 writes the merged particle
# table (no collective on the data path).  The solver is replaced by a
# deterministic CPU stand-in (the product's fista needs a GPU), so this checks
# the product's host logic only: the frame split, the all_gather_object merge
# and the per-rank outputs must reproduce a one-rank run byte for byte.

def _fake_frames(images, settings, frames):
    from types import SimpleNamespace

    from paper_1904_04884_b200.sparsevol import SparseVolume

    geom = settings.geom()
    out = []
    for t in frames:
        img = np.asarray(images[t])
        stack = np.zeros((geom.nz,) + img.shape, np.complex128)
        stack[t % geom.nz] = np.where(np.abs(img - img.mean()) > 2 * img.std(), img, 0.0)
        vol = SparseVolume.from_dense_stack(stack, geom)
        dets = [SimpleNamespace(blob_id=b, x_vox=1.5 * b + t, y_vox=2.0 * b, z_vox=float(t % geom.nz), x=1e-5 * b,
                                y=2e-5 * b, z=3e-3 + 1e-4 * t, volume=3 + b, peak_intensity=0.5 * t + b,
                                axis=None if b % 2 else (0.0, 0.0, 1.0), elongation=None if b % 2 else 1.5)
                for b in range(1, 2 + t % 3)]
        out.append((t, vol, dets, [10.0 - t, 9.0 - t]))
    return out


def _pipeline_rank(rank, world, port, cfg_path, frames_glob, out_dir):
    import torch.distributed as dist

    from paper_1904_04884_b200 import pipeline

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pipeline.reconstruct_frames = _fake_frames
    pipeline.run_reconstruct(pipeline.PipelineSettings.from_yaml(cfg_path), frames_glob, out_dir)
    dist.destroy_process_group()


def test_pipeline_frame_replicas_world2(tmp_path, monkeypatch):
    import torch.multiprocessing as mp

    from paper_1904_04884_b200 import pipeline

    d = golden("pipeline")
    rng = np.random.default_rng(3)
    frames = [d["frames"][t % len(d["frames"])] + rng.standard_normal(d["frames"][0].shape) for t in range(5)]
    for t, img in enumerate(frames):
        pipeline.save_image(tmp_path / f"hologram_{t:04d}.f32", np.asarray(img, np.float64))
    cfg = tmp_path / "cfg.yaml"
    cfg.write_text(str(d["config"]))
    pattern = str(tmp_path / "hologram_*.f32")
    # one rank, in process
    for k in ("RANK", "WORLD_SIZE"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setattr(pipeline, "reconstruct_frames", _fake_frames)
    one = tmp_path / "one"
    assert pipeline.run_reconstruct(pipeline.PipelineSettings.from_yaml(cfg), pattern, str(one)) == 5
    # two ranks over gloo
    two = tmp_path / "two"
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_pipeline_rank, args=(r, 2, port, str(cfg), pattern, str(two))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    names = sorted(os.listdir(one))
    assert names == sorted(os.listdir(two))
    assert "particles.tsv" in names and sum(n.startswith("volume_") for n in names) == 5
    for n in names:
        assert (one / n).read_bytes() == (two / n).read_bytes(), n
