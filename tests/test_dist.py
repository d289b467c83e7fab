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
