"""Python handle around one ``holo_handle`` (one geometry on one GPU, or one
z-shard of it).  PyTorch is used only as device-memory plumbing for the
operator-level entry points; the solve itself takes host or device buffers
straight through the C ABI.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native as nat

__all__ = ["HoloEngine", "session", "prox_session"]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def _stream_ptr(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class HoloEngine:
    """Owns a holo_handle.  ``shard=(rank, nranks, nccl_id_bytes)`` builds a
    z-sharded engine whose forward plane-sum is an NCCL allreduce."""

    def __init__(self, geom, device: int | None = None, shard=None):
        self.lib = nat.load()
        self.geom = geom
        torch = _torch()
        self.device = torch.cuda.current_device() if device is None else int(device)
        g = nat.geometry(geom)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            single = os.environ.get("HOLO_NCCL_SINGLE_RANK") == "1"  # exercise NCCL with one rank
            if shard is None or (shard[1] == 1 and not single):
                nat.check(self.lib.holo_create(ctypes.byref(g), self.device, ctypes.byref(h)), "holo_create")
            else:
                rank, nranks, nid = shard
                buf = ctypes.create_string_buffer(bytes(nid), 128)
                nat.check(self.lib.holo_create_sharded(ctypes.byref(g), self.device, buf, int(rank), int(nranks),
                                                       ctypes.byref(h)), "holo_create_sharded")
        self.h = h
        kb, ke = ctypes.c_int32(), ctypes.c_int32()
        nat.check(self.lib.holo_local_planes(h, ctypes.byref(kb), ctypes.byref(ke)))
        self.k_begin, self.k_end = kb.value, ke.value

    def enable_peer_reduction(self, all_gather_bytes):
        """Switch this z-shard's forward-spectrum allreduce from NCCL to the
        peer-memory kernels (holo_peer_export / holo_peer_import).
        ``all_gather_bytes(blob) -> list[bytes]`` returns every rank's blob in
        rank order (e.g. torch.distributed.all_gather_object)."""
        n = ctypes.c_int64()
        nat.check(self.lib.holo_peer_export(self.h, None, ctypes.byref(n)), "holo_peer_export")
        buf = ctypes.create_string_buffer(n.value)
        nat.check(self.lib.holo_peer_export(self.h, buf, ctypes.byref(n)), "holo_peer_export")
        blobs = all_gather_bytes(buf.raw[: n.value])
        assert all(len(b) == n.value for b in blobs)
        allb = ctypes.create_string_buffer(b"".join(blobs), n.value * len(blobs))
        nat.check(self.lib.holo_peer_import(self.h, allb, n.value), "holo_peer_import")

    @classmethod
    def local_group(cls, geom, nranks: int, device: int | None = None) -> list["HoloEngine"]:
        """``nranks`` z-shards of one geometry on ONE GPU whose two collectives
        are in-process device sums (holo_create_local_group): the sharded code
        path of ``shard=`` without NCCL, for tests.  Drive each engine's solve
        from its own thread (the solves meet in every collective)."""
        lib = nat.load()
        torch = _torch()
        dev = torch.cuda.current_device() if device is None else int(device)
        g = nat.geometry(geom)
        hs = (ctypes.c_void_p * nranks)()
        with torch.cuda.device(dev):
            nat.check(lib.holo_create_local_group(ctypes.byref(g), dev, nranks, hs), "holo_create_local_group")
        out = []
        for r in range(nranks):
            e = cls.__new__(cls)
            e.lib, e.geom, e.device, e.h = lib, geom, dev, ctypes.c_void_p(hs[r])
            kb, ke = ctypes.c_int32(), ctypes.c_int32()
            nat.check(lib.holo_local_planes(e.h, ctypes.byref(kb), ctypes.byref(ke)))
            e.k_begin, e.k_end = kb.value, ke.value
            out.append(e)
        return out

    @property
    def nz_local(self) -> int:
        return self.k_end - self.k_begin

    def close(self):
        if getattr(self, "h", None):
            self.lib.holo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ solver ---
    def operator_norm(self, real: bool = False) -> float:
        """Exact ||A||^2 (complex engine: nz; real engine: max_f sum_k cos^2)."""
        out = ctypes.c_double()
        nat.check(self.lib.holo_operator_norm(self.h, int(real), ctypes.byref(out)), "holo_operator_norm")
        return out.value

    def power_iteration(self, v0, iters: int = 10, real: bool = False) -> float:
        """solver.py:225-247 on the GPU from the given unit-norm start volume (local planes)."""
        torch = _torch()
        v = torch.as_tensor(np.asarray(v0, dtype=np.complex64)).to(f"cuda:{self.device}").contiguous()
        out = ctypes.c_double()
        nat.check(self.lib.holo_power_iteration(self.h, ctypes.c_void_p(v.data_ptr()), int(iters), int(real),
                                                ctypes.byref(out), _stream_ptr(torch)), "holo_power_iteration")
        return out.value

    def solve(self, b, cfg: nat.SolverConfig, stream=None):
        """b: host float64 array (ny, nx), or a CUDA float64 tensor (device path).
        Returns (code, Report, history)."""
        rep = nat.Report()
        if isinstance(b, np.ndarray):
            bb = np.ascontiguousarray(b, dtype=np.float64)
            code = self.lib.holo_solve(self.h, bb.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cfg),
                                       ctypes.byref(rep))
        else:
            torch = _torch()
            assert b.is_cuda and b.dtype == torch.float64 and b.is_contiguous()
            s = ctypes.c_void_p(stream) if stream is not None else _stream_ptr(torch)
            code = self.lib.holo_solve_device(self.h, ctypes.c_void_p(b.data_ptr()), ctypes.byref(cfg),
                                              ctypes.byref(rep), s)
        if code not in (nat.HOLO_OK, nat.HOLO_ERR_DIVERGED):
            nat.check(code, "holo_solve")
        return code, rep, self.history()

    def history(self) -> list[float]:
        n = ctypes.c_int32()
        nat.check(self.lib.holo_history(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=np.float64)
        nat.check(self.lib.holo_history(self.h, out.ctypes.data_as(ctypes.c_void_p), n.value, ctypes.byref(n)))
        return out[: n.value].tolist()

    def plane_nnz(self) -> np.ndarray:
        out = np.zeros(max(self.nz_local, 1), dtype=np.int64)
        nat.check(self.lib.holo_plane_nnz(self.h, out.ctypes.data_as(ctypes.c_void_p)))
        return out[: self.nz_local]

    def export_coo(self):
        """(plane_nnz, rows int32, cols int32, values complex128) of the local planes,
        written by the device straight into the returned arrays."""
        per = self.plane_nnz()
        tot = int(per.sum())
        rows = np.empty(max(tot, 1), np.int32)
        cols = np.empty(max(tot, 1), np.int32)
        vals = np.empty(max(tot, 1), np.complex128)
        n = ctypes.c_int64()
        nat.check(self.lib.holo_export_coo_host(self.h, rows.ctypes.data_as(ctypes.c_void_p),
                                                cols.ctypes.data_as(ctypes.c_void_p),
                                                vals.ctypes.data_as(ctypes.c_void_p), tot, ctypes.byref(n)))
        assert n.value == tot
        return per, rows[:tot], cols[:tot], vals[:tot]

    def solution_dense(self):
        """Dense complex64 solution of the local planes as a CUDA tensor (device copy)."""
        torch = _torch()
        ptr = ctypes.c_void_p()
        nat.check(self.lib.holo_solution_device(self.h, ctypes.byref(ptr)))
        out = torch.empty((self.nz_local,) + tuple(self.geom.plane_shape), dtype=torch.complex64,
                          device=f"cuda:{self.device}")
        torch.cuda.synchronize(self.device)
        cudart = ctypes.CDLL("libcudart.so.12")
        rc = cudart.cudaMemcpy(ctypes.c_void_p(out.data_ptr()), ptr, ctypes.c_size_t(out.numel() * 8), 3)
        if rc != 0:
            raise RuntimeError(f"cudaMemcpy failed ({rc})")
        return out

    # --------------------------------------------------------- operators ---
    def transfer(self, k0: int, k1: int, conj: bool = False):
        torch = _torch()
        out = torch.empty((k1 - k0, self.geom.ny, self.geom.nx), dtype=torch.complex64, device=f"cuda:{self.device}")
        nat.check(self.lib.holo_op_transfer(self.h, k0, k1, int(conj), ctypes.c_void_p(out.data_ptr()),
                                            _stream_ptr(torch)), "holo_op_transfer")
        return out.cpu().numpy().astype(np.complex128)

    def fft2(self, planes, inverse=False):
        torch = _torch()
        t = torch.as_tensor(np.asarray(planes, dtype=np.complex64)).to(f"cuda:{self.device}").contiguous()
        nat.check(self.lib.holo_op_fft2(self.h, ctypes.c_void_p(t.data_ptr()), t.shape[0], int(inverse),
                                        _stream_ptr(torch)), "holo_op_fft2")
        return t.cpu().numpy()

    def forward(self, dense_local):
        torch = _torch()
        x = torch.as_tensor(np.asarray(dense_local, dtype=np.complex64)).to(f"cuda:{self.device}").contiguous()
        out = torch.empty(self.geom.plane_shape, dtype=torch.float32, device=x.device)
        nat.check(self.lib.holo_op_forward(self.h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                           _stream_ptr(torch)), "holo_op_forward")
        return out.cpu().numpy().astype(np.float64)

    def adjoint(self, r, scale=1.0):
        torch = _torch()
        rt = torch.as_tensor(np.asarray(r, dtype=np.float32)).to(f"cuda:{self.device}").contiguous()
        out = torch.empty((self.nz_local,) + tuple(self.geom.plane_shape), dtype=torch.complex64, device=rt.device)
        nat.check(self.lib.holo_op_adjoint(self.h, ctypes.c_void_p(rt.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                           float(scale), _stream_ptr(torch)), "holo_op_adjoint")
        return out.cpu().numpy().astype(np.complex128)

    def prox_fl(self, stack, tau_l1, tau_tv, inner):
        torch = _torch()
        v = torch.as_tensor(np.asarray(stack, dtype=np.complex64)).to(f"cuda:{self.device}").contiguous()
        out = torch.empty_like(v)
        n, ny, nx = v.shape
        nat.check(self.lib.holo_op_prox_fl(self.h, ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                           n, ny, nx, float(tau_l1), float(tau_tv), int(inner), _stream_ptr(torch)),
                  "holo_op_prox_fl")
        return out.cpu().numpy().astype(np.complex128)


_cache: dict = {}
_cache_lock = threading.Lock()


def session(geom, device: int | None = None) -> HoloEngine:
    """Per-(geometry, device) engine, kept for reuse across calls (the
    reference CLI calls fista once per frame with one geometry)."""
    torch = _torch()
    dev = torch.cuda.current_device() if device is None else int(device)
    key = (geom.nx, geom.ny, geom.nz, geom.pitch, geom.dz, geom.z0, geom.wavelength, dev)
    with _cache_lock:
        eng = _cache.get(key)
        if eng is None:
            if len(_cache) >= 2:  # bound device memory held by cached engines
                old = _cache.pop(next(iter(_cache)))
                old.close()
            eng = HoloEngine(geom, dev)
            _cache[key] = eng
        return eng


class _ProxGeom:
    nx = ny = nz = 8
    pitch = dz = z0 = wavelength = 1.0
    plane_shape = (8, 8)


def prox_session() -> HoloEngine:
    """A minimal handle for the shape-free prox operator."""
    g = _ProxGeom()
    g.z0 = 0.0
    return session(g)


def clear_sessions():
    with _cache_lock:
        for e in _cache.values():
            e.close()
        _cache.clear()
