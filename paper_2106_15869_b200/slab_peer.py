"""Peer-memory z-slabs: the B200 multi-GPU path.

One 3D grid is sharded into z-slabs, one per rank; each rank keeps its planes
in its own phi buffer and workspace.  The persistent update / remedy kernels
read the neighbours' boundary planes of phi and of the decrease bitmap, and
activate cells on the neighbours' boundary planes, directly through
device-visible pointers, with one hierarchical barrier (grid, then cross-rank)
per iteration and global counts summed on the device -- no ghost copies, no
host round trips (C ABI: eik_mr_prepare / eik_mr_run).

* ``solve_emulated`` runs R ranks on ONE GPU as CTA groups of a single
  cooperative launch per phase (the ranks' kernels never wait on separate
  launches); this is how the multi-rank kernels are tested here.
* ``solve_distributed`` runs one rank per process/GPU; buffers come from
  torch symmetric memory (NVLink peer mappings through NVSwitch).
Results and every RunStats integer are identical to the single-device solve.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native
from .result import RunStats
from .slab import SlabPartition

INF = float("inf")


def _p(t):
    return C.c_void_p(t.data_ptr())


def _geom(shape, h):
    nz, ny, nx = shape
    return _native.Geom(nx, ny, nz, float(h), float(h), float(h), 3, 0, 0, 0)


def _ws_bytes(nx, ny, nz, h):
    g = _native.Geom(nx, ny, nz, float(h), float(h), float(h), 3, 0, 0, 0)
    n = C.c_size_t(0)
    _native.check(_native.lib().eik_workspace_size(C.byref(g), C.byref(n)))
    return int(n.value)


def _stats(st, hist):
    s = RunStats(iterations=int(st.iterations), solver_calls=int(st.solver_calls), peak_active=int(st.peak_active),
                 peak_remedy=int(st.peak_remedy), active_history=hist[: int(st.upd_iterations)].tolist())
    s.phi_writes = int(st.phi_writes)
    s.phases = {"update": {"iterations": int(st.upd_iterations), "solver_calls": int(st.upd_calls),
                           "converged": int(st.converged)},
                "build": {"solver_calls": int(st.build_calls), "remedy_size": int(st.remedy_size)},
                "remedy": {"iterations": int(st.rem_iterations), "solver_calls": int(st.rem_calls)}}
    s.device_ms = {"update": float(st.upd_ms), "build": float(st.build_ms), "remedy": float(st.rem_ms),
                   "total": float(st.total_ms)}
    s.gpu_launches = int(st.gpu_launches)
    return s


class EmulatedSlabs:
    """R peer-slab ranks on one device (buffers reusable across solves)."""

    def __init__(self, shape, h, R, device):
        nz, ny, nx = shape
        self.shape, self.h, self.R, self.dev = shape, float(h), R, torch.device(device)
        part = SlabPartition(nz, R)
        self.bounds = [part.bounds(r) for r in range(R)]
        self.phi = [torch.empty((z1 - z0, ny, nx), dtype=torch.float64, device=self.dev) for z0, z1 in self.bounds]
        self.ws = [torch.empty(_ws_bytes(nx, ny, z1 - z0, h), dtype=torch.uint8, device=self.dev)
                   for z0, z1 in self.bounds]
        self.ranks = (_native.Rank * R)(*[_native.Rank(t.data_ptr(), w.data_ptr(), z1 - z0)
                                          for t, w, (z0, z1) in zip(self.phi, self.ws, self.bounds)])

    def solve(self, speed, state, seeds, tol=1e-12):
        """speed/state: global (nz, ny, nx) CUDA tensors; seeds [(global linear, value)]."""
        nz, ny, nx = self.shape
        sp = [speed[z0:z1].contiguous() for z0, z1 in self.bounds]
        st = [state[z0:z1].clone() for z0, z1 in self.bounds]
        for t in self.phi:
            t.fill_(INF)
        spp = (C.c_void_p * self.R)(*[t.data_ptr() for t in sp])
        stp = (C.c_void_p * self.R)(*[t.data_ptr() for t in st])
        si = torch.as_tensor([c for c, _ in seeds], dtype=torch.int64, device=self.dev)
        sv = torch.as_tensor([v for _, v in seeds], dtype=torch.float64, device=self.dev)
        g = _geom(self.shape, self.h)
        stream = C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
        lib = _native.lib()
        _native.check(lib.eik_mr_prepare(C.byref(g), self.R, self.ranks, 0, self.R, spp, stp, _p(si), _p(sv),
                                         len(seeds), float(tol), stream))
        hcap = 40 * (nx + ny + nz) + 2
        hist = np.zeros(hcap, dtype=np.int64)
        out = _native.Stats()
        _native.check(lib.eik_mr_run(C.byref(g), self.R, self.ranks, 0, self.R, spp, stp, float(tol),
                                     hist.ctypes.data_as(C.c_void_p), hcap, C.byref(out), stream))
        phi = torch.cat(self.phi, dim=0)
        return phi, _stats(out, hist), torch.cat(st, dim=0)


def solve_emulated(shape, h, speed, state, seeds, R, tol=1e-12, device="cuda"):
    return EmulatedSlabs(shape, h, R, device).solve(speed, state, seeds, tol)


class DistributedSlabs:
    """One peer-slab rank per process/GPU over torch symmetric memory (NVLink)."""

    def __init__(self, shape, h, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        nz, ny, nx = shape
        self.shape, self.h = shape, float(h)
        self.rank, self.R = dist.get_rank(group), dist.get_world_size(group)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        part = SlabPartition(nz, self.R)
        self.bounds = [part.bounds(r) for r in range(self.R)]
        sizes = [(z1 - z0) * ny * nx * 8 + _ws_bytes(nx, ny, z1 - z0, h) for z0, z1 in self.bounds]
        per = (max(sizes) + 4095) // 4096 * 4096  # same allocation size on every rank
        self.buf = symm_mem.empty(per, dtype=torch.uint8, device=self.dev)
        self.hdl = symm_mem.rendezvous(self.buf, group=dist.group.WORLD if group is None else group)
        ranks = []
        for r, (z0, z1) in enumerate(self.bounds):
            b = self.buf if r == self.rank else self.hdl.get_buffer(r, (per,), torch.uint8)
            nphi = (z1 - z0) * ny * nx * 8
            ranks.append(_native.Rank(b.data_ptr(), b.data_ptr() + (nphi + 255) // 256 * 256, z1 - z0))
        self.ranks = (_native.Rank * self.R)(*ranks)
        z0, z1 = self.bounds[self.rank]
        self.phi = self.buf[: (z1 - z0) * ny * nx * 8].view(torch.float64).view(z1 - z0, ny, nx)

    def solve(self, speed_local, state_local, seeds, tol=1e-12):
        import torch.distributed as dist

        nz, ny, nx = self.shape
        self.phi.fill_(INF)
        spp = (C.c_void_p * 1)(speed_local.data_ptr())
        stp = (C.c_void_p * 1)(state_local.data_ptr())
        si = torch.as_tensor([c for c, _ in seeds], dtype=torch.int64, device=self.dev)
        sv = torch.as_tensor([v for _, v in seeds], dtype=torch.float64, device=self.dev)
        g = _geom(self.shape, self.h)
        stream = C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
        lib = _native.lib()
        _native.check(lib.eik_mr_prepare(C.byref(g), self.R, self.ranks, self.rank, self.rank + 1, spp, stp,
                                         _p(si), _p(sv), len(seeds), float(tol), stream))
        torch.cuda.synchronize(self.dev)
        dist.barrier()  # every rank's control blocks are reset before anyone reaches a world barrier
        hcap = 40 * (nx + ny + nz) + 2
        hist = np.zeros(hcap, dtype=np.int64)
        out = _native.Stats()
        _native.check(lib.eik_mr_run(C.byref(g), self.R, self.ranks, self.rank, self.rank + 1, spp, stp, float(tol),
                                     hist.ctypes.data_as(C.c_void_p), hcap, C.byref(out), stream))
        return self.phi, _stats(out, hist)
