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
import os
import threading

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

    def solve(self, speed_local, state_local, seeds, tol=1e-12, phi_local=None):
        """speed/state: this rank's planes (device); phi_local: its starting phi planes (any
        device, default +inf).  Returns (this rank's phi planes, global RunStats)."""
        import torch.distributed as dist

        nz, ny, nx = self.shape
        if phi_local is None:
            self.phi.fill_(INF)
        else:
            self.phi.copy_(phi_local, non_blocking=True)
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


# ---------------------------------------------------------------------------
# solve_ifim(..., devices=...): one process, several GPUs
# ---------------------------------------------------------------------------

def resolve_devices(devices):
    """``devices`` (int count or list of CUDA indices) or EIKONAL_DEVICES -> list of devices per
    z-slab rank, or None for the single-device path.  A device may appear more than once (its
    ranks then share one launch); ranks on one device must be contiguous."""
    if devices is None:
        env = os.environ.get("EIKONAL_DEVICES", "").strip()
        if not env:
            return None
        devices = int(env) if env.isdigit() else [int(v) for v in env.split(",") if v.strip()]
    if isinstance(devices, (int, np.integer)) and not isinstance(devices, bool):
        if devices < 1:
            raise ValueError(f"devices must be >= 1, got {devices}")
        if devices > torch.cuda.device_count():
            raise ValueError(f"devices={devices} but only {torch.cuda.device_count()} CUDA devices are visible")
        devices = list(range(int(devices)))
    devices = [int(d) for d in devices]
    if not devices:
        raise ValueError("devices is empty")
    n = torch.cuda.device_count()
    for d in devices:
        if not 0 <= d < n:
            raise ValueError(f"CUDA device {d} is not visible ({n} devices)")
    seen = []
    for d in devices:
        if seen and d != seen[-1] and d in seen:
            raise ValueError(f"ranks on one device must be contiguous, got {devices}")
        seen.append(d)
    return devices if len(devices) > 1 else None


def solve_multi(grid, idx, val, tol, devices):
    """Peer-slab solve of a Grid3D over ``devices`` (one z-slab rank per entry).  Mutates
    grid.phi / grid.state like the single-device solve; returns (RunStats, phi copy)."""
    from .grid import CellState

    if len(grid.phi.shape) != 3:
        raise ValueError("a multi-device solve shards z-slabs of a 3D grid (Grid3D)")
    nz, ny, nx = (int(v) for v in grid.phi.shape)
    R = len(devices)
    part = SlabPartition(nz, R)
    bounds = [part.bounds(r) for r in range(R)]
    h = float(grid.dx)
    if not (grid.dx == grid.dy == grid.dz):
        raise ValueError("3D grids require dx == dy == dz")

    def src(a):
        return a if isinstance(a, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(a))

    phi_src, sp_src, st_src = src(grid.phi), src(grid.speed), src(grid.state)
    lib = _native.lib()
    for a in sorted(set(devices)):
        for b in sorted(set(devices)):
            if a != b:
                _native.check(lib.eik_peer_enable(a, b))
    phis, sps, sts, wss = [], [], [], []
    for q, (z0, z1) in enumerate(bounds):
        dev = torch.device("cuda", devices[q])
        phis.append(phi_src[z0:z1].to(dev, torch.float64).contiguous())
        sps.append(sp_src[z0:z1].to(dev, torch.float64).contiguous())
        sts.append(st_src[z0:z1].to(dev, torch.uint8).contiguous().clone())
        wss.append(torch.empty(_ws_bytes(nx, ny, z1 - z0, h), dtype=torch.uint8, device=dev))
    ranks = (_native.Rank * R)(*[_native.Rank(t.data_ptr(), w.data_ptr(), z1 - z0)
                                  for t, w, (z0, z1) in zip(phis, wss, bounds)])
    groups = []  # (device, r_begin, r_end)
    for q, d in enumerate(devices):
        if groups and groups[-1][0] == d:
            groups[-1][2] = q + 1
        else:
            groups.append([d, q, q + 1])
    g = _geom((nz, ny, nx), h)
    hcap = 40 * (nx + ny + nz) + 2
    outs, hists, errs = {}, {}, {}
    seeds = {}
    for d, rb, re in groups:
        dev = torch.device("cuda", d)
        with torch.cuda.device(dev):
            seeds[d] = (torch.as_tensor(idx, dtype=torch.int64, device=dev),
                        torch.as_tensor(val, dtype=torch.float64, device=dev))
            spp = (C.c_void_p * (re - rb))(*[t.data_ptr() for t in sps[rb:re]])
            stp = (C.c_void_p * (re - rb))(*[t.data_ptr() for t in sts[rb:re]])
            stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
            _native.check(lib.eik_mr_prepare(C.byref(g), R, ranks, rb, re, spp, stp, _p(seeds[d][0]),
                                             _p(seeds[d][1]), len(idx), float(tol), stream))

    def run(d, rb, re):
        dev = torch.device("cuda", d)
        try:
            with torch.cuda.device(dev):
                spp = (C.c_void_p * (re - rb))(*[t.data_ptr() for t in sps[rb:re]])
                stp = (C.c_void_p * (re - rb))(*[t.data_ptr() for t in sts[rb:re]])
                stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
                hist = np.zeros(hcap, dtype=np.int64)
                out = _native.Stats()
                rc = lib.eik_mr_run(C.byref(g), R, ranks, rb, re, spp, stp, float(tol),
                                    hist.ctypes.data_as(C.c_void_p), hcap, C.byref(out), stream)
                outs[d], hists[d] = out, hist
                if rc:
                    errs[d] = (rc, lib.eik_last_error().decode(errors="replace"))
        except Exception as e:  # pragma: no cover - surfaced below
            errs[d] = (-1, repr(e))

    threads = [threading.Thread(target=run, args=tuple(gr)) for gr in groups]
    for t in threads:  # every device's persistent kernels must be resident together (cross-rank barrier)
        t.start()
    for t in threads:
        t.join()
    if errs:
        rc, msg = next(iter(errs.values()))
        if rc == 2:
            raise RuntimeError(msg)
        raise RuntimeError(f"multi-device solve failed: {msg}")
    d0 = groups[0][0]
    stats = _stats(outs[d0], hists[d0])
    # write back (in place, like the single-device solve)
    for q, (z0, z1) in enumerate(bounds):
        if isinstance(grid.phi, torch.Tensor):
            grid.phi[z0:z1].copy_(phis[q].to(grid.phi.device))
        else:
            grid.phi[z0:z1] = phis[q].cpu().numpy()
    flat = grid.state.reshape(-1)
    for c in idx:
        flat[c] = CellState.SOURCE
    phi = grid.phi.copy() if isinstance(grid.phi, np.ndarray) else grid.phi.clone()
    return stats, phi
