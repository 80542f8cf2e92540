"""Per-rank B200 engine for the z-slab protocol (paper_2106_15869_b200/slab.py).

Each rank holds its planes [z0, z1) plus one ghost plane per side on its GPU
and runs the same kernels as the single-device solve in slab mode
(EIK_GEOM_SLAB): one bulk-synchronous step per call, local counts out, ghost
planes / activation requests / decrease planes exchanged by the driver
(NCCL through torch.distributed on a multi-GPU box, or ThreadComm for the
lockstep emulation on one device).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native
from .ifim import Workspace
from .slab import SlabEngine, SlabPartition, SlabSolver

INF = float("inf")


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


class SlabGpuEngine(SlabEngine):
    def __init__(self, shape, h, speed, state, z0, z1, device, tol=1e-12):
        nz, ny, nx = shape
        self.shape, self.h, self.tol = shape, float(h), float(tol)
        self.z0, self.z1, self.nl = z0, z1, z1 - z0
        self.nx, self.ny = nx, ny
        self.dev = torch.device(device)
        L = self.nl + 2
        self.geom = _native.Geom(nx, ny, L, self.h, self.h, self.h, 3, 0, _native.EIK_GEOM_SLAB, 0)
        zs = [min(max(z, 0), nz - 1) for z in range(z0 - 1, z1 + 1)]

        def planes(a, dtype):
            a = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(a))
            return a.reshape(nz, ny, nx)[zs].to(self.dev, dtype).contiguous()

        self.speed = planes(speed, torch.float64)
        self.state = planes(state, torch.uint8)
        self.state[0].zero_()
        self.state[-1].zero_()
        self.phi = torch.full((L, ny, nx), INF, dtype=torch.float64, device=self.dev)
        self.ws = Workspace(self.geom, self.dev)
        off = (C.c_int64 * 4)()
        _native.check(_native.lib().eik_workspace_offsets(C.byref(self.geom), off))
        N, W = L * ny * nx, (nx + 31) // 32
        buf = self.ws.buf
        self.phi2 = buf[off[0]:off[0] + N * 8].view(torch.float64).view(L, ny, nx)
        self.touched = buf[off[1]:off[1] + L * ny * W * 4].view(torch.int32).view(L, ny, W)
        self.D = [buf[off[k]:off[k] + L * ny * W * 4].view(torch.int32).view(L, ny, W) for k in (2, 3)]
        self.bufs = (self.phi, self.phi2)
        self.cur = 0  # phi buffer holding the current values
        self.it = 0
        self.r = 0
        self.reset_counters()

    def reset_counters(self):
        """Local remedy counters + kernel time (bench roofline) and launch count."""
        self.rem_calls_local = self.rem_decs_local = 0
        self.rem_ms = 0.0
        self.launches = 0

    @property
    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    # ---- SlabEngine ----------------------------------------------------
    def boundary_planes(self):
        P = self.bufs[self.cur]
        return P[1].clone(), P[self.nl].clone()

    def set_ghosts(self, lo, hi):
        P = self.bufs[self.cur]
        P[0].copy_(lo) if lo is not None else P[0].fill_(INF)
        P[self.nl + 1].copy_(hi) if hi is not None else P[self.nl + 1].fill_(INF)

    def init_active(self, seeds):
        nx, ny = self.nx, self.ny
        idx, val = [], []
        for c, v in seeds:
            z, rem = divmod(int(c), nx * ny)
            if self.z0 - 1 <= z <= self.z1:
                idx.append((z - self.z0 + 1) * nx * ny + rem)
                val.append(float(v))
        si = torch.as_tensor(idx, dtype=torch.int64, device=self.dev)
        sv = torch.as_tensor(val, dtype=torch.float64, device=self.dev)
        n = C.c_int64(0)
        _native.check(_native.lib().eik_slab_update_init(
            C.byref(self.geom), _p(self.phi), _p(self.speed), _p(self.state), _p(si), _p(sv), len(idx), self.tol,
            self.ws.ptr, self.ws.nbytes, C.byref(n), self._stream))
        self.cur, self.it = 0, 0
        self.launches += 4  # seeds, prep, initial activation (+ memsets)
        return int(n.value)

    def update_local(self):
        _native.check(_native.lib().eik_slab_update_iter(
            C.byref(self.geom), _p(self.phi), _p(self.speed), _p(self.state), self.tol, self.it, self.ws.ptr,
            self.ws.nbytes, self._stream))
        self.launches += 2  # update iteration + request application
        self.it += 1
        self.cur = self.it & 1
        req_lo = self.touched[0].clone()
        req_hi = self.touched[self.nl + 1].clone()
        self.touched[0].zero_()
        self.touched[self.nl + 1].zero_()
        return req_lo, req_hi

    def apply_requests(self, got_lo, got_hi):
        n = C.c_int64(0)
        _native.check(_native.lib().eik_slab_apply_requests(
            C.byref(self.geom), _p(got_lo), _p(got_hi), self.it - 1, self.ws.ptr, self.ws.nbytes, C.byref(n),
            self._stream))
        return int(n.value)

    def build_local(self):
        free, flagged = C.c_int64(0), C.c_int64(0)
        _native.check(_native.lib().eik_slab_build(
            C.byref(self.geom), _p(self.phi), _p(self.speed), _p(self.state), self.tol, self.ws.ptr, self.ws.nbytes,
            C.byref(free), C.byref(flagged), self._stream))
        self.cur, self.r = 0, 0
        self.launches += 2
        return int(free.value), int(flagged.value)

    def remedy_boundary_d(self):
        if self.r == 0:
            z = torch.zeros_like(self.D[0][1])
            return z, z.clone()
        Dl = self.D[(self.r - 1) & 1]
        return Dl[1].clone(), Dl[self.nl].clone()

    def remedy_local(self, g_lo, g_hi, first):
        if self.r > 0:  # ghost rows of D_{r-1}, read by round r's dilation
            Dp = self.D[(self.r - 1) & 1]
            Dp[0].copy_(g_lo) if g_lo is not None else Dp[0].zero_()
            Dp[self.nl + 1].copy_(g_hi) if g_hi is not None else Dp[self.nl + 1].zero_()
        calls, decs = C.c_int64(0), C.c_int64(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(_native.lib().eik_slab_remedy_round(
            C.byref(self.geom), _p(self.phi), _p(self.speed), _p(self.state), self.tol, self.r, self.ws.ptr,
            self.ws.nbytes, C.byref(calls), C.byref(decs), self._stream))
        e1.record()
        e1.synchronize()
        self.rem_ms += e0.elapsed_time(e1)
        self.rem_calls_local += int(calls.value)
        self.rem_decs_local += int(decs.value)
        self.launches += 1
        self.r += 1
        self.cur = self.r & 1
        return int(calls.value), int(decs.value)

    def result(self):
        return self.bufs[self.cur][1:self.nl + 1]


def solve_ifim_slabs(shape, h, speed, state, seeds, comm, tol=1e-12, device=None):
    """One rank's share of a z-sharded 3D solve; returns (owned phi planes, SlabStats)."""
    part = SlabPartition(shape[0], comm.world)
    z0, z1 = part.bounds(comm.rank)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    e = SlabGpuEngine(shape, h, speed, state, z0, z1, dev, tol)
    s = sum(shape)
    st = SlabSolver(e, comm, (40 * s, 20 * s), tensor_device=dev).solve(seeds)
    return e.result(), st
