"""GPU fixpoint reference and verification reductions.

    solve_fixpoint(grid, bc, tol=1e-12, workers=1, max_passes=None)   E/oracle.py:22-70
    max_residual(grid)                                                 E/harness.py:147-162

Same semantics as the reference: full-grid Jacobi passes phi <- min(phi, U),
stop when nothing decreased or the largest decrease is below tol, RuntimeError
past the cap (10*(nx+ny), 10*(nx+ny+nz) in 3D); stats.iterations = passes,
stats.solver_calls = passes x free cells.  Runs in the sm_100a engine
(k_fixpoint / k_residual), bit-identical to the CPU restatement.
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np
import torch

from . import _native
from .grid import seed_linear
from .ifim import (_check_tol, _DeviceGrid, _host_mark_sources, _HostResult, _ptr, geometry, resolve_workers,
                   workspace)
from .result import RunStats, SolverResult


def solve_fixpoint(grid, bc, tol: float = 1e-12, workers: int = 1, max_passes: int | None = None) -> SolverResult:
    t0 = time.perf_counter()
    _check_tol(tol)
    resolve_workers(workers)
    idx, val = seed_linear(grid, bc)
    dg = _DeviceGrid(grid)
    geom = geometry(grid)
    ws = workspace(geom, dg.device)
    ws.gen += 1
    si = torch.as_tensor(idx, dtype=torch.int64, device=dg.device)
    sv = torch.as_tensor(val, dtype=torch.float64, device=dg.device)
    st = _native.Stats()
    out = _HostResult(dg)
    rc = _native.lib(geom.dtype).eik_solve_fixpoint(C.byref(geom), _ptr(dg.phi), _ptr(dg.speed), _ptr(dg.state), _ptr(si),
                                          _ptr(sv), len(idx), float(tol), int(max_passes or 0), ws.ptr, ws.nbytes,
                                          C.byref(st), dg.stream)
    phi = None
    if dg.host:
        _host_mark_sources(grid, idx)
        phi = out.commit()
    _native.check(rc, geom.dtype)
    stats = RunStats(iterations=int(st.iterations), solver_calls=int(st.solver_calls))
    stats.device_ms = {"total": float(st.total_ms)}
    stats.gpu_launches = int(st.gpu_launches)
    if phi is None:
        phi = grid.phi.copy() if isinstance(grid.phi, np.ndarray) else grid.phi.clone()
    stats.wall_time = time.perf_counter() - t0
    return SolverResult(phi=phi, stats=stats)


def max_residual(grid) -> float:
    """Largest |phi - update(neighbours)| over free cells with finite phi (0.0 if none)."""
    dg = _DeviceGrid(grid)
    geom = geometry(grid)
    ws = workspace(geom, dg.device)
    ws.gen += 1
    out = C.c_double(0.0)
    _native.check(_native.lib(geom.dtype).eik_max_residual(C.byref(geom), _ptr(dg.phi), _ptr(dg.speed), _ptr(dg.state),
                                                 ws.ptr, ws.nbytes, C.byref(out), dg.stream))
    return float(out.value)
