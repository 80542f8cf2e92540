"""solve_fim on the GPU (E/fim.py:62-144).

The paper's comparison baseline: an active list whose every iteration also
re-checks the neighbours of the active cells (the per-cell cost iFIM drops).
Same signature, in-place semantics, errors and statistics as the reference;
phi and every RunStats integer are bit-identical to it (C ABI eik_solve_fim).
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


def solve_fim(grid, bc, tol: float = 1e-12, workers: int = 1) -> SolverResult:
    """E/fim.py:62-144 on the device (2D, and its 3D generalisation on Grid3D)."""
    t0 = time.perf_counter()
    _check_tol(tol)  # E/fim.py:64-65
    resolve_workers(workers)
    idx, val = seed_linear(grid, bc)  # apply_boundary validation (E/grid.py:204-211)
    dg = _DeviceGrid(grid)
    geom = geometry(grid)
    ws = workspace(geom, dg.device)
    ws.gen += 1
    si = torch.as_tensor(idx, dtype=torch.int64, device=dg.device)
    sv = torch.as_tensor(val, dtype=torch.float64, device=dg.device)
    st = _native.Stats()
    out = _HostResult(dg)
    rc = _native.lib(geom.dtype).eik_solve_fim(C.byref(geom), _ptr(dg.phi), _ptr(dg.speed), _ptr(dg.state), _ptr(si),
                                               _ptr(sv), len(idx), float(tol), ws.ptr, ws.nbytes, C.byref(st),
                                               dg.stream)
    phi = None
    if dg.host:
        _host_mark_sources(grid, idx)
        phi = out.commit()
    _native.check(rc, geom.dtype)
    stats = RunStats(iterations=int(st.iterations), solver_calls=int(st.solver_calls),
                     peak_active=int(st.peak_active))
    stats.phi_writes = int(st.phi_writes)
    stats.device_ms = {"total": float(st.total_ms)}
    stats.gpu_launches = int(st.gpu_launches)
    if phi is None:
        phi = grid.phi.copy() if isinstance(grid.phi, np.ndarray) else grid.phi.clone()
    stats.wall_time = time.perf_counter() - t0
    return SolverResult(phi=phi, stats=stats)
