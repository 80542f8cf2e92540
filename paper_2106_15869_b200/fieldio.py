"""Binary field snapshots.

The reference's text format (E/harness.py:326-380, CSV rows ``i,j,phi``) is out
of scope here and infeasible at 512^3-1024^3 (1e9 rows);
small 2D fields can still go through the reference's own exporter.
``export_field_npy`` / ``import_field_npy`` write the field as a raw float64
``.npy`` array plus a JSON geometry sidecar, streamed plane-chunk by
plane-chunk from the device (no full host copy of the field), and read it back
memory-mapped.  The returned grid is a field container: unit speed, all-FAR
state.
"""
from __future__ import annotations

import json

import numpy as np
import torch

from .grid import Grid, Grid3D, new_grid

_CHUNK_BYTES = 1 << 28


def _geometry(grid) -> dict:
    if getattr(grid, "ndim", 2) == 3:
        return {"ndim": 3, "nx": grid.nx, "ny": grid.ny, "nz": grid.nz, "h": grid.h, "origin": list(grid.origin)}
    return {"ndim": 2, "nx": grid.nx, "ny": grid.ny, "dx": grid.dx, "dy": grid.dy, "origin": list(grid.origin)}


def export_field_npy(grid, path: str) -> None:
    """phi as a float64 .npy at ``path`` (+ ``path + '.json'`` geometry), streamed from the device
    (or copied from host arrays) in chunks of planes / rows."""
    phi = grid.phi
    shape = tuple(int(v) for v in phi.shape)
    out = np.lib.format.open_memmap(path, mode="w+", dtype=np.float64, shape=shape)
    row_bytes = 8 * int(np.prod(shape[1:]))
    step = max(1, _CHUNK_BYTES // row_bytes)
    for a in range(0, shape[0], step):
        b = min(shape[0], a + step)
        if isinstance(phi, torch.Tensor):
            out[a:b] = phi[a:b].detach().to("cpu", torch.float64).numpy()
        else:
            out[a:b] = np.asarray(phi[a:b], dtype=np.float64)
    out.flush()
    del out
    with open(path + ".json", "w") as fh:
        json.dump(_geometry(grid), fh)


def import_field_npy(path: str, device=None):
    """Read a snapshot written by export_field_npy: Grid / Grid3D with phi loaded (on ``device``
    if given, else a host array), unit speed and all-FAR state."""
    with open(path + ".json") as fh:
        geo = json.load(fh)
    arr = np.load(path, mmap_mode="r")
    if arr.dtype != np.float64:
        raise ValueError(f"{path}: expected float64 data, got {arr.dtype}")
    if geo["ndim"] == 3:
        shape = (geo["nz"], geo["ny"], geo["nx"])
    else:
        shape = (geo["ny"], geo["nx"])
    if tuple(arr.shape) != shape:
        raise ValueError(f"{path}: array shape {arr.shape} does not match the geometry {shape}")
    if device is not None:
        phi = torch.empty(shape, dtype=torch.float64, device=device)
        rows = max(1, _CHUNK_BYTES // (8 * int(np.prod(shape[1:]))))
        for a in range(0, shape[0], rows):
            b = min(shape[0], a + rows)
            phi[a:b].copy_(torch.from_numpy(np.ascontiguousarray(arr[a:b])))
        speed = torch.ones(shape, dtype=torch.float64, device=device)
        state = torch.zeros(shape, dtype=torch.uint8, device=device)
    else:
        phi = np.array(arr)
        speed = np.ones(shape)
        state = np.zeros(shape, dtype=np.uint8)
    if geo["ndim"] == 3:
        return Grid3D(geo["nx"], geo["ny"], geo["nz"], geo["h"], tuple(geo["origin"]), phi, speed, state)
    return Grid(geo["nx"], geo["ny"], geo["dx"], geo["dy"], tuple(geo["origin"]), phi, speed, state)
