"""Field snapshots.

``export_field_csv`` / ``import_field_csv`` keep the reference's text format
(E/harness.py:326-380: a geometry line, then ``i,j,phi`` rows with repr
values, bit-exact round trip) for 2D grids.  At 512^3-1024^3 a text file is
infeasible (1e9 rows), so ``export_field_npy`` / ``import_field_npy`` write the
same content as a raw float64 ``.npy`` array plus a JSON geometry sidecar,
streamed plane-chunk by plane-chunk from the device (no full host copy of the
field), and read it back memory-mapped.  Like the CSV import, the returned grid
is a field container: unit speed, all-FAR state.
"""
from __future__ import annotations

import json

import numpy as np
import torch

from .grid import Grid, Grid3D, new_grid

_CHUNK_BYTES = 1 << 28


def export_field_csv(grid: Grid, path: str) -> None:
    """E/harness.py:326-342 (2D)."""
    if getattr(grid, "ndim", 2) != 2:
        raise ValueError("the CSV snapshot format is 2D (use export_field_npy for 3D fields)")
    phi = grid.phi.detach().cpu().numpy() if isinstance(grid.phi, torch.Tensor) else np.asarray(grid.phi)
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"{grid.nx},{grid.ny},{grid.dx!r},{grid.dy!r},{grid.origin[0]!r},{grid.origin[1]!r}\n")
        for j in range(grid.ny):
            for i in range(grid.nx):
                fh.write(f"{i},{j},{float(phi[j, i])!r}\n")


def import_field_csv(path: str) -> Grid:
    """E/harness.py:345-380: geometry + phi; unit speed, all-FAR state; malformed input raises."""
    with open(path, "r", encoding="ascii") as fh:
        header = fh.readline()
        parts = header.strip().split(",")
        if len(parts) != 6:
            raise ValueError(f"{path}:1: expected 6 header fields nx,ny,dx,dy,x0,y0, got {len(parts)}")
        try:
            nx, ny = int(parts[0]), int(parts[1])
            dx, dy, x0, y0 = (float(p) for p in parts[2:])
        except ValueError:
            raise ValueError(f"{path}:1: malformed header {header.strip()!r}") from None
        grid = new_grid(nx, ny, dx, dy, origin=(x0, y0), speed=1.0)
        count = 0
        for lineno, line in enumerate(fh, start=2):
            if not line.strip():
                continue
            fields = line.strip().split(",")
            if len(fields) != 3:
                raise ValueError(f"{path}:{lineno}: expected i,j,phi, got {line.strip()!r}")
            try:
                i, j, value = int(fields[0]), int(fields[1]), float(fields[2])
            except ValueError:
                raise ValueError(f"{path}:{lineno}: malformed row {line.strip()!r}") from None
            if not (0 <= i < nx and 0 <= j < ny):
                raise ValueError(f"{path}:{lineno}: cell ({i}, {j}) outside {nx}x{ny} grid")
            grid.phi[j, i] = value
            count += 1
        if count != nx * ny:
            raise ValueError(f"{path}: expected {nx * ny} cell rows, found {count}")
    return grid


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
