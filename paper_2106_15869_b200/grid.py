"""Grid, speed, source and boundary conventions of the reference, plus 3D.

2D mirrors E/grid.py (E = /root/reference/pkg/src/eikonal) exactly: arrays of
shape (ny, nx), linear index ``j * nx + i``, cell centre ``origin + (i*dx,
j*dy)``, phi = +inf for unreached cells, speed 0 => Blocked (E/grid.py:1-8,
108-144).  3D is the extension SURVEY.md §8b asks for: arrays of shape
(nz, ny, nx), linear index ``(k * ny + j) * nx + i``, cubic cells
(dx == dy == dz; the reference has no anisotropic 3D solver).

The arrays may be numpy arrays, CPU torch tensors or CUDA torch tensors; the
solvers run on the GPU either way and update ``phi``/``state`` in place.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Any, Callable, NamedTuple

import numpy as np

INF = float("inf")


class CellState(IntEnum):
    """E/grid.py:21-26."""

    FAR = 0
    ACTIVE = 1
    SOURCE = 2
    REMEDY = 3
    BLOCKED = 4


class CellIndex(NamedTuple):
    """E/grid.py:29-34."""

    i: int
    j: int

    def linear(self, nx: int) -> int:
        return self.j * nx + self.i


class CellIndex3D(NamedTuple):
    i: int
    j: int
    k: int

    def linear(self, nx: int, ny: int) -> int:
        return (self.k * ny + self.j) * nx + self.i


@dataclass
class Grid:
    """E/grid.py:54-79: phi / speed / state of shape (ny, nx)."""

    nx: int
    ny: int
    dx: float
    dy: float
    origin: tuple
    phi: Any = field(repr=False)
    speed: Any = field(repr=False)
    state: Any = field(repr=False)

    ndim = 2

    @property
    def shape(self) -> tuple:
        return (self.ny, self.nx)

    def in_bounds(self, i: int, j: int) -> bool:
        return 0 <= i < self.nx and 0 <= j < self.ny

    def cell_center(self, i: int, j: int) -> tuple:
        return (self.origin[0] + i * self.dx, self.origin[1] + j * self.dy)

    def cell_centers(self):
        x = self.origin[0] + self.dx * np.arange(self.nx)
        y = self.origin[1] + self.dy * np.arange(self.ny)
        return np.meshgrid(x, y)


@dataclass
class Grid3D:
    """Cubic 3D grid: phi / speed / state of shape (nz, ny, nx), spacing h."""

    nx: int
    ny: int
    nz: int
    h: float
    origin: tuple
    phi: Any = field(repr=False)
    speed: Any = field(repr=False)
    state: Any = field(repr=False)

    ndim = 3

    @property
    def dx(self) -> float:
        return self.h

    @property
    def dy(self) -> float:
        return self.h

    @property
    def dz(self) -> float:
        return self.h

    @property
    def shape(self) -> tuple:
        return (self.nz, self.ny, self.nx)

    def in_bounds(self, i: int, j: int, k: int) -> bool:
        return 0 <= i < self.nx and 0 <= j < self.ny and 0 <= k < self.nz

    def cell_center(self, i: int, j: int, k: int) -> tuple:
        return (self.origin[0] + i * self.h, self.origin[1] + j * self.h, self.origin[2] + k * self.h)


@dataclass(frozen=True)
class BoundaryCondition:
    """Pinned source cells (E/grid.py:82-105); cells are CellIndex or CellIndex3D."""

    seeds: tuple

    def __post_init__(self):
        seen = set()
        norm = []
        for cell, value in self.seeds:
            cell = CellIndex(int(cell[0]), int(cell[1])) if len(cell) == 2 else \
                CellIndex3D(int(cell[0]), int(cell[1]), int(cell[2]))
            if not math.isfinite(value):
                raise ValueError(f"seed value for {cell} must be finite, got {value}")
            if cell in seen:
                raise ValueError(f"duplicate seed cell {cell}")
            seen.add(cell)
            norm.append((cell, float(value)))
        object.__setattr__(self, "seeds", tuple(norm))

    def __len__(self) -> int:
        return len(self.seeds)

    def merged_with(self, other: "BoundaryCondition") -> "BoundaryCondition":
        return BoundaryCondition(self.seeds + other.seeds)


def _speed_array(speed, shape, coords):
    if callable(speed):
        f = np.vectorize(speed, otypes=[np.float64])(*coords())
    else:
        f = np.asarray(speed, dtype=np.float64)
        if f.ndim == 0:
            f = np.full(shape, float(f))
    if f.shape != shape:
        raise ValueError(f"speed array shape {f.shape} does not match grid {shape}")
    if np.any(f < 0) or not np.all(np.isfinite(f)):
        raise ValueError("speed must be finite and non-negative everywhere")
    return f


def new_grid(nx: int, ny: int, dx: float, dy: float, origin=(0.0, 0.0),
             speed: float | np.ndarray | Callable = 1.0) -> Grid:
    """E/grid.py:108-144: phi = +inf, zero speed => Blocked, negative speed rejected."""
    if nx < 1 or ny < 1:
        raise ValueError(f"grid must have at least one cell, got {nx}x{ny}")
    if dx <= 0 or dy <= 0:
        raise ValueError(f"grid spacing must be positive, got dx={dx}, dy={dy}")

    def coords():
        x = origin[0] + dx * np.arange(nx)
        y = origin[1] + dy * np.arange(ny)
        return np.meshgrid(x, y)

    f = _speed_array(speed, (ny, nx), coords)
    phi = np.full((ny, nx), INF)
    state = np.full((ny, nx), CellState.FAR, dtype=np.uint8)
    state[f == 0.0] = CellState.BLOCKED
    return Grid(nx, ny, float(dx), float(dy), (float(origin[0]), float(origin[1])), phi, f.copy(), state)


def new_grid_3d(nx: int, ny: int, nz: int, h: float, origin=(0.0, 0.0, 0.0),
                speed: float | np.ndarray | Callable = 1.0) -> Grid3D:
    """3D analogue of new_grid: arrays of shape (nz, ny, nx), cubic spacing h."""
    if nx < 1 or ny < 1 or nz < 1:
        raise ValueError(f"grid must have at least one cell, got {nx}x{ny}x{nz}")
    if h <= 0:
        raise ValueError(f"grid spacing must be positive, got h={h}")

    def coords():
        z, y, x = np.meshgrid(origin[2] + h * np.arange(nz), origin[1] + h * np.arange(ny),
                              origin[0] + h * np.arange(nx), indexing="ij")
        return x, y, z

    f = _speed_array(speed, (nz, ny, nx), coords)
    phi = np.full((nz, ny, nx), INF)
    state = np.full((nz, ny, nx), CellState.FAR, dtype=np.uint8)
    state[f == 0.0] = CellState.BLOCKED
    return Grid3D(nx, ny, nz, float(h), tuple(float(o) for o in origin), phi, f.copy(), state)


def _state_at(grid, lin: list[int]) -> list[int]:
    st = grid.state
    if hasattr(st, "device") and not isinstance(st, np.ndarray):  # torch tensor
        import torch

        idx = torch.as_tensor(lin, dtype=torch.int64, device=st.device)
        return st.reshape(-1).index_select(0, idx).cpu().tolist()
    flat = np.asarray(st).reshape(-1)
    return [int(flat[c]) for c in lin]


def seed_linear(grid, bc) -> tuple[list[int], list[float]]:
    """Validate a boundary condition like apply_boundary (E/grid.py:199-211).

    Every seed is checked (non-empty, in bounds, not Blocked) before anything
    is written.  Returns the linear indices and values.
    """
    if len(bc) == 0:
        raise ValueError("boundary condition has no seeds")
    idx, val = [], []
    three = getattr(grid, "ndim", 2) == 3
    for cell, value in bc.seeds:
        if three:
            if len(cell) != 3:
                raise ValueError(f"3D grid needs (i, j, k) seed cells, got {cell}")
            i, j, k = (int(c) for c in cell)
            if not grid.in_bounds(i, j, k):
                raise ValueError(f"seed cell ({i}, {j}, {k}) is outside the {grid.nx}x{grid.ny}x{grid.nz} grid")
            idx.append((k * grid.ny + j) * grid.nx + i)
        else:
            i, j = int(cell[0]), int(cell[1])
            if not grid.in_bounds(i, j):
                raise ValueError(f"seed cell ({i}, {j}) is outside the {grid.nx}x{grid.ny} grid")
            idx.append(j * grid.nx + i)
        val.append(float(value))
    states = _state_at(grid, idx)
    for (cell, _), s in zip(bc.seeds, states):
        if s == CellState.BLOCKED:
            coords = ", ".join(str(int(c)) for c in cell)
            raise ValueError(f"seed cell ({coords}) is blocked (zero speed)")
    return idx, val


def seed_point(grid, cell, value: float) -> BoundaryCondition:
    """E/grid.py:158-165 (2D or 3D cell)."""
    if getattr(grid, "ndim", 2) == 3:
        i, j, k = (int(c) for c in cell)
        if not grid.in_bounds(i, j, k):
            raise ValueError(f"seed cell ({i}, {j}, {k}) is outside the grid")
        if _state_at(grid, [(k * grid.ny + j) * grid.nx + i])[0] == CellState.BLOCKED:
            raise ValueError(f"seed cell ({i}, {j}, {k}) is blocked (zero speed)")
        return BoundaryCondition(((CellIndex3D(i, j, k), float(value)),))
    i, j = int(cell[0]), int(cell[1])
    if not grid.in_bounds(i, j):
        raise ValueError(f"seed cell ({i}, {j}) is outside the {grid.nx}x{grid.ny} grid")
    if _state_at(grid, [j * grid.nx + i])[0] == CellState.BLOCKED:
        raise ValueError(f"seed cell ({i}, {j}) is blocked (zero speed)")
    return BoundaryCondition(((CellIndex(i, j), float(value)),))


def reset_field(grid) -> None:
    """E/grid.py:226-231: clear phi and solver state, keep speed and Blocked flags."""
    grid.phi.fill_(INF) if hasattr(grid.phi, "fill_") else grid.phi.fill(INF)
    st = grid.state
    keep = st == CellState.BLOCKED
    if hasattr(st, "fill_"):
        st.fill_(CellState.FAR)
    else:
        st.fill(CellState.FAR)
    st[keep] = CellState.BLOCKED
