"""Shortest paths over a solved travel-time field: the downstream consumer of phi
(E/pathplan.py:248-330) and the Example 4 barrier-map pipeline
(E/pathplan.py:173-214, E/harness.py:88-94, E/cli.py:154-187).

The field is solved on the GPU (``solve_ifim`` / ``run_method``).  The descent itself is a serial
walk of a few hundred fixed-length steps, so it runs on the host over one copy of phi and state,
as the survey prescribes; a CUDA grid is copied to the host once.

Semantics follow the reference walk exactly (same sampling, same candidate order and tie rule,
same float operation order), so a bit-identical phi gives a bit-identical polyline:

* node gradients never read across walls: central differences where both axis neighbours are
  usable, one-sided toward the usable side otherwise, zero for an isolated node or a bad node
  (blocked, or phi = +inf);
* values and gradients are bilinear samples over the usable corners with renormalised weights;
* each step tries the full gradient step, then its x and y projections (clamped to the domain),
  and keeps the lowest sampled value below the current one; the walk ends in a source cell.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .grid import CellIndex, CellState, Grid, new_grid, seed_point


def _host(a) -> np.ndarray:
    return a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)


# --------------------------------------------------------------------------- barrier maps

@dataclass
class BarrierMap:
    """Occupancy grid (E/pathplan.py:28-44): ``blocked[j, i]`` is True inside a barrier."""

    width: int
    height: int
    blocked: np.ndarray

    def __post_init__(self) -> None:
        if self.width < 1 or self.height < 1:
            raise ValueError(f"map dimensions must be >= 1, got {self.width}x{self.height}")
        if self.blocked.shape != (self.height, self.width):
            raise ValueError(f"blocked array shape {self.blocked.shape} does not match "
                             f"declared dimensions {self.height}x{self.width}")


def barrier_speed(bmap: BarrierMap) -> np.ndarray:
    """Speed 0 inside barriers, 1 elsewhere (E/pathplan.py:166-168)."""
    return np.where(bmap.blocked, 0.0, 1.0)


def synthetic_barrier_map(n: int) -> BarrierMap:
    """The bundled n x n two-wall map (E/pathplan.py:171-193): full-width walls at rows n/3 and
    2n/3 with staggered gaps [7n/16, 3n/4) and [n/8, 7n/16)."""
    if n < 16:
        raise ValueError(f"synthetic map needs n >= 16, got {n}")
    blocked = np.zeros((n, n), dtype=bool)
    for row, (g0, g1) in ((round(n / 3), (round(7 * n / 16), round(3 * n / 4))),
                          (round(2 * n / 3), (round(n / 8), round(7 * n / 16)))):
        blocked[row] = True
        blocked[row, g0:g1] = False
    return BarrierMap(width=n, height=n, blocked=blocked)


def synthetic_endpoints(n: int) -> tuple[CellIndex, CellIndex]:
    """(start, goal) of the synthetic map (E/pathplan.py:196-200)."""
    return CellIndex(round(5 * n / 8), round(n / 6)), CellIndex(round(n / 4), round(5 * n / 6))


# --------------------------------------------------------------------------- descent

@dataclass
class PathPolyline:
    """Steepest-descent path, query point first, source cell last (E/pathplan.py:203-215)."""

    points: list[tuple[float, float]]
    phi: list[float] = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.points)

    def to_csv(self, path: str) -> None:
        with open(path, "w", encoding="ascii") as fh:
            fh.writelines(f"{x!r},{y!r},{v!r}\n" for (x, y), v in zip(self.points, self.phi))


def _axis_gradient(work: np.ndarray, bad: np.ndarray, axis: int, h: float) -> np.ndarray:
    """d(work)/d(axis) at every node without reading across walls (E/pathplan.py:218-241)."""
    w = np.moveaxis(work, axis, 0)
    b = np.moveaxis(bad, axis, 0)
    lo = np.concatenate([w[:1], w[:-1]])  # edge-replicated neighbours
    hi = np.concatenate([w[1:], w[-1:]])
    blo = np.concatenate([np.ones_like(b[:1]), b[:-1]])  # outside the grid counts as bad
    bhi = np.concatenate([b[1:], np.ones_like(b[-1:])])
    central = (hi - lo) / (2.0 * h)
    one_hi = (hi - w) / h
    one_lo = (w - lo) / h
    g = np.where(blo, np.where(bhi, 0.0, one_hi), np.where(bhi, one_lo, central))
    g[b] = 0.0
    return np.moveaxis(g, 0, axis)


class _Surface:
    """Bilinear sampling of node arrays over the usable nodes (E/pathplan.py:244-271)."""

    def __init__(self, usable: np.ndarray, x0: float, y0: float, dx: float, dy: float):
        self.usable, self.x0, self.y0, self.dx, self.dy = usable, x0, y0, dx, dy
        self.ny, self.nx = usable.shape

    def __call__(self, arr: np.ndarray, x: float, y: float):
        u, v = (x - self.x0) / self.dx, (y - self.y0) / self.dy
        i0 = min(max(int(math.floor(u)), 0), self.nx - 2)
        j0 = min(max(int(math.floor(v)), 0), self.ny - 2)
        fu = min(max(u - i0, 0.0), 1.0)
        fv = min(max(v - j0, 0.0), 1.0)
        total = acc = 0.0
        # corner order and weight expressions fixed: the sums are bit-identical to the reference
        for jj, ii, wgt in ((j0, i0, (1 - fu) * (1 - fv)), (j0, i0 + 1, fu * (1 - fv)),
                            (j0 + 1, i0, (1 - fu) * fv), (j0 + 1, i0 + 1, fu * fv)):
            if self.usable[jj, ii]:
                total += wgt
                acc += wgt * arr[jj, ii]
        return float(acc / total) if total > 0.0 else None

    def cell(self, x: float, y: float) -> tuple[int, int]:
        i = min(max(int(round((x - self.x0) / self.dx)), 0), self.nx - 1)
        j = min(max(int(round((y - self.y0) / self.dy)), 0), self.ny - 1)
        return i, j


def gradient_descent_path(grid: Grid, start: tuple[float, float], step: float) -> PathPolyline:
    """Walk fixed-length steps down the interpolated travel time from ``start`` to a source cell
    (E/pathplan.py:274-330).  Raises ValueError for a bad step / start / unsolved field and
    RuntimeError when the descent stalls or exceeds its 4*(nx+ny)/step budget."""
    nx, ny = grid.nx, grid.ny
    if nx < 2 or ny < 2:
        raise ValueError("path extraction needs at least a 2x2 grid")
    if not 0 < step <= min(grid.dx, grid.dy):
        raise ValueError(f"step must be in (0, min(dx, dy)] = (0, {min(grid.dx, grid.dy)}], got {step}")
    phi = _host(grid.phi).astype(np.float64, copy=False)
    state = _host(grid.state)
    source = state == CellState.SOURCE
    if not source.any():
        raise ValueError("grid has no source cells to descend toward")
    bad = (state == CellState.BLOCKED) | ~np.isfinite(phi)
    if bad.all():
        raise ValueError("field has no finite values; solve the grid first")
    work = np.where(bad, 0.0, phi)
    gx = _axis_gradient(work, bad, 1, grid.dx)
    gy = _axis_gradient(work, bad, 0, grid.dy)
    x0, y0 = grid.origin
    surf = _Surface(~bad, x0, y0, grid.dx, grid.dy)

    x, y = float(start[0]), float(start[1])
    i, j = surf.cell(x, y)
    if abs(x - (x0 + i * grid.dx)) > grid.dx or abs(y - (y0 + j * grid.dy)) > grid.dy:
        raise ValueError(f"start point {start} lies outside the grid domain")
    if state[j, i] == CellState.BLOCKED:
        raise ValueError(f"start point {start} lies in a blocked cell ({i}, {j})")
    if not np.isfinite(phi[j, i]):
        raise ValueError(f"start point {start} lies in an unreached cell ({i}, {j})")

    xmax, ymax = x0 + (nx - 1) * grid.dx, y0 + (ny - 1) * grid.dy
    value = surf(work, x, y)
    path = PathPolyline(points=[(x, y)], phi=[value])
    budget = int(math.ceil(4 * (nx + ny) / step))
    for _ in range(budget):
        i, j = surf.cell(x, y)
        if source[j, i]:
            return path
        dvx, dvy = surf(gx, x, y), surf(gy, x, y)
        norm = math.hypot(dvx, dvy) if dvx is not None and dvy is not None else 0.0
        if not math.isfinite(norm) or norm == 0.0:
            raise RuntimeError(f"descent stalled at ({x}, {y}): vanishing gradient")
        mx, my = step * dvx / norm, step * dvy / norm
        best = None
        for cx, cy in ((x - mx, y - my), (x - mx, y), (x, y - my)):  # full step, then its projections
            cx, cy = min(max(cx, x0), xmax), min(max(cy, y0), ymax)
            ci, cj = surf.cell(cx, cy)
            if bad[cj, ci]:
                continue
            cv = surf(work, cx, cy)
            if cv is not None and cv < value and (best is None or cv < best[0]):
                best = (cv, cx, cy)
        if best is None:
            raise RuntimeError(f"descent stalled at ({x}, {y}): no step of length {step} decreases the value")
        value, x, y = best
        path.points.append((x, y))
        path.phi.append(value)
    raise RuntimeError(f"descent exceeded step budget of {budget} steps without reaching a source")


# --------------------------------------------------------------------------- Example 4 pipeline

def plan_path(bmap: BarrierMap, start: CellIndex, goal: CellIndex, step: float = 0.5, method: str = "ifim",
              device=None, tol: float = 1e-12):
    """Barrier map -> speed -> GPU solve from ``start`` -> descent from ``goal``'s centre
    (E/cli.py:154-187 ``plan``).  Returns (grid, SolverResult, PathPolyline)."""
    import torch

    from .harness import run_method

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    grid = new_grid(bmap.width, bmap.height, 1.0, 1.0, origin=(0.0, 0.0), speed=barrier_speed(bmap))
    grid.phi = torch.as_tensor(np.asarray(grid.phi), device=dev)
    grid.speed = torch.as_tensor(np.asarray(grid.speed), device=dev)
    grid.state = torch.as_tensor(np.asarray(grid.state), device=dev)
    result = run_method(method, grid, seed_point(grid, start, 0.0), tol=tol)
    return grid, result, gradient_descent_path(grid, grid.cell_center(goal.i, goal.j), step)
