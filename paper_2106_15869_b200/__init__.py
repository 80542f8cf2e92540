"""B200-native iFIM (improved fast iterative method, arXiv 2106.15869).

Drop-in for the reference package's iFIM path (``eikonal.solve_ifim`` and the
staged ``ifim_update_step`` / ``build_remedy_set`` / ``ifim_remedy_step``),
with the reference's grid / speed / source / result conventions, extended to
3D cubic grids.  All solving happens in hand-written sm_100a CUDA kernels
behind the C ABI in include/eik_ifim.h; there is no CPU fallback.
"""
from .grid import (
    INF,
    BoundaryCondition,
    CellIndex,
    CellIndex3D,
    CellState,
    Grid,
    Grid3D,
    new_grid,
    new_grid_3d,
    reset_field,
    seed_linear,
    seed_point,
)
from .fieldio import export_field_npy, import_field_npy
from .fim import solve_fim
from .fixpoint import max_residual, solve_fixpoint
from .harness import METHOD_NAMES, PARALLEL_METHODS, field_digest, field_max_diff, field_sha256, run_method
from .ifim import (
    RemedySet,
    build_remedy_set,
    clear_workspaces,
    ifim_remedy_step,
    ifim_update_step,
    resolve_workers,
    solve_ifim,
)
from .pathplan import (
    BarrierMap,
    PathPolyline,
    barrier_speed,
    gradient_descent_path,
    plan_path,
    synthetic_barrier_map,
    synthetic_endpoints,
)
from .result import RunStats, SolverResult

__version__ = "0.1.0"

__all__ = [
    "INF", "BoundaryCondition", "CellIndex", "CellIndex3D", "CellState", "Grid", "Grid3D", "METHOD_NAMES",
    "PARALLEL_METHODS", "RemedySet", "RunStats", "SolverResult", "build_remedy_set", "clear_workspaces",
    "export_field_npy", "field_digest", "field_max_diff", "field_sha256", "import_field_npy", "ifim_remedy_step", "ifim_update_step", "new_grid", "new_grid_3d",
    "reset_field", "resolve_workers", "run_method", "seed_linear", "seed_point", "solve_fim", "solve_ifim", "solve_fixpoint",
    "max_residual", "BarrierMap", "PathPolyline", "barrier_speed", "gradient_descent_path", "plan_path",
    "synthetic_barrier_map", "synthetic_endpoints",
]
