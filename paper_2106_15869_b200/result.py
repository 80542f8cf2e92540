"""Solver output containers (E/result.py:9-27) with device-side extras."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any


@dataclass
class RunStats:
    # E/result.py:9-18, same names and meaning
    iterations: int = 0
    solver_calls: int = 0
    peak_active: int = 0
    peak_remedy: int = 0
    wall_time: float = 0.0
    active_history: list | None = None
    # extras measured by the B200 engine (not in the reference)
    phi_writes: int = 0
    phases: dict = field(default_factory=dict)
    device_ms: dict = field(default_factory=dict)
    gpu_launches: int = 0


@dataclass
class SolverResult:
    """E/result.py:21-27.  ``phi`` is a numpy array for host grids and a torch
    tensor for CUDA-resident grids."""

    phi: Any
    stats: RunStats
    accepted_order: Any = field(default=None, repr=False)
