"""Dispatch and parity helpers for the iFIM path (E/harness.py:54-57, 121-179).

``run_method`` keeps the reference's string dispatch (the plugin point every
CLI command goes through, E/harness.py:121-144).  "ifim", "fim" (the paper's
baseline, E/fim.py) and "oracle" (the fixpoint ground truth, E/oracle.py) are
served by this package; fmm and fsm are out of scope and raise
like an unknown method would.
"""
from __future__ import annotations

import hashlib

import numpy as np
import torch

from .fim import solve_fim
from .fixpoint import max_residual, solve_fixpoint  # noqa: F401  (re-exported)
from .ifim import solve_ifim
from .result import SolverResult

METHOD_NAMES = ("fim", "ifim", "oracle")
PARALLEL_METHODS = frozenset({"fim", "ifim", "oracle"})


def run_method(method: str, grid, bc, tol: float = 1e-12, workers: int = 1) -> SolverResult:
    """E/harness.py:121-144 restricted to the accelerated method."""
    if method == "fim":
        return solve_fim(grid, bc, tol=tol, workers=workers)
    if method == "ifim":
        return solve_ifim(grid, bc, tol=tol, workers=workers)
    if method == "oracle":
        return solve_fixpoint(grid, bc, tol=tol, workers=workers)
    raise ValueError(f"unknown method {method!r}, expected one of {METHOD_NAMES}")


def _np(a):
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def field_max_diff(a, b) -> float:
    """E/harness.py:165-174: max |a - b|, equal same-sign infinities count as 0."""
    a, b = _np(a), _np(b)
    if a.shape != b.shape:
        raise ValueError(f"field shapes differ: {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    with np.errstate(invalid="ignore"):
        diff = np.abs(a - b)
    return float(np.where(both_inf, 0.0, diff).max())


def field_sha256(phi) -> str:
    """E/harness.py:177-179: digest of the raw float64 bytes."""
    return hashlib.sha256(np.ascontiguousarray(_np(phi)).tobytes()).hexdigest()
