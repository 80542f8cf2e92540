"""The TMA brick remedy engine (k_remedy_b, csrc/eik_remedy_tma.cuh) against the oracle and the
reference fixtures: E/ifim.py:164-218 bit for bit.  EIK_REMEDY=brick selects it (3D, single
device, nx * sizeof(real) a multiple of 16 bytes, grid at least one brick plus halo); every test
checks that it actually ran (eik_last_remedy_engine).

Covers ragged grids (nx not a multiple of 32, ny / nz not multiples of 8), grid-edge bricks (the
TMA zero fill replaced by +inf), blocked cells and several seeds, and re-runs the 3D golden /
oracle / full-size tests of the other modules under this engine."""
import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik
from oracle import cpu
from paper_2106_15869_b200 import _native
from test_gpu_fullsize import test_fullsize_composed_equals_oracle_digests  # noqa: F401
from test_gpu_parity import test_3d_golden_cases_bit_exact, test_3d_vs_oracle  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def brick_engine(monkeypatch):
    monkeypatch.setenv("EIK_REMEDY", "brick")
    yield


def _random_problem(rng):
    nz, ny = (int(v) for v in rng.integers(10, 41, 2))
    nx = int(rng.integers(18, 60)) * 2  # even: 16-byte rows for float64
    shape = (nz, ny, nx)
    kind = int(rng.integers(0, 3))
    if kind == 0:
        kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
        b = int(rng.integers(3, 9))
        F = np.where(((ii // b) + (jj // b) + (kk // b)) % 2 == 0, 1.0, float(rng.uniform(0.005, 0.1)))
    elif kind == 1:
        F = np.exp(rng.normal(0.0, 1.0, size=shape))
    else:
        F = rng.uniform(0.1, 10.0, size=shape)
    F[rng.random(shape) < rng.uniform(0.0, 0.2)] = 0.0
    free = np.flatnonzero(F.ravel() > 0)
    k = int(min(free.size, rng.integers(1, 5)))
    seeds = [int(c) for c in rng.choice(free, k, replace=False)]
    vals = [float(v) for v in rng.uniform(0.0, 2.0, k)] if rng.random() < 0.5 else [0.0] * k
    return shape, float(rng.uniform(0.3, 2.0)), F, seeds, vals


@pytest.mark.parametrize("chunk", range(4))
def test_random_ragged_grids_bit_exact(chunk):
    rng = np.random.default_rng(7100 + chunk)
    ran = 0
    for _ in range(6):
        shape, h, F, seeds, vals = _random_problem(rng)
        nz, ny, nx = shape
        state = np.where(F == 0, 4, 0).astype(np.uint8)  # speed 0 = blocked (E/grid.py:21-26)
        ref = cpu.solve_ifim(shape, h, F, seeds, vals, state=state)
        g = eik.Grid3D(nx, ny, nz, h, (0.0, 0.0, 0.0), np.full(shape, np.inf), F.copy(), state.copy())
        bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v)
                                         for c, v in zip(seeds, vals)))
        res = eik.solve_ifim(g, bc)
        if res.stats.peak_remedy:
            assert _native.last_remedy_engine() == "brick"
            ran += 1
        assert np.array_equal(res.phi.view(np.uint64), ref.phi.view(np.uint64)), shape
        s, o = res.stats, ref.stats
        assert (s.iterations, s.solver_calls, s.peak_active, s.peak_remedy, s.phi_writes) == (
            o["iterations"], o["solver_calls"], o["peak_active"], o["peak_remedy"], o["phi_writes"]), shape
        assert list(s.active_history) == list(ref.active_history)
    assert ran > 0


def test_staged_remedy_uses_the_brick_engine():
    """build_remedy_set -> ifim_remedy_step (E/ifim.py:137-218) on a device grid: RunStats of the
    staged remedy equal the oracle's."""
    n = 48
    kk, jj, ii = np.mgrid[0:n, 0:n, 0:n]
    F = np.where(((ii // 6) + (jj // 6) + (kk // 6)) % 2 == 0, 1.0, 0.02)
    dev = torch.device("cuda:0")
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), float("inf"), dtype=torch.float64, device=dev),
                   torch.as_tensor(F, device=dev), torch.zeros((n, n, n), dtype=torch.uint8, device=dev))
    bc = eik.seed_point(g, eik.CellIndex3D(n // 2, n // 2, n // 2), 0.0)
    eik.ifim_update_step(g, bc)
    phi = g.phi.cpu().numpy().ravel().copy()
    state = g.state.cpu().numpy().ravel().copy()
    member, _ = cpu.build_remedy((n, n, n), 1.0, phi, F.ravel(), state)
    want = cpu.remedy_step((n, n, n), 1.0, phi, F.ravel(), state, member)
    remedy, _ = eik.build_remedy_set(g)
    got = eik.ifim_remedy_step(g, remedy)
    assert _native.last_remedy_engine() == "brick"
    assert (got.iterations, got.solver_calls, got.peak_remedy, got.phi_writes) == (
        want["iterations"], want["solver_calls"], want["peak_remedy"], want["phi_writes"])
    assert np.array_equal(g.phi.cpu().numpy().ravel().view(np.uint64), phi.view(np.uint64))


def test_ineligible_grids_fall_back_to_the_list_engine():
    """Odd nx (rows not 16-byte multiples) cannot be TMA-staged: the member-list engine runs."""
    shape = (12, 12, 37)
    F = np.where(np.arange(np.prod(shape)).reshape(shape) % 5 == 0, 0.05, 1.0)
    ref = cpu.solve_ifim(shape, 1.0, F, [7], [0.0])
    g = eik.Grid3D(37, 12, 12, 1.0, (0.0, 0.0, 0.0), np.full(shape, np.inf), F.copy(), np.zeros(shape, np.uint8))
    res = eik.solve_ifim(g, eik.seed_point(g, eik.CellIndex3D(7, 0, 0), 0.0))
    assert res.stats.peak_remedy > 0 and _native.last_remedy_engine() == "list"
    assert np.array_equal(res.phi.view(np.uint64), ref.phi.view(np.uint64))
