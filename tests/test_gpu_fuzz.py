"""Randomised parity net: 60 small random problems (2D uniform / anisotropic, 3D; ragged
shapes, blocked cells, several seeds with non-zero values, wide speed ranges) solved by the GPU
engine and the CPU oracle must agree bit for bit in phi, state and every statistic.  FIM too."""
import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik
from oracle import cpu

pytestmark = pytest.mark.gpu


def _problem(rng):
    dim = int(rng.choice([2, 3]))
    if dim == 2:
        ny, nx = (int(v) for v in rng.integers(1, 70, 2))
        shape = (ny, nx)
        spacing = (float(rng.uniform(0.2, 2.0)), float(rng.uniform(0.2, 2.0))) if rng.random() < 0.5 else (0.5, 0.5)
    else:
        shape = tuple(int(v) for v in rng.integers(1, 28, 3))
        spacing = float(rng.uniform(0.2, 2.0))
    kind = int(rng.integers(0, 3))
    if kind == 0:
        F = np.exp(rng.normal(0.0, 1.0, size=shape))
    elif kind == 1:
        F = np.where(rng.random(shape) < 0.5, 1.0, float(rng.uniform(0.005, 0.2)))
    else:
        F = rng.uniform(0.1, 10.0, size=shape)
    F[rng.random(shape) < rng.uniform(0.0, 0.3)] = 0.0
    free = np.flatnonzero(F.ravel() > 0)
    if free.size == 0:
        F.ravel()[0] = 1.0
        free = np.array([0])
    k = int(min(free.size, rng.integers(1, 6)))
    seeds = [int(c) for c in rng.choice(free, k, replace=False)]
    vals = [float(v) for v in rng.uniform(0.0, 2.0, k)] if rng.random() < 0.5 else [0.0] * k
    return shape, spacing, F, seeds, vals


def _grid(shape, spacing, F, state):
    if len(shape) == 2:
        ny, nx = shape
        return eik.Grid(nx, ny, spacing[0], spacing[1], (0.0, 0.0), np.full(shape, np.inf), F.copy(), state.copy())
    nz, ny, nx = shape
    return eik.Grid3D(nx, ny, nz, spacing, (0.0, 0.0, 0.0), np.full(shape, np.inf), F.copy(), state.copy())


def _bc(shape, seeds, vals):
    if len(shape) == 2:
        nx = shape[1]
        return eik.BoundaryCondition(tuple((eik.CellIndex(c % nx, c // nx), v) for c, v in zip(seeds, vals)))
    ny, nx = shape[1], shape[2]
    return eik.BoundaryCondition(tuple((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v)
                                       for c, v in zip(seeds, vals)))


@pytest.mark.parametrize("chunk", range(6))
def test_random_problems_bit_exact(chunk):
    rng = np.random.default_rng(1000 + chunk)
    for _ in range(10):
        shape, spacing, F, seeds, vals = _problem(rng)
        state = np.where(F == 0, 4, 0).astype(np.uint8)
        ref = cpu.solve_ifim(shape, spacing, F, seeds, vals, state=state, threads=1)
        g = _grid(shape, spacing, F, state)
        res = eik.solve_ifim(g, _bc(shape, seeds, vals))
        assert np.array_equal(np.asarray(res.phi).view(np.uint64), ref.phi.view(np.uint64)), (shape, spacing)
        assert np.array_equal(g.state, ref.state)
        st = res.stats
        assert (st.iterations, st.solver_calls, st.peak_active, st.peak_remedy, st.phi_writes) == (
            ref.stats["iterations"], ref.stats["solver_calls"], ref.stats["peak_active"], ref.stats["peak_remedy"],
            ref.stats["phi_writes"]), (shape, spacing)
        assert st.active_history == ref.active_history
        fr = cpu.solve_fim(shape, spacing, F, seeds, vals, state=state)
        g2 = _grid(shape, spacing, F, state)
        fg = eik.solve_fim(g2, _bc(shape, seeds, vals))
        assert np.array_equal(np.asarray(fg.phi).view(np.uint64), fr.phi.view(np.uint64)), (shape, spacing)
        assert (fg.stats.iterations, fg.stats.solver_calls, fg.stats.peak_active) == (
            fr.stats["iterations"], fr.stats["solver_calls"], fr.stats["peak_active"])


def test_random_3d_problems_peer_slabs():
    """Random 3D problems through the multi-rank peer-slab kernels (R ranks emulated on one GPU)."""
    from paper_2106_15869_b200.slab_peer import solve_emulated

    rng = np.random.default_rng(77)
    done = 0
    while done < 12:
        shape, spacing, F, seeds, vals = _problem(rng)
        if len(shape) != 3 or shape[0] < 2:
            continue
        state = np.where(F == 0, 4, 0).astype(np.uint8)
        R = int(rng.integers(1, min(shape[0], 6) + 1))
        ref = cpu.solve_ifim(shape, spacing, F, seeds, vals, state=state, threads=1)
        dev = torch.device("cuda:0")
        phi, st, state_out = solve_emulated(shape, spacing, torch.as_tensor(F, device=dev),
                                            torch.as_tensor(state, device=dev), list(zip(seeds, vals)), R)
        assert np.array_equal(phi.cpu().numpy().view(np.uint64), ref.phi.view(np.uint64)), (shape, R)
        assert (st.solver_calls, st.iterations, st.peak_remedy) == (
            ref.stats["solver_calls"], ref.stats["iterations"], ref.stats["peak_remedy"]), (shape, R)
        assert st.active_history == ref.active_history
        done += 1
