"""GPU FIM (E/fim.py:62-144) against the live reference's
golden fixtures (2D) and the 3D generalisation (tests/golden/fim*.json), and
against the CPU oracle on random problems: phi bytes and every statistic."""
import hashlib

import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik
from oracle import cpu

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_fim_2d_matches_reference(cases2d, fim2d):
    meta, Z = cases2d
    fmeta, _ = fim2d
    for name, m in meta.items():
        g = eik.Grid(m["nx"], m["ny"], m["dx"], m["dy"], (0.0, 0.0), np.full((m["ny"], m["nx"]), np.inf),
                     Z[name + "__speed"].copy(), Z[name + "__state0"].copy())
        nx = m["nx"]
        bc = eik.BoundaryCondition(tuple((eik.CellIndex(int(c) % nx, int(c) // nx), float(v))
                                         for c, v in zip(Z[name + "__seed_idx"], Z[name + "__seed_val"])))
        r = eik.run_method("fim", g, bc)
        f = fmeta[name]
        assert sha(r.phi) == f["sha256"], name
        assert (r.stats.iterations, r.stats.solver_calls, r.stats.peak_active) == (
            f["iterations"], f["solver_calls"], f["peak_active"]), name


def test_fim_3d_matches_golden(cases3d, fim3d):
    meta, Z = cases3d
    fmeta, _ = fim3d
    for name, m in meta.items():
        nx, ny, nz = m["nx"], m["ny"], m["nz"]
        dev = torch.device("cuda:0")
        g = eik.Grid3D(nx, ny, nz, m["h"], (0.0, 0.0, 0.0),
                       torch.full((nz, ny, nx), np.inf, dtype=torch.float64, device=dev),
                       torch.as_tensor(Z[name + "__speed"].reshape(nz, ny, nx), device=dev),
                       torch.as_tensor(Z[name + "__state0"].reshape(nz, ny, nx), device=dev))
        bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(int(c) % nx, (int(c) // nx) % ny, int(c) // (nx * ny)), float(v))
                                         for c, v in zip(Z[name + "__seed_idx"], Z[name + "__seed_val"])))
        r = eik.solve_fim(g, bc)
        f = fmeta[name]
        assert sha(r.phi.cpu().numpy()) == f["sha256"], name
        assert (r.stats.iterations, r.stats.solver_calls, r.stats.peak_active) == (
            f["iterations"], f["solver_calls"], f["peak_active"]), name


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_fim_vs_oracle_random_3d(seed):
    rng = np.random.default_rng(seed)
    nz, ny, nx = 20, 23, 37
    F = np.exp(rng.normal(0.0, 0.7, size=(nz, ny, nx)))
    F[rng.random((nz, ny, nx)) < 0.05] = 0.0
    free = np.flatnonzero(F.ravel() > 0)
    seeds = [int(c) for c in rng.choice(free, 3, replace=False)]
    state = np.where(F == 0, 4, 0).astype(np.uint8)
    ref = cpu.solve_fim((nz, ny, nx), 0.7, F, seeds, [0.0, 0.2, 0.5], state=state)
    g = eik.Grid3D(nx, ny, nz, 0.7, (0.0, 0.0, 0.0), np.full((nz, ny, nx), np.inf), F.copy(), state.copy())
    bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v)
                                     for c, v in zip(seeds, [0.0, 0.2, 0.5])))
    r = eik.solve_fim(g, bc)
    assert np.array_equal(np.asarray(r.phi).view(np.uint64), ref.phi.view(np.uint64))
    assert (r.stats.iterations, r.stats.solver_calls, r.stats.peak_active) == (
        ref.stats["iterations"], ref.stats["solver_calls"], ref.stats["peak_active"])
    assert r.stats.phi_writes == ref.stats["phi_writes"]


def test_fim_and_ifim_reach_the_same_field():
    """T/test_fim.py:18-24 / :69-80: both methods reach the fixpoint (1e-9)."""
    n = 96
    k = np.arange(n) // 12
    F = np.where(((k[:, None, None] + k[None, :, None] + k[None, None, :]) % 2) == 0, 1.0, 0.05)
    dev = torch.device("cuda:0")
    mk = lambda: eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=torch.float64, device=dev),
                            torch.as_tensor(F, device=dev), torch.zeros((n, n, n), dtype=torch.uint8, device=dev))
    g1, g2 = mk(), mk()
    bc = eik.seed_point(g1, (5, 60, 30), 0.0)
    a = eik.solve_fim(g1, bc)
    b = eik.solve_ifim(g2, bc)
    assert eik.field_max_diff(a.phi, b.phi) <= 1e-9
    assert eik.max_residual(g1) <= 1e-9


def test_fim_errors_and_trivial_cases():
    g = eik.new_grid(4, 4, 1.0, 1.0)
    with pytest.raises(ValueError):
        eik.solve_fim(g, eik.seed_point(g, (0, 0), 0.0), tol=0.0)
    bc = eik.BoundaryCondition(tuple((eik.CellIndex(i, j), 0.1 * (i + j)) for i in range(4) for j in range(4)))
    r = eik.solve_fim(g, bc)  # T/test_fim.py:43-51
    assert r.stats.iterations == 0 and r.stats.solver_calls == 0 and abs(r.phi[2, 3] - 0.5) < 1e-15
