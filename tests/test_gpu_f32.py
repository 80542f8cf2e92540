"""float32 perf mode (libeik_ifim_f32.so): float32 phi/speed select the
float32 engine; its field must agree with the float64 (bit-exact) solve within max-rel 1e-5
over the reached cells, with the same reachability."""
import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik

pytestmark = pytest.mark.gpu
REL = 1e-5  # north_star: max-rel 1e-5 in fp32


def max_rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    fa, fb = np.isfinite(a), np.isfinite(b)
    assert np.array_equal(fa, fb)
    m = fa & (np.abs(b) > 0)
    return float((np.abs(a[m] - b[m]) / np.abs(b[m])).max()) if m.any() else 0.0


def grids3d(n, F, seeds, dtype):
    dev = torch.device("cuda:0")
    F = torch.as_tensor(F, device=dev)
    return eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=dtype, device=dev),
                      F.to(dtype), torch.zeros((n, n, n), dtype=torch.uint8, device=dev)), \
        eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in seeds))


@pytest.mark.parametrize("kind", ["checker", "const16", "smooth"])
def test_f32_matches_f64_3d(kind):
    n = 64
    rng = np.random.default_rng(2106)
    k, j, i = np.mgrid[0:n, 0:n, 0:n]
    if kind == "checker":
        F = np.where(((i // 8) + (j // 8) + (k // 8)) % 2 == 0, 1.0, 0.01)
        seeds = [(32, 32, 32)]
    elif kind == "const16":
        F = np.ones((n, n, n))
        seeds = [tuple(int(v) for v in rng.integers(0, n, 3)) for _ in range(16)]
    else:
        F = np.exp(0.5 * np.sin(0.2 * i) * np.cos(0.15 * j + 0.1 * k))
        seeds = [(5, 7, 9), (50, 40, 30)]
    g64, bc = grids3d(n, F, seeds, torch.float64)
    g32, _ = grids3d(n, F, seeds, torch.float32)
    r64 = eik.solve_ifim(g64, bc)
    r32 = eik.solve_ifim(g32, bc)
    assert r32.phi.dtype == torch.float32
    assert max_rel(r32.phi.cpu().numpy(), r64.phi.cpu().numpy()) <= REL
    assert torch.equal(g32.state, g64.state)


def test_f32_2d_sinusoid_host_numpy():
    n = 256
    x = (np.arange(n) + 0.5) / n
    F = 1.0 + 0.5 * np.sin(2 * np.pi * x)[None, :] * np.sin(2 * np.pi * x)[:, None]
    g64 = eik.new_grid(n, n, 1.0 / n, 1.0 / n, speed=F)
    g32 = eik.Grid(n, n, 1.0 / n, 1.0 / n, (0.0, 0.0), np.full((n, n), np.inf, dtype=np.float32), F.astype(np.float32),
                   g64.state.copy())
    bc = eik.BoundaryCondition((((40, 50), 0.0), ((200, 180), 0.0)))
    r64 = eik.solve_ifim(g64, bc)
    r32 = eik.solve_ifim(g32, bc)
    assert isinstance(r32.phi, np.ndarray) and r32.phi.dtype == np.float32
    assert max_rel(r32.phi, r64.phi) <= REL
    assert np.array_equal(g32.phi, r32.phi)


def test_f32_staged_equals_solve_and_fixpoint_agrees():
    n = 48
    k, j, i = np.mgrid[0:n, 0:n, 0:n]
    F = np.where(((i // 6) + (j // 6) + (k // 6)) % 2 == 0, 1.0, 0.05)
    g1, bc = grids3d(n, F, [(10, 20, 30)], torch.float32)
    g2, _ = grids3d(n, F, [(10, 20, 30)], torch.float32)
    full = eik.solve_ifim(g1, bc)
    up = eik.ifim_update_step(g2, bc)
    rs, calls = eik.build_remedy_set(g2)
    rem = eik.ifim_remedy_step(g2, rs)
    assert torch.equal(g2.phi, full.phi)
    assert up.solver_calls + calls + rem.solver_calls == full.stats.solver_calls
    g3, _ = grids3d(n, F, [(10, 20, 30)], torch.float32)
    fx = eik.solve_fixpoint(g3, bc)
    assert max_rel(fx.phi.cpu().numpy(), full.phi.cpu().numpy()) <= REL
    phimax = float(full.phi[torch.isfinite(full.phi)].max())
    assert eik.max_residual(g1) <= REL * phimax  # a few float32 ulps of the largest value


def test_f32_multi_device_rejected():
    g, bc = grids3d(16, np.ones((16, 16, 16)), [(3, 3, 3)], torch.float32)
    with pytest.raises(ValueError, match="float64"):
        eik.solve_ifim(g, bc, devices=[0, 0])
