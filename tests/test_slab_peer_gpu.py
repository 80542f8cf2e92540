"""Peer-memory slabs (the multi-GPU kernels) emulated on one GPU: R ranks as CTA
groups of one cooperative launch, neighbour planes read through device
pointers.  Bit-identical to the single-device solve and to the oracle."""
import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik
from oracle import cpu
from paper_2106_15869_b200.slab_peer import solve_emulated

pytestmark = pytest.mark.gpu


def problem(kind):
    rng = np.random.default_rng(5)
    if kind == "checker":
        nz, ny, nx = 24, 20, 40
        kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
        F = np.where(((ii // 4) + (jj // 4) + (kk // 4)) % 2 == 0, 1.0, 0.01)
    elif kind == "walls":
        nz, ny, nx = 13, 16, 37
        kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
        F = np.exp(0.5 * np.sin(0.5 * ii) * np.cos(0.3 * jj + 0.2 * kk))
        F[6, 3:14, 2:30] = 0.0
        F[3, 0:10, 10:12] = 0.0
    else:
        nz, ny, nx = 20, 18, 33
        F = np.ones((nz, ny, nx))
    free = np.flatnonzero(F.ravel() > 0)
    seeds = [(int(c), float(v)) for c, v in zip(rng.choice(free, 4, replace=False), (0.0, 0.3, 0.0, 1.0))]
    state = np.where(F == 0, 4, 0).astype(np.uint8)
    return (nz, ny, nx), 0.5, F, state, seeds


@pytest.mark.parametrize("R", [1, 2, 3, 5])
@pytest.mark.parametrize("kind", ["checker", "walls", "const"])
def test_peer_slabs_bit_identical(R, kind):
    shape, h, F, state, seeds = problem(kind)
    ref = cpu.solve_ifim(shape, h, F, [c for c, _ in seeds], [v for _, v in seeds], state=state, threads=8)
    dev = torch.device("cuda:0")
    phi, st, state_out = solve_emulated(shape, h, torch.as_tensor(F, device=dev), torch.as_tensor(state, device=dev),
                                        seeds, R)
    assert np.array_equal(phi.cpu().numpy().view(np.uint64), ref.phi.view(np.uint64))
    assert (st.iterations, st.solver_calls, st.peak_active, st.peak_remedy) == (
        ref.stats["iterations"], ref.stats["solver_calls"], ref.stats["peak_active"], ref.stats["peak_remedy"])
    assert st.active_history == ref.active_history
    assert st.phi_writes == ref.stats["phi_writes"]
    assert np.array_equal(state_out.cpu().numpy(), ref.state)


@pytest.mark.slow
def test_peer_slabs_512_matches_single():
    n = 256
    k = torch.arange(n, device="cuda") // (n // 16)
    F = torch.where(((k[:, None, None] + k[None, :, None] + k[None, None, :]) % 2) == 0, torch.tensor(1.0, dtype=torch.float64), torch.tensor(0.01, dtype=torch.float64))
    state = torch.zeros((n, n, n), dtype=torch.uint8, device="cuda")
    c = n // 2
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=torch.float64, device="cuda"),
                   F, state.clone())
    single = eik.solve_ifim(g, eik.seed_point(g, (c, c, c), 0.0))
    phi, st, _ = solve_emulated((n, n, n), 1.0, F, state, [((c * n + c) * n + c, 0.0)], 4)
    assert torch.equal(phi, single.phi)
    assert st.solver_calls == single.stats.solver_calls and st.active_history == single.stats.active_history


def test_distributed_peer_slabs_symmetric_memory():
    """DistributedSlabs through torch symmetric memory under torchrun (1 rank per GPU present)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = torch.cuda.device_count()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        os.path.join(root, "tools", "peer_slab_check.py")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "bit-identical=True" in r.stdout


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_solve_ifim_devices_kwarg(devices):
    """solve_ifim(..., devices=...) shards a Grid3D over z-slab ranks; several ranks on one
    device share a launch.  Field, state and stats equal the single-device solve."""
    shape, h, F, state, seeds = problem("walls")
    nz, ny, nx = shape
    bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v) for c, v in seeds))
    g1 = eik.new_grid_3d(nx, ny, nz, h, speed=F)
    ref = eik.solve_ifim(g1, bc)
    g2 = eik.new_grid_3d(nx, ny, nz, h, speed=F)
    res = eik.solve_ifim(g2, bc, devices=devices)
    assert np.array_equal(res.phi.view(np.uint64), ref.phi.view(np.uint64))
    assert np.array_equal(g2.phi.view(np.uint64), g1.phi.view(np.uint64)) and np.array_equal(g2.state, g1.state)
    a, b = res.stats, ref.stats
    assert (a.iterations, a.solver_calls, a.peak_active, a.peak_remedy, a.active_history) == \
        (b.iterations, b.solver_calls, b.peak_active, b.peak_remedy, b.active_history)


def test_devices_env_and_2d_rejected(monkeypatch):
    shape, h, F, state, seeds = problem("checker")
    nz, ny, nx = shape
    dev = torch.device("cuda:0")
    mk = lambda: eik.Grid3D(nx, ny, nz, h, (0.0, 0.0, 0.0), torch.full(shape, np.inf, dtype=torch.float64, device=dev),
                            torch.as_tensor(F, device=dev), torch.as_tensor(state, device=dev))
    bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v) for c, v in seeds))
    g1 = mk()
    ref = eik.solve_ifim(g1, bc)
    monkeypatch.setenv("EIKONAL_DEVICES", "0,0,0,0")
    g2 = mk()
    res = eik.solve_ifim(g2, bc)
    assert torch.equal(res.phi, ref.phi) and res.stats.solver_calls == ref.stats.solver_calls
    g2d = eik.new_grid(16, 16, 1.0, 1.0)
    with pytest.raises(ValueError, match="3D"):
        eik.solve_ifim(g2d, eik.seed_point(g2d, (3, 3), 0.0))
