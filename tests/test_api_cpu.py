"""Host-side API semantics of the drop-in boundary (no GPU needed): grid and
boundary conventions mirror E/grid.py, validation happens before anything is
written, and the product path refuses to run without a CUDA device."""
import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik


def test_new_grid_conventions():
    """E/grid.py:108-144."""
    F = np.ones((3, 4))
    F[1, 2] = 0.0
    g = eik.new_grid(4, 3, 0.5, 0.25, origin=(1.0, 2.0), speed=F)
    assert g.shape == (3, 4) and g.phi.shape == (3, 4)
    assert np.isinf(g.phi).all()
    assert g.state[1, 2] == eik.CellState.BLOCKED and g.state[0, 0] == eik.CellState.FAR
    assert g.cell_center(2, 1) == (2.0, 2.25)
    assert eik.CellIndex(2, 1).linear(4) == 6
    with pytest.raises(ValueError):
        eik.new_grid(4, 3, 1.0, 1.0, speed=-np.ones((3, 4)))
    with pytest.raises(ValueError):
        eik.new_grid(4, 3, 0.0, 1.0)
    with pytest.raises(ValueError):
        eik.new_grid(4, 3, 1.0, 1.0, speed=np.ones((4, 3)))
    g = eik.new_grid(5, 4, 1.0, 1.0, speed=lambda x, y: x + y + 1.0)
    assert g.speed[3, 4] == 8.0


def test_new_grid_3d_conventions():
    F = np.ones((2, 3, 4))
    F[1, 2, 3] = 0.0
    g = eik.new_grid_3d(4, 3, 2, 0.5, speed=F)
    assert g.shape == (2, 3, 4) and g.dx == g.dy == g.dz == 0.5
    assert g.state[1, 2, 3] == eik.CellState.BLOCKED
    assert eik.CellIndex3D(3, 2, 1).linear(4, 3) == 23
    g = eik.new_grid_3d(3, 3, 3, 1.0, speed=lambda x, y, z: 1.0 + z)
    assert g.speed[2, 0, 0] == 3.0


def test_boundary_condition_validation():
    """E/grid.py:82-105."""
    with pytest.raises(ValueError):
        eik.BoundaryCondition(((eik.CellIndex(0, 0), float("inf")),))
    with pytest.raises(ValueError):
        eik.BoundaryCondition(((eik.CellIndex(0, 0), 0.0), ((0, 0), 1.0)))
    bc = eik.BoundaryCondition((((1, 2), 0.5),)).merged_with(eik.BoundaryCondition((((3, 0), 0.0),)))
    assert len(bc) == 2 and bc.seeds[0][0] == eik.CellIndex(1, 2)
    bc3 = eik.BoundaryCondition((((1, 2, 3), 0.0),))
    assert isinstance(bc3.seeds[0][0], eik.CellIndex3D)


def test_seed_validation_happens_before_any_write():
    """apply_boundary validates every seed before writing (E/grid.py:204-215)."""
    F = np.ones((5, 5))
    F[2, 2] = 0.0
    g = eik.new_grid(5, 5, 1.0, 1.0, speed=F)
    with pytest.raises(ValueError):
        eik.seed_linear(g, eik.BoundaryCondition(()))
    with pytest.raises(ValueError):
        eik.seed_linear(g, eik.BoundaryCondition((((0, 0), 0.0), ((2, 2), 0.0))))
    with pytest.raises(ValueError):
        eik.seed_linear(g, eik.BoundaryCondition((((0, 0), 0.0), ((5, 0), 0.0))))
    assert np.isinf(g.phi).all()
    idx, val = eik.seed_linear(g, eik.BoundaryCondition((((1, 3), 0.25),)))
    assert idx == [16] and val == [0.25]
    with pytest.raises(ValueError):
        eik.seed_point(g, (2, 2), 0.0)
    g3 = eik.new_grid_3d(3, 4, 5, 1.0)
    assert eik.seed_linear(g3, eik.seed_point(g3, (2, 3, 4), 1.0)) == ([59], [1.0])


def test_resolve_workers():
    """E/parallel.py:28-42."""
    assert eik.resolve_workers(3) == 3
    assert eik.resolve_workers(0) >= 1
    with pytest.raises(ValueError):
        eik.resolve_workers(-1)


def test_run_method_dispatch():
    g = eik.new_grid(4, 4, 1.0, 1.0)
    with pytest.raises(ValueError):
        eik.run_method("fmm", g, eik.seed_point(g, (0, 0), 0.0))
    assert eik.METHOD_NAMES == ("fim", "ifim", "oracle")


def test_field_helpers_match_reference_semantics():
    """E/harness.py:165-179."""
    a = np.array([[0.0, np.inf], [1.0, 2.0]])
    b = np.array([[0.5, np.inf], [1.0, 1.0]])
    assert eik.field_max_diff(a, b) == 1.0
    assert eik.field_max_diff(torch.tensor(a), torch.tensor(a)) == 0.0
    with pytest.raises(ValueError):
        eik.field_max_diff(a, b[:1])
    import hashlib

    assert eik.field_sha256(a) == hashlib.sha256(a.tobytes()).hexdigest()


def test_tol_is_validated_first():
    g = eik.new_grid(8, 8, 1.0, 1.0)
    for fn in (lambda: eik.solve_ifim(g, eik.seed_point(g, (0, 0), 0.0), tol=-1e-9),
               lambda: eik.ifim_update_step(g, eik.seed_point(g, (0, 0), 0.0), tol=0.0),
               lambda: eik.build_remedy_set(g, tol=0.0),
               lambda: eik.ifim_remedy_step(g, eik.RemedySet(member=np.zeros(64, bool)), tol=-1.0)):
        with pytest.raises(ValueError):
            fn()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    g = eik.new_grid(8, 8, 1.0, 1.0)
    with pytest.raises(RuntimeError, match="CUDA"):
        eik.solve_ifim(g, eik.seed_point(g, (0, 0), 0.0))
    assert np.isinf(g.phi).all()


def test_remedy_set_host_side():
    """E/ifim.py:64-72: the work list is ``cells`` (default []), ``member`` only marks membership."""
    member = np.zeros(16, dtype=bool)
    member[[3, 7]] = True
    rs = eik.RemedySet(member=member)
    assert len(rs) == 0 and rs.cells == []
    rs2 = eik.RemedySet(member=member.copy(), cells=[3, 7])
    assert len(rs2) == 2
    rs2._drain()
    assert len(rs2) == 0 and not rs2.member.any()
    rs3 = eik.RemedySet(member=member.copy(), cells=[7])
    rs3._drain()
    assert rs3.member.tolist() == [i == 3 for i in range(16)]  # members outside the work list stay


def test_remedy_set_rejects_lists_the_set_engine_cannot_mirror():
    member = np.zeros(16, dtype=bool)
    member[[3, 7]] = True
    for cells in ([3, 3], [3, 5], [99]):
        with pytest.raises(ValueError):
            eik.RemedySet(member=member, cells=cells)._device_masks((16,), torch.device("cpu"))


def test_resolve_devices(monkeypatch):
    """devices= / EIKONAL_DEVICES selection for the multi-device z-slab solve."""
    from paper_2106_15869_b200.slab_peer import resolve_devices

    monkeypatch.delenv("EIKONAL_DEVICES", raising=False)
    assert resolve_devices(None) is None
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 4)
    assert resolve_devices(1) is None and resolve_devices([2]) is None
    assert resolve_devices(3) == [0, 1, 2]
    assert resolve_devices([1, 1, 3]) == [1, 1, 3]
    for bad in (0, 5, [0, 1, 0], [4], []):
        with pytest.raises(ValueError):
            resolve_devices(bad)
    monkeypatch.setenv("EIKONAL_DEVICES", "2")
    assert resolve_devices(None) == [0, 1]
    monkeypatch.setenv("EIKONAL_DEVICES", "0,0,2")
    assert resolve_devices(None) == [0, 0, 2]


def test_field_npy_round_trip_3d(tmp_path):
    """Binary snapshot for fields too large for CSV."""
    g = eik.new_grid_3d(7, 5, 4, 0.25, origin=(1.0, 2.0, 3.0))
    g.phi[:] = np.random.default_rng(2).random((4, 5, 7))
    g.phi[0, 0, 0] = np.inf
    p = str(tmp_path / "f.npy")
    eik.export_field_npy(g, p)
    h = eik.import_field_npy(p)
    assert isinstance(h, eik.Grid3D) and (h.nx, h.ny, h.nz, h.h, h.origin) == (7, 5, 4, 0.25, (1.0, 2.0, 3.0))
    assert np.array_equal(h.phi.view(np.uint64), g.phi.view(np.uint64)) and (h.state == 0).all()
    t = eik.Grid3D(7, 5, 4, 0.25, (0.0, 0.0, 0.0), torch.from_numpy(g.phi.copy()), torch.ones((4, 5, 7)),
                   torch.zeros((4, 5, 7), dtype=torch.uint8))
    eik.export_field_npy(t, p)
    assert np.array_equal(np.load(p).view(np.uint64), g.phi.view(np.uint64))


def test_result_split_accounts_every_byte(monkeypatch):
    """bench's e2e byte counts come from ifim._HostResult.result_split, which must mirror commit():
    every chunk of the result goes either by a second DMA or by a host copy."""
    from paper_2106_15869_b200.ifim import _HostResult

    n = 512 ** 3 * 8
    for frac, want_dma in (("0", 0), ("1", n), ("0.25", n // 4), ("0.5", n // 2)):
        monkeypatch.setenv("EIK_RESULT_DMA_FRAC", frac)
        dma, host = _HostResult.result_split(n, 8)
        assert dma + host == n and dma == want_dma, (frac, dma, host)
    monkeypatch.delenv("EIK_RESULT_DMA_FRAC")
    dma, host = _HostResult.result_split(1000 * 8, 8)  # one short chunk
    assert dma + host == 8000
