"""GPU parity: the sm_100a engine (through the C ABI) against the golden fixtures
from the live reference and against the CPU oracle.  Bit-exact float64 phi and
equal RunStats integers (iterations, solver_calls, peak_active, peak_remedy,
active_history) are required everywhere."""
import hashlib
import os

import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik
from paper_2106_15869_b200 import _native
from oracle import cpu

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def grid2d(m, Z, name, on_device):
    g = eik.Grid(m["nx"], m["ny"], m["dx"], m["dy"], (0.0, 0.0), np.full((m["ny"], m["nx"]), np.inf),
                 Z[name + "__speed"].copy(), Z[name + "__state0"].copy())
    if on_device:
        g.phi, g.speed, g.state = (torch.as_tensor(a, device=DEV) for a in (g.phi, g.speed, g.state))
    return g


def bc_from(Z, name, nx, ny=None):
    seeds = []
    for c, v in zip(Z[name + "__seed_idx"].tolist(), Z[name + "__seed_val"].tolist()):
        if ny is None:
            seeds.append((eik.CellIndex(c % nx, c // nx), v))
        else:
            seeds.append((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v))
    return eik.BoundaryCondition(tuple(seeds))


def check_stats(stats, m):
    assert stats.iterations == m["iterations"]
    assert stats.solver_calls == m["solver_calls"]
    assert stats.peak_active == m["peak_active"]
    assert stats.peak_remedy == m["peak_remedy"]
    assert stats.active_history == m["active_history"]
    assert stats.solver_calls == sum(stats.active_history) + m["build_calls"] + m["rem_calls"]


@pytest.mark.parametrize("on_device", [False, True], ids=["host", "device"])
def test_2d_golden_cases_bit_exact(cases2d, on_device):
    meta, Z = cases2d
    for name, m in meta.items():
        g = grid2d(m, Z, name, on_device)
        res = eik.solve_ifim(g, bc_from(Z, name, m["nx"]))
        assert sha(res.phi) == m["sha256"], name
        assert sha(g.phi) == m["sha256"], name  # mutated in place
        check_stats(res.stats, m)
        st = g.state.cpu().numpy() if on_device else g.state
        assert np.count_nonzero(st == eik.CellState.SOURCE) == len(Z[name + "__seed_idx"])


def test_3d_golden_cases_bit_exact(cases3d):
    meta, Z = cases3d
    for name, m in meta.items():
        F = Z[name + "__speed"].reshape(m["nz"], m["ny"], m["nx"])
        g = eik.new_grid_3d(m["nx"], m["ny"], m["nz"], m["h"], speed=F)
        res = eik.solve_ifim(g, bc_from(Z, name, m["nx"], m["ny"]))
        assert sha(res.phi) == m["sha256"], name
        check_stats(res.stats, m)


def test_staged_api_matches_phases(cases2d):
    meta, Z = cases2d
    for name in ("ex2_48", "ex5_64", "pocket_24", "aniso_53x37", "sealed_40x20"):
        m = meta[name]
        g = grid2d(m, Z, name, True)
        up = eik.ifim_update_step(g, bc_from(Z, name, m["nx"]))
        assert up.iterations == m["upd_iterations"] and up.solver_calls == m["upd_calls"]
        assert up.peak_active == m["peak_active"] and up.active_history == m["active_history"]
        assert sha(g.phi) == m["sha256_update"]
        before = g.phi.clone()
        remedy, calls = eik.build_remedy_set(g)
        assert torch.equal(before, g.phi)  # T/test_ifim.py:61-66
        assert calls == m["build_calls"] and len(remedy) == m["remedy_size"]
        if name + "__member0" in Z:
            assert np.array_equal(remedy.member.cpu().numpy().ravel(), Z[name + "__member0"].ravel()), name
        rm = eik.ifim_remedy_step(g, remedy)
        assert rm.iterations == m["rem_iterations"] and rm.solver_calls == m["rem_calls"]
        assert rm.peak_remedy == m["peak_remedy"]
        assert len(remedy) == 0
        assert sha(g.phi) == m["sha256"]


def test_single_stale_cell_repaired(staged2d):
    """T/test_ifim.py:86-97 replayed on golden data from the reference."""
    Z = staged2d
    ny, nx = Z["stale_phi_in"].shape
    dx = float(Z["stale_dx"][0])
    g = eik.Grid(nx, ny, dx, dx, (-10.0, -10.0), Z["stale_phi_in"].copy(), Z["stale_speed"].copy(),
                 Z["stale_state"].copy())
    remedy, calls = eik.build_remedy_set(g)
    assert calls == int(Z["stale_build_calls"][0])
    assert np.array_equal(np.asarray(remedy.member).ravel(), Z["stale_member"].ravel())
    assert eik.CellIndex(14, 20).linear(nx) in set(remedy.cells)
    rm = eik.ifim_remedy_step(g, remedy)
    assert [rm.iterations, rm.solver_calls, rm.peak_remedy] == Z["stale_rem_stats"].tolist()
    assert np.array_equal(g.phi.view(np.uint64), Z["stale_phi_out"].view(np.uint64))
    assert eik.field_max_diff(g.phi, Z["stale_fixpoint"]) <= 1e-9


def test_user_built_remedy_set(staged2d):
    Z = staged2d
    ny, nx = Z["stale_phi_in"].shape
    dx = float(Z["stale_dx"][0])
    g = eik.Grid(nx, ny, dx, dx, (-10.0, -10.0), Z["stale_phi_in"].copy(), Z["stale_speed"].copy(),
                 Z["stale_state"].copy())
    member = Z["stale_member"].copy()
    rs = eik.RemedySet(member=member, cells=np.flatnonzero(member).tolist())
    rm = eik.ifim_remedy_step(g, rs)
    assert [rm.iterations, rm.solver_calls, rm.peak_remedy] == Z["stale_rem_stats"].tolist()
    assert np.array_equal(g.phi.view(np.uint64), Z["stale_phi_out"].view(np.uint64))
    assert len(rs) == 0 and not member.any()


@pytest.mark.gpu
def test_hand_built_remedy_sets_match_the_reference():
    """RemedySet(member) alone is empty; members outside ``cells`` are never relaxed or enqueued
    (E/ifim.py:64-72, :184-213); fixtures from the live reference (tests/golden/make_remedy_sets.py)."""
    Z = np.load(os.path.join(GOLDEN, "remedy_sets.npz"))

    def grid():
        return eik.Grid(24, 24, 1.0, 1.0, (0.0, 0.0), Z["phi_in"].copy(), Z["speed"].copy(), Z["state"].copy())

    g = grid()
    st = eik.ifim_remedy_step(g, eik.RemedySet(member=Z["member"].copy()))
    assert [st.iterations, st.solver_calls, st.peak_remedy] == Z["a_stats"].tolist()
    assert np.array_equal(g.phi.view(np.uint64), Z["a_phi"].view(np.uint64))
    g = grid()
    rs = eik.RemedySet(member=Z["member"].copy(), cells=Z["b_cells"].tolist())
    st = eik.ifim_remedy_step(g, rs)
    assert [st.iterations, st.solver_calls, st.peak_remedy] == Z["b_stats"].tolist()
    assert np.array_equal(g.phi.view(np.uint64), Z["b_phi"].view(np.uint64))
    assert np.array_equal(np.asarray(rs.member), Z["b_member_after"])
    g = grid()
    st = eik.ifim_remedy_step(g, eik.RemedySet(member=Z["member"].copy(), cells=np.flatnonzero(Z["member"]).tolist()))
    assert [st.iterations, st.solver_calls, st.peak_remedy] == Z["c_stats"].tolist()
    assert np.array_equal(g.phi.view(np.uint64), Z["c_phi"].view(np.uint64))


def test_local_solver_bitwise(local_vectors):
    """All 16,384 reference vectors (T/test_acceptance.py:149-161, per-vector spacing) and the
    near-tie 3D vectors through the GPU solvers: 2D uniform (kind 0) and the 3D walk upd3u
    (kind 2), bit for bit."""
    import ctypes as C

    L = local_vectors
    lib = _native.lib()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731

    def run(kind, a, b, c, f, dx):
        # per-element spacings (dx <= 0: the spacing of element i is passed in out[i])
        T = [torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64), device=DEV) for v in (a, b, c, f)]
        out = torch.as_tensor(np.ascontiguousarray(dx, dtype=np.float64), device=DEV).clone()
        _native.check(lib.eik_local_solve(kind, P(T[0]), P(T[1]), P(T[2]), P(T[3]), -1.0, 0.0, P(out), len(a), s))
        return out.cpu().numpy().view(np.uint64)

    n = len(L["a"])
    assert np.array_equal(run(0, L["a"], L["b"], L["c"], L["f"], L["dx"]), L["u2"][:n].view(np.uint64))
    assert np.array_equal(run(2, L["a"], L["b"], L["c"], L["f"], L["dx"]), L["u3"].view(np.uint64))
    assert np.array_equal(run(2, L["c"], L["a"], L["b"], L["f"], L["dx"]), L["u3p"].view(np.uint64))
    assert np.array_equal(run(2, L["ta"], L["tb"], L["tc"], L["tf"], L["td"]), L["t3"].view(np.uint64))


def test_local_solver_bitwise_batched():
    """Whole batches at fixed spacing vs the oracle (itself pinned to the reference)."""
    import ctypes as C

    rng = np.random.default_rng(11)
    n = 1 << 16
    a = rng.uniform(-50, 50, n)
    b = a + rng.uniform(-3, 3, n) * rng.choice([1.0, 1e-6, 0.0], n)
    c = a + rng.uniform(-3, 3, n)
    b[rng.random(n) < 0.1] = np.inf
    c[rng.random(n) < 0.1] = np.inf
    f = 10.0 ** rng.uniform(-2, 2, n)
    lib = _native.lib()
    T = {k: torch.as_tensor(v, device=DEV) for k, v in dict(a=a, b=b, c=c, f=f).items()}
    out = torch.empty_like(T["a"])
    P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for kind, dx, dy, ref in ((0, 0.7, 0.7, cpu.local_2d_uniform(a, b, f, 0.7)),
                              (1, 0.7, 1.3, cpu.local_2d_aniso(a, b, f, 0.7, 1.3)),
                              (2, 0.9, 0.9, cpu.local_3d_uniform(a, b, c, f, 0.9))):
        _native.check(lib.eik_local_solve(kind, P(T["a"]), P(T["b"]), P(T["c"]), P(T["f"]), dx, dy, P(out), n, s))
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64)), kind


def _checker3d(n, blk):
    kk, jj, ii = np.mgrid[0:n, 0:n, 0:n]
    return np.where(((ii // blk) + (jj // blk) + (kk // blk)) % 2 == 0, 1.0, 0.01)


@pytest.mark.parametrize("shape,kind", [((40, 40, 40), "checker"), ((33, 47, 29), "smooth"),
                                        ((64, 64, 64), "multi"), ((1, 1, 70), "line")])
def test_3d_vs_oracle(shape, kind):
    nz, ny, nx = shape
    rng = np.random.default_rng(3)
    if kind == "checker":
        F = _checker3d(nx, 5)
        seeds = [((nz // 2 * ny + ny // 2) * nx + nx // 2, 0.0)]
    elif kind == "smooth":
        kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
        F = np.exp(0.5 * np.sin(0.3 * ii) * np.cos(0.2 * jj + 0.1 * kk))
        F[10, 5:40, 3:20] = 0.0
        seeds = [(0, 0.0), (nx * ny * nz - 1, 2.5)]
    elif kind == "multi":
        F = np.ones(shape)
        seeds = [(int(c), 0.0) for c in rng.choice(nx * ny * nz, 16, replace=False)]
    else:
        F = np.ones(shape)
        seeds = [(10, 0.0)]
    h = 0.5
    g = eik.new_grid_3d(nx, ny, nz, h, speed=F)
    bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v) for c, v in seeds))
    res = eik.solve_ifim(g, bc)
    ref = cpu.solve_ifim(shape, h, F, [c for c, _ in seeds], [v for _, v in seeds], threads=8)
    assert np.array_equal(res.phi.view(np.uint64), ref.phi.view(np.uint64))
    s = res.stats
    assert (s.iterations, s.solver_calls, s.peak_active, s.peak_remedy) == (
        ref.stats["iterations"], ref.stats["solver_calls"], ref.stats["peak_active"], ref.stats["peak_remedy"])
    assert s.active_history == ref.active_history
    assert s.phi_writes == ref.stats["phi_writes"]


def test_2d_larger_vs_oracle():
    n = 300
    h = 1 / (n - 1)
    x = h * np.arange(n)
    xx, yy = np.meshgrid(x, x)
    F = 1 + 0.5 * np.sin(2 * np.pi * xx) * np.sin(2 * np.pi * yy)
    rng = np.random.default_rng(2106)
    cells = set()
    while len(cells) < 8:
        cells.add(tuple(int(v) for v in rng.integers(0, n, 2)))
    cells = sorted(cells)
    g = eik.new_grid(n, n, h, h, speed=F)
    res = eik.solve_ifim(g, eik.BoundaryCondition(tuple((eik.CellIndex(i, j), 0.0) for i, j in cells)))
    ref = cpu.solve_ifim((n, n), (h, h), F, [j * n + i for i, j in cells], [0.0] * len(cells), threads=8)
    assert np.array_equal(res.phi.view(np.uint64), ref.phi.view(np.uint64))
    assert res.stats.solver_calls == ref.stats["solver_calls"]
    assert res.stats.active_history == ref.active_history


def test_errors_match_reference():
    g = eik.new_grid(8, 8, 1.0, 1.0)
    with pytest.raises(ValueError):
        eik.solve_ifim(g, eik.seed_point(g, eik.CellIndex(0, 0), 0.0), tol=-1e-9)
    with pytest.raises(ValueError):
        eik.solve_ifim(g, eik.BoundaryCondition(()))
    F = np.ones((8, 8))
    F[2, 3] = 0.0
    g = eik.new_grid(8, 8, 1.0, 1.0, speed=F)
    with pytest.raises(ValueError):
        eik.solve_ifim(g, eik.BoundaryCondition(((eik.CellIndex(3, 2), 0.0),)))
    with pytest.raises(ValueError):
        eik.solve_ifim(g, eik.BoundaryCondition(((eik.CellIndex(9, 2), 0.0),)))
    assert np.isinf(g.phi).all()  # nothing written before validation


def test_all_seeded_zero_iterations():
    g = eik.new_grid(4, 4, 1.0, 1.0)
    bc = eik.BoundaryCondition(tuple((eik.CellIndex(i, j), 0.1 * (i + j)) for i in range(4) for j in range(4)))
    st = eik.ifim_update_step(g, bc)
    assert st.iterations == 0 and st.solver_calls == 0 and st.active_history == []
    res = eik.solve_ifim(eik.new_grid(4, 4, 1.0, 1.0), bc)
    assert res.stats.iterations == 0 and res.stats.solver_calls == 0


def test_repeat_solves_reuse_workspace():
    n = 64
    F = _checker3d(n, 8)
    outs = set()
    for _ in range(3):
        g = eik.new_grid_3d(n, n, n, 1.0, speed=F)
        res = eik.solve_ifim(g, eik.seed_point(g, (32, 32, 32), 0.0))
        outs.add((sha(res.phi), res.stats.solver_calls))
    assert len(outs) == 1


def test_host_grid_large_result_copy_is_independent():
    """Host grids >= 2^22 cells take the overlapped result copy (_HostResult): the caller's
    phi and SolverResult.phi both hold the solved field and do not alias."""
    n = 160
    k = np.arange(n) // 10
    F = np.where(((k[:, None, None] + k[None, :, None] + k[None, None, :]) % 2) == 0, 1.0, 0.01)
    for pinned in (False, True):
        phi = torch.full((n, n, n), np.inf, dtype=torch.float64)
        st = torch.zeros((n, n, n), dtype=torch.uint8)
        sp = torch.from_numpy(F)
        if pinned:
            phi, st, sp = phi.pin_memory(), st.pin_memory(), sp.pin_memory()
        g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), phi, sp, st)
        res = eik.solve_ifim(g, eik.seed_point(g, (80, 80, 80), 0.0))
        dev = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=torch.float64,
                                                                    device="cuda"),
                         torch.from_numpy(F).cuda(), torch.zeros((n, n, n), dtype=torch.uint8, device="cuda"))
        ref = eik.solve_ifim(dev, eik.seed_point(dev, (80, 80, 80), 0.0))
        assert torch.equal(res.phi, ref.phi.cpu()) and torch.equal(g.phi, ref.phi.cpu())
        assert res.phi.data_ptr() != g.phi.data_ptr()
        g.phi.fill_(0.0)
        assert torch.equal(res.phi, ref.phi.cpu())
    gn = eik.new_grid_3d(n, n, n, 1.0, speed=F)
    res = eik.solve_ifim(gn, eik.seed_point(gn, (80, 80, 80), 0.0))
    assert isinstance(res.phi, np.ndarray) and np.array_equal(res.phi, gn.phi) and not np.shares_memory(res.phi, gn.phi)
    assert np.array_equal(res.phi, ref.phi.cpu().numpy())


def _cfg2(n):
    """BASELINE.json configs[1]: 2D n^2 on [0,1]^2, F = 1 + 0.5 sin(2 pi x) sin(2 pi y)
    at the cell centres, 8 distinct random point seeds (rng 2106)."""
    h = 1 / (n - 1)
    x = h * np.arange(n)
    xx, yy = np.meshgrid(x, x)
    F = 1 + 0.5 * np.sin(2 * np.pi * xx) * np.sin(2 * np.pi * yy)
    rng = np.random.default_rng(2106)
    cells = []
    while len(cells) < 8:
        c = tuple(int(v) for v in rng.integers(0, n, 2))
        if c not in cells:
            cells.append(c)
    return h, F, cells


@pytest.mark.slow
def test_cfg2_1024_bit_exact_vs_oracle():
    n = 1024
    h, F, cells = _cfg2(n)
    g = eik.new_grid(n, n, h, h, speed=F)
    res = eik.solve_ifim(g, eik.BoundaryCondition(tuple((eik.CellIndex(i, j), 0.0) for i, j in cells)))
    ref = cpu.solve_ifim((n, n), (h, h), F, [j * n + i for i, j in cells], [0.0] * len(cells), threads=16)
    assert np.array_equal(res.phi.view(np.uint64), ref.phi.view(np.uint64))
    assert (res.stats.solver_calls, res.stats.iterations, res.stats.peak_remedy) == (
        ref.stats["solver_calls"], ref.stats["iterations"], ref.stats["peak_remedy"])
    assert res.stats.active_history == ref.active_history


@pytest.mark.slow
def test_cfg2_full_size_properties():
    """cfg2 at its full 4096^2: iFIM reaches the GPU fixpoint field and satisfies the equation."""
    n = 4096
    h, F, cells = _cfg2(n)
    dev = torch.device("cuda:0")
    mk = lambda: eik.Grid(n, n, h, h, (0.0, 0.0), torch.full((n, n), np.inf, dtype=torch.float64, device=dev),
                          torch.as_tensor(F, device=dev), torch.zeros((n, n), dtype=torch.uint8, device=dev))
    bc = eik.BoundaryCondition(tuple((eik.CellIndex(i, j), 0.0) for i, j in cells))
    g1, g2 = mk(), mk()
    a = eik.solve_ifim(g1, bc)
    b = eik.solve_fixpoint(g2, bc)
    assert eik.field_max_diff(a.phi, b.phi) <= 1e-9
    assert eik.max_residual(g1) <= 1e-9
    assert a.stats.peak_remedy > 0 and a.stats.solver_calls > n * n


def test_concurrent_solves_from_threads():
    """Concurrent calls on different grids are allowed: two threads solving
    same-shape grids at once get their own workspaces and the single-thread results."""
    import threading

    n = 48
    k = np.arange(n) // 6
    F1 = np.where(((k[:, None, None] + k[None, :, None] + k[None, None, :]) % 2) == 0, 1.0, 0.02)
    F2 = np.exp(0.3 * np.sin(np.arange(n)[None, None, :] * 0.3) * np.ones((n, n, n)))
    refs, outs, errs = [], [None, None], []
    for F in (F1, F2):
        g = eik.new_grid_3d(n, n, n, 1.0, speed=F)
        refs.append(eik.solve_ifim(g, eik.seed_point(g, (5, 9, 13), 0.0)).phi)

    def run(i, F):
        try:
            for _ in range(3):
                g = eik.new_grid_3d(n, n, n, 1.0, speed=F)
                outs[i] = eik.solve_ifim(g, eik.seed_point(g, (5, 9, 13), 0.0)).phi
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i, F)) for i, F in enumerate((F1, F2))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    for o, r in zip(outs, refs):
        assert np.array_equal(o.view(np.uint64), r.view(np.uint64))
