"""The CPU oracle (oracle/eik_oracle.c) pinned to golden vectors from the live
reference (tests/golden/make_golden.py).  CPU only."""
import hashlib
import os

import numpy as np
import pytest

from oracle import cpu

REF_SRC = "/root/reference/pkg/src"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_local_solvers_bitwise_vs_reference(local_vectors):
    """T/test_local_solver.py:170-188 + T/test_acceptance.py:149-194 generator."""
    L = local_vectors
    assert np.array_equal(bits(cpu.local_2d_uniform(L["a"], L["b"], L["f"], L["dx"])), bits(L["u2"]))
    assert np.array_equal(bits(cpu.local_2d_aniso(L["a"], L["b"], L["f"], L["dx"], L["dy"])), bits(L["a2"]))
    assert np.array_equal(bits(cpu.local_3d_uniform(L["a"], L["b"], L["c"], L["f"], L["dx"])), bits(L["u3"]))
    assert np.array_equal(bits(cpu.local_3d_uniform(L["c"], L["a"], L["b"], L["f"], L["dx"])), bits(L["u3p"]))
    # near-tie branch-walk vectors
    assert np.array_equal(bits(cpu.local_3d_uniform(L["ta"], L["tb"], L["tc"], L["tf"], L["td"])), bits(L["t3"]))


def test_local_solver_closed_forms():
    """T/test_local_solver.py:55-87."""
    lib = cpu.lib()
    assert abs(lib.orc_update_2d_uniform(0.0, 0.0, 1.0, 1.0) - 1 / np.sqrt(2)) < 1e-15
    assert abs(lib.orc_update_2d_aniso(0.0, 0.0, 1.0, 1.0, 2.0) - 2 / np.sqrt(5)) < 1e-15
    assert abs(lib.orc_update_3d_uniform(0.0, 0.0, 0.0, 1.0, 1.0) - 1 / np.sqrt(3)) < 1e-15
    assert abs(lib.orc_update_3d_uniform(0.0, 0.0, 1.0, 1.0, 1.0) - 1 / np.sqrt(2)) < 1e-15
    assert lib.orc_update_2d_uniform(0.0, np.inf, 2.0, 1.0) == 0.5
    assert lib.orc_update_3d_uniform(4.0, np.inf, np.inf, 1.0, 1.0) == 5.0
    assert lib.orc_update_3d_uniform(np.inf, np.inf, np.inf, 1.0, 1.0) == np.inf


@pytest.mark.parametrize("threads", [1, 4])
def test_2d_engine_matches_reference_golden(cases2d, threads):
    meta, Z = cases2d
    for name, m in meta.items():
        r = cpu.solve_ifim((m["ny"], m["nx"]), (m["dx"], m["dy"]), Z[name + "__speed"], Z[name + "__seed_idx"],
                           Z[name + "__seed_val"], state=Z[name + "__state0"], threads=threads)
        assert sha(r.phi) == m["sha256"], name
        s = r.stats
        assert (s["iterations"], s["solver_calls"], s["peak_active"], s["peak_remedy"]) == (
            m["iterations"], m["solver_calls"], m["peak_active"], m["peak_remedy"]), name
        assert r.active_history == m["active_history"], name
        assert r.phases["build"]["remedy_size"] == m["remedy_size"]
        assert r.phases["build"]["solver_calls"] == m["build_calls"]


@pytest.mark.parametrize("threads", [1, 4])
def test_3d_engine_matches_golden(cases3d, threads):
    meta, Z = cases3d
    for name, m in meta.items():
        r = cpu.solve_ifim((m["nz"], m["ny"], m["nx"]), m["h"], Z[name + "__speed"], Z[name + "__seed_idx"],
                           Z[name + "__seed_val"], state=Z[name + "__state0"], threads=threads)
        assert sha(r.phi) == m["sha256"], name
        assert r.stats["solver_calls"] == m["solver_calls"] and r.active_history == m["active_history"], name
        assert r.stats["peak_remedy"] == m["peak_remedy"], name


def test_staged_stale_cell(staged2d):
    """T/test_ifim.py:86-97 on the reference's own perturbed field."""
    Z = staged2d
    ny, nx = Z["stale_phi_in"].shape
    dx = float(Z["stale_dx"][0])
    phi = Z["stale_phi_in"].ravel().copy()
    speed = Z["stale_speed"].ravel().copy()
    state = Z["stale_state"].ravel().copy()
    member, b = cpu.build_remedy((ny, nx), (dx, dx), phi, speed, state)
    assert b["solver_calls"] == int(Z["stale_build_calls"][0])
    assert np.array_equal(member.astype(bool), Z["stale_member"].ravel())
    st = cpu.remedy_step((ny, nx), (dx, dx), phi, speed, state, member)
    assert [st["iterations"], st["solver_calls"], st["peak_remedy"]] == Z["stale_rem_stats"].tolist()
    assert np.array_equal(bits(phi), bits(Z["stale_phi_out"].ravel()))


def test_fixpoint_agrees_with_ifim(cases2d):
    """solve_fixpoint (E/oracle.py:22-70) vs solve_ifim within 1e-9 (T/test_ifim.py:23-30)."""
    meta, Z = cases2d
    for name in ("ex2_48", "ex3_48", "ex5_48", "pocket_24", "checker_64"):
        m = meta[name]
        shape, sp = (m["ny"], m["nx"]), (m["dx"], m["dy"])
        fx, _ = cpu.solve_fixpoint(shape, sp, Z[name + "__speed"], Z[name + "__seed_idx"], Z[name + "__seed_val"])
        r = cpu.solve_ifim(shape, sp, Z[name + "__speed"], Z[name + "__seed_idx"], Z[name + "__seed_val"])
        fin = np.isfinite(fx)
        assert np.array_equal(fin, np.isfinite(r.phi))
        assert np.max(np.abs(fx[fin] - r.phi[fin])) <= 1e-9, name


def test_3d_fixpoint_agreement():
    n = 20
    rng = np.random.default_rng(4)
    F = np.exp(0.4 * rng.standard_normal((n, n, n)))
    seeds = [int(c) for c in rng.choice(n ** 3, 3, replace=False)]
    fx, _ = cpu.solve_fixpoint((n, n, n), 1.0, F, seeds, [0.0] * 3)
    r = cpu.solve_ifim((n, n, n), 1.0, F, seeds, [0.0] * 3, threads=4)
    assert np.max(np.abs(fx - r.phi)) <= 1e-9


def test_cap_and_validation_errors():
    with pytest.raises(ValueError):
        cpu.solve_ifim((4, 4), (1.0, 1.0), np.ones(16), [0], [0.0], tol=0.0)
    F = np.ones(16)
    F[5] = 0.0
    with pytest.raises(ValueError):
        cpu.solve_ifim((4, 4), (1.0, 1.0), F, [5], [0.0])


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="live reference not mounted")
def test_oracle_vs_live_reference_random_grids():
    """Fresh random fields (not in the fixtures) against the live reference, when present."""
    import sys

    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from eikonal.grid import BoundaryCondition, CellIndex, new_grid
    from eikonal.ifim import solve_ifim

    rng = np.random.default_rng(123)
    for trial in range(3):
        ny, nx = rng.integers(8, 40, 2)
        F = rng.uniform(0.05, 3.0, (ny, nx))
        F[rng.random((ny, nx)) < 0.08] = 0.0
        free = np.flatnonzero(F.ravel() > 0)
        picks = rng.choice(free, 3, replace=False)
        dx, dy = (1.0, 1.0) if trial != 2 else (0.8, 1.1)
        g = new_grid(int(nx), int(ny), dx, dy, speed=F)
        bc = BoundaryCondition(tuple((CellIndex(int(c % nx), int(c // nx)), 0.1 * k) for k, c in enumerate(picks)))
        state0 = g.state.copy()
        ref = solve_ifim(g, bc)
        r = cpu.solve_ifim((int(ny), int(nx)), (dx, dy), F, picks, [0.1 * k for k in range(3)], state=state0)
        assert np.array_equal(bits(r.phi), bits(ref.phi))
        assert r.stats["solver_calls"] == ref.stats.solver_calls
        assert r.active_history == ref.stats.active_history


def test_fim_2d_matches_reference_golden(cases2d, fim2d):
    """orc_solve_fim (E/fim.py:62-144) vs the live reference solve_fim on the cases2d inputs."""
    meta, Z = cases2d
    fmeta, FZ = fim2d
    for name, m in meta.items():
        r = cpu.solve_fim((m["ny"], m["nx"]), (m["dx"], m["dy"]), Z[name + "__speed"], Z[name + "__seed_idx"],
                          Z[name + "__seed_val"], state=Z[name + "__state0"])
        f = fmeta[name]
        assert sha(r.phi) == f["sha256"], name
        assert (r.stats["iterations"], r.stats["solver_calls"], r.stats["peak_active"]) == (
            f["iterations"], f["solver_calls"], f["peak_active"]), name


def test_fim_3d_matches_golden(cases3d, fim3d):
    meta, Z = cases3d
    fmeta, FZ = fim3d
    for name, m in meta.items():
        r = cpu.solve_fim((m["nz"], m["ny"], m["nx"]), m["h"], Z[name + "__speed"], Z[name + "__seed_idx"],
                          Z[name + "__seed_val"], state=Z[name + "__state0"])
        f = fmeta[name]
        assert sha(r.phi) == f["sha256"], name
        assert (r.stats["iterations"], r.stats["solver_calls"], r.stats["peak_active"]) == (
            f["iterations"], f["solver_calls"], f["peak_active"]), name


def test_fim_and_ifim_agree_on_the_fixpoint(cases2d):
    """T/test_fim.py:18-24: FIM and iFIM both reach the fixpoint field (within 1e-9)."""
    meta, Z = cases2d
    for name in ("ex2_48", "ex5_48", "pocket_24", "checker_64"):
        m = meta[name]
        args = ((m["ny"], m["nx"]), (m["dx"], m["dy"]), Z[name + "__speed"], Z[name + "__seed_idx"],
                Z[name + "__seed_val"])
        a = cpu.solve_fim(*args, state=Z[name + "__state0"]).phi
        b = cpu.solve_ifim(*args, state=Z[name + "__state0"]).phi
        fin = np.isfinite(b)
        assert np.array_equal(np.isfinite(a), fin)
        assert np.abs(a[fin] - b[fin]).max() <= 1e-9, name
