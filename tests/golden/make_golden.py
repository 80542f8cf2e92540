"""Generate the golden fixtures under tests/golden/ from the LIVE reference.

Run in the authoring container only (the GPU box has no /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

What it writes (all small, committed):

* ``cases2d.npz`` + ``cases2d.json`` -- 2D engine cases solved by the reference
  ``eikonal.ifim`` (E/ifim.py:75-235): inputs (speed, state, seeds, spacing),
  the final phi, the phase-by-phase RunStats integers and active_history.
  Includes make_example 1..5 (E/harness.py:77-118), the cfg1 analogue, the
  slow-pocket test field (T/test_ifim.py:43-58), a checkerboard, a sinusoid
  with several point seeds, an anisotropic grid (dx != dy) and walls.
* ``staged2d.npz`` -- the staged-API cases of T/test_ifim.py:79-126 (a single
  stale cell repaired from a converged field; all-seeded grid).
* ``local_solver.npz`` -- the 100k-sample generator of
  T/test_acceptance.py:149-161 (rng 20260815), first 16384 samples, with the
  reference outputs of update_2d_uniform / update_2d_aniso /
  update_3d_uniform (E/local_solver.py:39-157), plus the sha256 of all 100k
  3D outputs.
* ``fim2d.json`` / ``fim3d.json`` (+ ``.npz`` phi) -- FIM (E/fim.py:62-144, SURVEY.md
  §8f rank 3) on the inputs of cases2d / cases3d: the reference ``solve_fim`` in 2D,
  ``fim3d_py`` (a literal 3D generalisation calling ``update_3d_uniform``) in 3D.
* ``cases3d.npz`` + ``cases3d.json`` -- 3D engine cases.  The reference has no
  3D engine, so these come from ``ifim3d_py`` below: a literal
  3D generalisation of E/ifim.py that calls the reference's own scalar
  ``update_3d_uniform`` for every local solve.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from eikonal.grid import BoundaryCondition, CellIndex, CellState, new_grid, seed_point  # noqa: E402
from eikonal.fim import solve_fim  # noqa: E402
from eikonal.harness import field_sha256, make_example  # noqa: E402
from eikonal.ifim import build_remedy_set, ifim_remedy_step, ifim_update_step  # noqa: E402
from eikonal.local_solver import update_2d_aniso, update_2d_uniform, update_3d_uniform  # noqa: E402

INF = float("inf")


def _seeds_arrays(grid, bc):
    idx = np.array([c.linear(grid.nx) for c, _ in bc.seeds], dtype=np.int64)
    val = np.array([v for _, v in bc.seeds], dtype=np.float64)
    return idx, val


def solve_staged_2d(grid, bc):
    """solve_ifim (E/ifim.py:221-235) with the phase stats kept separately."""
    speed = grid.speed.copy()
    state0 = grid.state.copy()
    phi0 = grid.phi.copy()
    up = ifim_update_step(grid, bc)
    phi_after_update = grid.phi.copy()
    remedy, build_calls = build_remedy_set(grid)
    remedy_size = len(remedy)
    member0 = remedy.member.copy()
    rm = ifim_remedy_step(grid, remedy)
    return dict(
        speed=speed, state0=state0, phi0=phi0, phi=grid.phi.copy(), phi_update=phi_after_update,
        member0=member0,
        stats=dict(
            upd_iterations=up.iterations, upd_calls=up.solver_calls, peak_active=up.peak_active,
            build_calls=build_calls, remedy_size=remedy_size,
            rem_iterations=rm.iterations, rem_calls=rm.solver_calls, peak_remedy=rm.peak_remedy,
            iterations=up.iterations + rm.iterations,
            solver_calls=up.solver_calls + build_calls + rm.solver_calls,
            active_history=list(up.active_history),
            sha256=field_sha256(grid.phi), sha256_update=field_sha256(phi_after_update),
        ),
    )


def cases_2d():
    out = {}
    for ex in (1, 2, 3, 4, 5):
        for n in (32, 48, 64):
            g, bc = make_example(ex, n)
            out[f"ex{ex}_{n}"] = (g, bc)
    # cfg1 analogue: 2D 256^2, F=1, centre point (BASELINE.json configs[0])
    g = new_grid(256, 256, 1.0, 1.0)
    out["cfg1_256"] = (g, seed_point(g, CellIndex(128, 128), 0.0))
    # slow pocket (T/test_ifim.py:43-58)
    sp = np.ones((24, 24))
    sp[8:16, 8:16] = 0.05
    g = new_grid(24, 24, 1.0, 1.0, speed=sp)
    out["pocket_24"] = (g, seed_point(g, CellIndex(0, 0), 0.0))
    # checkerboard 1:100, 8-cell blocks (SURVEY.md Appendix B generator, smaller blocks)
    n = 64
    jj, ii = np.mgrid[0:n, 0:n]
    F = np.where(((ii // 8) + (jj // 8)) % 2 == 0, 1.0, 0.01)
    g = new_grid(n, n, 1.0, 1.0, speed=F)
    out["checker_64"] = (g, seed_point(g, CellIndex(n // 2, n // 2), 0.0))
    # cfg2 analogue: sinusoid on [0,1]^2 with 4 point seeds
    for n in (64, 96):
        h = 1 / (n - 1)
        x = h * np.arange(n)
        xx, yy = np.meshgrid(x, x)
        g = new_grid(n, n, h, h, origin=(0.0, 0.0), speed=1 + 0.5 * np.sin(2 * np.pi * xx) * np.sin(2 * np.pi * yy))
        cells = set()
        rng = np.random.default_rng(1)
        while len(cells) < 4:
            cells.add(tuple(int(v) for v in rng.integers(0, n, 2)))
        bc = BoundaryCondition(tuple((CellIndex(i, j), 0.0) for i, j in sorted(cells)))
        out[f"sinus_{n}"] = (g, bc)
    # anisotropic spacing (E/_kernels.py:61-88 path), rectangular grid, random speed
    rng = np.random.default_rng(7)
    F = rng.uniform(0.2, 2.0, size=(37, 53))
    F[10:12, 5:40] = 0.0  # a wall (Blocked)
    g = new_grid(53, 37, 0.7, 1.3, speed=F)
    out["aniso_53x37"] = (g, BoundaryCondition(((CellIndex(3, 3), 0.0), (CellIndex(40, 30), 1.5))))
    # ragged, tiny, 1-wide
    g = new_grid(1, 17, 1.0, 1.0)
    out["line_1x17"] = (g, seed_point(g, CellIndex(0, 5), 0.0))
    g = new_grid(33, 1, 0.5, 0.5)
    out["line_33x1"] = (g, seed_point(g, CellIndex(20, 0), 0.25))
    g = new_grid(3, 3, 1.0, 1.0)
    out["three_3x3"] = (g, seed_point(g, CellIndex(1, 1), 0.0))
    # sealed pocket: blocked ring leaves unreachable +inf cells (E/ifim.py:140-142)
    F = np.ones((20, 40))
    F[5, 5:15] = 0.0
    F[14, 5:15] = 0.0
    F[5:15, 5] = 0.0
    F[5:15, 14] = 0.0
    g = new_grid(40, 20, 1.0, 1.0, speed=F)
    out["sealed_40x20"] = (g, seed_point(g, CellIndex(30, 10), 0.0))
    return out


def write_cases_2d():
    arrays = {}
    meta = {}
    for name, (g, bc) in cases_2d().items():
        idx, val = _seeds_arrays(g, bc)
        r = solve_staged_2d(g, bc)
        keep_phi = g.nx * g.ny <= 64 * 96
        arrays[f"{name}__speed"] = r["speed"]
        arrays[f"{name}__state0"] = r["state0"]
        arrays[f"{name}__seed_idx"] = idx
        arrays[f"{name}__seed_val"] = val
        if keep_phi:
            arrays[f"{name}__phi"] = r["phi"]
            arrays[f"{name}__phi_update"] = r["phi_update"]
            arrays[f"{name}__member0"] = r["member0"]
        meta[name] = dict(nx=g.nx, ny=g.ny, dx=g.dx, dy=g.dy, has_phi=keep_phi, **r["stats"])
        print(name, meta[name]["iterations"], meta[name]["solver_calls"], meta[name]["peak_active"],
              meta[name]["peak_remedy"], meta[name]["sha256"][:16])
    np.savez_compressed(os.path.join(HERE, "cases2d.npz"), **arrays)
    with open(os.path.join(HERE, "cases2d.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def write_staged_2d():
    from eikonal.oracle import solve_fixpoint

    arrays = {}
    # T/test_ifim.py:86-97 -- converged field, one cell corrupted upward, rebuilt and repaired
    g, bc = make_example(1, 32)
    from eikonal.ifim import solve_ifim

    solve_ifim(g, bc)
    g.phi[20, 14] += 0.3
    arrays["stale_phi_in"] = g.phi.copy()
    arrays["stale_state"] = g.state.copy()
    arrays["stale_speed"] = g.speed.copy()
    remedy, calls = build_remedy_set(g)
    arrays["stale_member"] = remedy.member.copy()
    arrays["stale_build_calls"] = np.array([calls])
    rm = ifim_remedy_step(g, remedy)
    arrays["stale_phi_out"] = g.phi.copy()
    arrays["stale_rem_stats"] = np.array([rm.iterations, rm.solver_calls, rm.peak_remedy])
    arrays["stale_dx"] = np.array([g.dx])
    # fixpoint reference field for the same example (E/oracle.py:22-70)
    g2, bc2 = make_example(1, 32)
    arrays["stale_fixpoint"] = solve_fixpoint(g2, bc2).phi
    np.savez_compressed(os.path.join(HERE, "staged2d.npz"), **arrays)


def write_local_solver():
    # generator of T/test_acceptance.py:149-161
    rng = np.random.default_rng(20260815)
    count = 100_000
    mag = 10.0 ** rng.uniform(-3.0, 6.0, size=count)
    base = rng.uniform(-1.0, 1.0, size=count) * mag
    off1 = rng.uniform(-2.0, 2.0, size=count) * mag * 10.0 ** rng.uniform(-12.0, 0.0, size=count)
    off2 = rng.uniform(-2.0, 2.0, size=count) * mag * 10.0 ** rng.uniform(-12.0, 0.0, size=count)
    inf1 = rng.random(count) < 0.12
    inf2 = rng.random(count) < 0.12
    speeds = 10.0 ** rng.uniform(-3.0, 3.0, size=count)
    dxs = 10.0 ** rng.uniform(-3.0, 2.0, size=count)
    dys = 10.0 ** rng.uniform(-3.0, 2.0, size=count)
    a = base.copy()
    b = np.where(inf1, INF, base + off1)
    c = np.where(inf2, INF, base + off2)
    u2 = np.empty(count)
    a2 = np.empty(count)
    u3 = np.empty(count)
    u3p = np.empty(count)
    for k in range(count):
        u2[k] = update_2d_uniform(float(a[k]), float(b[k]), float(speeds[k]), float(dxs[k]))
        a2[k] = update_2d_aniso(float(a[k]), float(b[k]), float(speeds[k]), float(dxs[k]), float(dys[k]))
        u3[k] = update_3d_uniform(float(a[k]), float(b[k]), float(c[k]), float(speeds[k]), float(dxs[k]))
        # a permuted call with the third axis first: exercises the sort
        u3p[k] = update_3d_uniform(float(c[k]), float(a[k]), float(b[k]), float(speeds[k]), float(dxs[k]))
    # near-tie inputs that walk the 3D branch state machine (spread ~ delta)
    rng2 = np.random.default_rng(99)
    m = 16384
    ta = rng2.uniform(0, 10, m)
    tb = ta + rng2.uniform(0, 1.5, m) * rng2.choice([1.0, 0.5, 0.0], m)
    tc = ta + rng2.uniform(0, 1.5, m)
    tf = 10.0 ** rng2.uniform(-1, 1, m)
    td = rng2.uniform(0.5, 1.5, m)
    t3 = np.array([update_3d_uniform(float(x), float(y), float(z), float(f), float(d))
                   for x, y, z, f, d in zip(ta, tb, tc, tf, td)])
    keep = 16384
    np.savez_compressed(
        os.path.join(HERE, "local_solver.npz"),
        a=a[:keep], b=b[:keep], c=c[:keep], f=speeds[:keep], dx=dxs[:keep], dy=dys[:keep],
        u2=u2[:keep], a2=a2[:keep], u3=u3[:keep], u3p=u3p[:keep],
        sha_u3_all=np.frombuffer(hashlib.sha256(u3.tobytes()).digest(), dtype=np.uint8),
        sha_u2_all=np.frombuffer(hashlib.sha256(u2.tobytes()).digest(), dtype=np.uint8),
        sha_a2_all=np.frombuffer(hashlib.sha256(a2.tobytes()).digest(), dtype=np.uint8),
        ta=ta, tb=tb, tc=tc, tf=tf, td=td, t3=t3,
    )


# ---------------------------------------------------------------------------
# 3D: literal generalisation of E/ifim.py using the reference's update_3d_uniform
# ---------------------------------------------------------------------------

_FAR, _ACTIVE, _CONVERGED = 0, 1, 2


def _nbrs3(idx, nx, ny, nz):
    i = idx % nx
    r = idx // nx
    j = r % ny
    k = r // ny
    if i > 0:
        yield idx - 1
    if i < nx - 1:
        yield idx + 1
    if j > 0:
        yield idx - nx
    if j < ny - 1:
        yield idx + nx
    if k > 0:
        yield idx - nx * ny
    if k < nz - 1:
        yield idx + nx * ny


def _value3(phi, speed, c, nx, ny, nz, h):
    # padded snapshot reads (E/_kernels.py:21-38) with a z axis
    i = c % nx
    r = c // nx
    j = r % ny
    k = r // ny
    w = phi[c - 1] if i > 0 else INF
    e = phi[c + 1] if i < nx - 1 else INF
    s = phi[c - nx] if j > 0 else INF
    n = phi[c + nx] if j < ny - 1 else INF
    d = phi[c - nx * ny] if k > 0 else INF
    u = phi[c + nx * ny] if k < nz - 1 else INF
    return update_3d_uniform(min(w, e), min(s, n), min(d, u), float(speed[c]), h)


def ifim3d_py(nx, ny, nz, h, speed, state, seeds, tol=1e-12):
    """E/ifim.py:75-235 in 3D. speed/state flat arrays; seeds = [(linear, value)]."""
    n = nx * ny * nz
    phi = np.full(n, INF)
    state = state.copy()
    # apply_boundary (E/grid.py:199-215)
    for c, v in seeds:
        phi[c] = v
        state[c] = CellState.SOURCE
    blocked = state == CellState.BLOCKED
    seed = state == CellState.SOURCE
    label = np.zeros(n, dtype=np.uint8)
    active = []
    for c, _ in seeds:
        for nb in _nbrs3(c, nx, ny, nz):
            if not blocked[nb] and not seed[nb] and label[nb] == _FAR:
                label[nb] = _ACTIVE
                active.append(nb)
    hist = []
    upd_calls = 0
    peak_active = len(active)
    it = 0
    cap = 40 * (nx + ny + nz)
    while active:
        it += 1
        assert it <= cap
        hist.append(len(active))
        snap = phi.copy()
        values = [_value3(snap, speed, c, nx, ny, nz, h) for c in active]
        upd_calls += len(active)
        surv = []
        for c, v in zip(active, values):
            old = phi[c]
            if v == old or abs(v - old) <= tol:
                label[c] = _CONVERGED
                for nb in _nbrs3(c, nx, ny, nz):
                    if phi[nb] == INF and not blocked[nb] and label[nb] == _FAR:
                        label[nb] = _ACTIVE
                        surv.append(nb)
            else:
                phi[c] = v
                surv.append(c)
        active = surv
        peak_active = max(peak_active, len(active))
    phi_update = phi.copy()
    # build_remedy_set (E/ifim.py:137-161)
    free = ~blocked & ~seed
    cells = np.flatnonzero(free)
    snap = phi.copy()
    vals = np.array([_value3(snap, speed, c, nx, ny, nz, h) for c in cells])
    with np.errstate(invalid="ignore"):
        moved = np.abs(vals - phi[cells]) > tol
    member = np.zeros(n, dtype=bool)
    member[cells[moved]] = True
    rcells = [int(c) for c in cells[moved]]
    remedy_size = len(rcells)
    member0 = member.copy()
    build_calls = len(cells)
    # ifim_remedy_step (E/ifim.py:164-218)
    rem_calls = 0
    peak_remedy = len(rcells)
    rit = 0
    rcap = 20 * (nx + ny + nz)
    while rcells:
        rit += 1
        assert rit <= rcap
        snap = phi.copy()
        values = [_value3(snap, speed, c, nx, ny, nz, h) for c in rcells]
        rem_calls += len(rcells)
        surv = []
        dec = []
        for c, v in zip(rcells, values):
            if v < phi[c] - tol:
                phi[c] = v
                dec.append(c)
                surv.append(c)
            else:
                member[c] = False
        for c in dec:
            for nb in _nbrs3(c, nx, ny, nz):
                if not member[nb] and not blocked[nb] and not seed[nb]:
                    member[nb] = True
                    surv.append(nb)
        rcells = surv
        peak_remedy = max(peak_remedy, len(rcells))
    stats = dict(
        upd_iterations=it, upd_calls=upd_calls, peak_active=peak_active, build_calls=build_calls,
        remedy_size=remedy_size, rem_iterations=rit, rem_calls=rem_calls, peak_remedy=peak_remedy,
        iterations=it + rit, solver_calls=upd_calls + build_calls + rem_calls, active_history=hist,
        sha256=hashlib.sha256(phi.tobytes()).hexdigest(),
        sha256_update=hashlib.sha256(phi_update.tobytes()).hexdigest(),
    )
    return phi, phi_update, member0, state, stats


def cases_3d():
    out = {}
    # constant speed, centre seed
    n = 12
    out["const_12"] = (n, n, n, 1.0, np.ones(n ** 3), [((6 * n + 6) * n + 6, 0.0)])
    # constant speed, several random seeds (cfg3 family)
    rng = np.random.default_rng(2106)
    n = 14
    picks = set()
    while len(picks) < 4:
        picks.add(int(rng.integers(0, n ** 3)))
    out["multi_14"] = (n, n, n, 1.0, np.ones(n ** 3), [(c, 0.0) for c in sorted(picks)])
    # checkerboard 1:100 (cfg4 family), 4-cell blocks
    n = 16
    kk, jj, ii = np.mgrid[0:n, 0:n, 0:n]
    F = np.where(((ii // 4) + (jj // 4) + (kk // 4)) % 2 == 0, 1.0, 0.01).ravel()
    out["checker_16"] = (n, n, n, 1.0, F, [((8 * n + 8) * n + 8, 0.0)])
    # smooth random speed + obstacles, non-cubic box (cfg5 family)
    nx, ny, nz = 13, 11, 9
    rng = np.random.default_rng(5)
    kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
    g = np.sin(0.7 * ii + 0.3) * np.cos(0.5 * jj) + 0.5 * np.sin(0.9 * kk + 1.0)
    F = np.exp(0.5 * g)
    F[4, 2:9, 3:10] = 0.0  # a slab wall with a gap ring
    F = F.ravel()
    out["smooth_13x11x9"] = (nx, ny, nz, 0.5, F, [(0, 0.0), (nx * ny * nz - 1, 0.3)])
    return out


def write_cases_3d():
    arrays = {}
    meta = {}
    for name, (nx, ny, nz, h, F, seeds) in cases_3d().items():
        F = np.asarray(F, dtype=np.float64)
        state = np.where(F == 0.0, CellState.BLOCKED, CellState.FAR).astype(np.uint8)
        phi, phi_u, member0, _st, stats = ifim3d_py(nx, ny, nz, h, F, state, seeds)
        arrays[f"{name}__speed"] = F
        arrays[f"{name}__state0"] = state
        arrays[f"{name}__seed_idx"] = np.array([c for c, _ in seeds], dtype=np.int64)
        arrays[f"{name}__seed_val"] = np.array([v for _, v in seeds], dtype=np.float64)
        arrays[f"{name}__phi"] = phi
        arrays[f"{name}__phi_update"] = phi_u
        arrays[f"{name}__member0"] = member0
        meta[name] = dict(nx=nx, ny=ny, nz=nz, h=h, **stats)
        print(name, stats["iterations"], stats["solver_calls"], stats["peak_active"], stats["peak_remedy"])
    np.savez_compressed(os.path.join(HERE, "cases3d.npz"), **arrays)
    with open(os.path.join(HERE, "cases3d.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def fim3d_py(nx, ny, nz, h, speed, state, seeds, tol=1e-12):
    """E/fim.py:62-144 in 3D (six neighbours, update_3d_uniform). Returns (phi, stats)."""
    n = nx * ny * nz
    phi = np.full(n, INF)
    state = state.copy()
    for c, v in seeds:
        phi[c] = v
        state[c] = CellState.SOURCE
    blocked = state == CellState.BLOCKED
    seed = state == CellState.SOURCE
    FAR, ACT, SET = 0, 1, 2
    label = np.zeros(n, dtype=np.uint8)
    active = []
    for c, _ in seeds:
        for nb in _nbrs3(c, nx, ny, nz):
            if not blocked[nb] and not seed[nb] and label[nb] == FAR:
                label[nb] = ACT
                active.append(nb)
    it, calls, peak = 0, 0, len(active)
    cap = 40 * (nx + ny + nz)
    while active:
        it += 1
        assert it <= cap
        snap = phi.copy()
        values = [_value3(snap, speed, c, nx, ny, nz, h) for c in active]
        calls += len(active)
        surv = []
        for c, v in zip(active, values):
            old = phi[c]
            if v == old or abs(v - old) <= tol:
                label[c] = SET
            else:
                phi[c] = v
                surv.append(c)
        check = []
        for c in active:
            for nb in _nbrs3(c, nx, ny, nz):
                if blocked[nb] or seed[nb] or label[nb] == ACT:
                    continue
                if phi[nb] == INF:
                    label[nb] = ACT
                    surv.append(nb)
                else:
                    check.append(nb)
        active = surv
        if check:
            snap = phi.copy()
            values = [_value3(snap, speed, c, nx, ny, nz, h) for c in check]
            calls += len(check)
            for c, v in zip(check, values):
                if label[c] == ACT:
                    continue
                if v < phi[c] - tol:
                    phi[c] = v
                    label[c] = ACT
                    active.append(c)
        peak = max(peak, len(active))
    return phi, dict(iterations=it, solver_calls=calls, peak_active=peak,
                     sha256=hashlib.sha256(phi.tobytes()).hexdigest())


def write_fim():
    meta2, arr2 = {}, {}
    for name, (g, bc) in cases_2d().items():
        r = solve_fim(g, bc)
        st = r.stats
        meta2[name] = dict(iterations=st.iterations, solver_calls=st.solver_calls, peak_active=st.peak_active,
                           sha256=field_sha256(r.phi))
        if g.nx * g.ny <= 64 * 96:
            arr2[f"{name}__phi"] = r.phi
        print("fim", name, st.iterations, st.solver_calls, st.peak_active)
    np.savez_compressed(os.path.join(HERE, "fim2d.npz"), **arr2)
    with open(os.path.join(HERE, "fim2d.json"), "w") as fh:
        json.dump(meta2, fh, indent=1, sort_keys=True)
    meta3, arr3 = {}, {}
    for name, (nx, ny, nz, h, F, seeds) in cases_3d().items():
        F = np.asarray(F, dtype=np.float64)
        state = np.where(F == 0.0, CellState.BLOCKED, CellState.FAR).astype(np.uint8)
        phi, st = fim3d_py(nx, ny, nz, h, F, state, seeds)
        meta3[name] = st
        arr3[f"{name}__phi"] = phi
        print("fim3d", name, st["iterations"], st["solver_calls"], st["peak_active"])
    np.savez_compressed(os.path.join(HERE, "fim3d.npz"), **arr3)
    with open(os.path.join(HERE, "fim3d.json"), "w") as fh:
        json.dump(meta3, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["fim"]:
        write_fim()
        sys.exit(0)
    write_local_solver()
    write_staged_2d()
    write_cases_2d()
    write_cases_3d()
    write_fim()
