"""Full-size parity for the BASELINE.json configs (E/ifim.py:221-235).

tests/golden/fullsize.json holds the oracle's digests of each config at the size BASELINE.json
names (cfg5 at 512^3), made by tests/golden/make_fullsize.py with oracle/eik_oracle.c (pinned to
the live reference by tests/test_oracle.py).  The GPU solve must reproduce every RunStats
integer, the active_history, the frozen set after the update step, the remedy set R_0 of the build
pass and the phi bytes -- staged (the three reference steps) and composed (solve_ifim).
"""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import bench
import paper_2106_15869_b200 as eik

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "fullsize.json")) as fh:
    DB = json.load(fh)
KEYS = [k for k in ("cfg1@256", "cfg3@256", "cfg2@4096", "cfg4@512", "cfg5@512") if k in DB]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make(rec):
    config, n = rec["config"], rec["n"]
    h, F, seeds = bench.workload_np(config, n)
    F = np.ascontiguousarray(F)
    assert sha(F) == rec["speed_sha256"], "speed field differs from the digested one"
    Fd = torch.as_tensor(F, device=DEV)
    phi = torch.full(F.shape, float("inf"), dtype=torch.float64, device=DEV)
    st = torch.zeros(F.shape, dtype=torch.uint8, device=DEV)
    if F.ndim == 2:
        g = eik.Grid(n, n, h, h, (0.0, 0.0), phi, Fd, st)
        bc = eik.BoundaryCondition(tuple((eik.CellIndex(i, j), 0.0) for i, j in seeds))
    else:
        g = eik.Grid3D(n, n, n, h, (0.0, 0.0, 0.0), phi, Fd, st)
        bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in seeds))
    return g, bc


@pytest.mark.slow
@pytest.mark.parametrize("key", KEYS)
def test_fullsize_staged_equals_oracle_digests(key):
    rec = DB[key]
    torch.cuda.empty_cache()
    g, bc = make(rec)
    up = eik.ifim_update_step(g, bc)
    u = rec["update"]
    assert (up.iterations, up.solver_calls, up.peak_active, up.phi_writes) == (
        u["iterations"], u["solver_calls"], u["peak_active"], u["phi_writes"])
    assert up.phases["update"]["converged"] == u["converged"] == u["frozen"]
    hist = np.asarray(up.active_history, dtype=np.int64)
    assert hist.size == u["history_len"] and sha(hist) == u["active_history_sha256"]
    free = (g.state != 4) & (g.state != 2)
    frozen = free & torch.isfinite(g.phi)
    assert int(frozen.sum()) == u["frozen"]
    assert eik.field_sha256(frozen.to(torch.uint8)) == u["frozen_sha256"]
    assert eik.field_sha256(g.phi) == u["phi_sha256"]
    remedy, calls = eik.build_remedy_set(g)
    b = rec["build"]
    assert (calls, len(remedy)) == (b["calls"], b["remedy_size"])
    assert eik.field_sha256(remedy._dev["mask"]) == b["member_sha256"]
    rm = eik.ifim_remedy_step(g, remedy)
    m = rec["remedy"]
    assert (rm.iterations, rm.solver_calls, rm.peak_remedy, rm.phi_writes) == (
        m["iterations"], m["solver_calls"], m["peak_remedy"], m["phi_writes"])
    assert eik.field_sha256(g.phi) == rec["phi_sha256"]
    del g, remedy
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("key", KEYS)
def test_fullsize_composed_equals_oracle_digests(key):
    rec = DB[key]
    torch.cuda.empty_cache()
    g, bc = make(rec)
    res = eik.solve_ifim(g, bc)
    s, want = res.stats, rec["stats"]
    assert (s.iterations, s.solver_calls, s.peak_active, s.peak_remedy, s.phi_writes) == (
        want["iterations"], want["solver_calls"], want["peak_active"], want["peak_remedy"], want["phi_writes"])
    assert sha(np.asarray(s.active_history, dtype=np.int64)) == rec["update"]["active_history_sha256"]
    assert eik.field_sha256(res.phi) == rec["phi_sha256"]
    assert int(torch.isfinite(res.phi).sum()) == rec["phi_finite"]
    del g, res
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_cfg5_1024_gpu_crosscheck_digest():
    """cfg5 at its BASELINE size (1024^3), where no oracle run exists: the composed solve (auto
    remedy engine) reproduces the digest that the member-list kernel, the TMA brick pipeline and
    the emulated two-rank peer-slab kernels agreed on (tests/golden/fullsize_gpu.json, made by
    tools/make_gpu_crosscheck.py): phi (chunked device SHA-256) and every RunStats integer."""
    from paper_2106_15869_b200.harness import field_digest

    with open(os.path.join(HERE, "golden", "fullsize_gpu.json")) as fh:
        rec = json.load(fh)["cfg5@1024"]
    w = bench.make_workload(torch, DEV, "cfg5", 1024)
    assert field_digest(w.F) == rec["speed_field_digest"]
    g = w.grid(eik, torch.full(w.shape, float("inf"), dtype=torch.float64, device=DEV), w.F,
               torch.zeros(w.shape, dtype=torch.uint8, device=DEV))
    res = eik.solve_ifim(g, w.bc(eik))
    s, ph = res.stats, res.stats.phases
    got = {"iterations": s.iterations, "solver_calls": s.solver_calls, "peak_active": s.peak_active,
           "peak_remedy": s.peak_remedy, "phi_writes": s.phi_writes, "upd_iterations": ph["update"]["iterations"],
           "rem_iterations": ph["remedy"]["iterations"], "remedy_size": ph["build"]["remedy_size"],
           "frozen": ph["update"]["converged"],
           "active_history_sha256": hashlib.sha256(np.asarray(s.active_history, dtype=np.int64).tobytes()).hexdigest(),
           "phi_field_digest": field_digest(res.phi)}
    assert got == {k: rec[k] for k in got}
    del g, res
    eik.clear_workspaces()
    torch.cuda.empty_cache()
