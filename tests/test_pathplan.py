"""Path planning over a solved field (E/pathplan.py:274-330) and the
Example 4 barrier-map pipeline (E/cli.py:154-187).

Golden paths come from the live reference (tests/golden/make_pathplan.py).  CPU tests walk the
oracle's phi (oracle/eik_oracle.c, bit-exact to the reference) and the reference's own
validation cases (T/test_pathplan.py); the GPU test runs the whole pipeline with the field
solved by the CUDA engine."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import paper_2106_15869_b200 as eik
from oracle import cpu
from paper_2106_15869_b200 import pathplan as pp

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "pathplan.json")) as fh:
    CASES = json.load(fh)


def _speed(rec):
    n = rec["n"]
    return pp.barrier_speed(pp.synthetic_barrier_map(n)) if rec["kind"] == "example4" else np.ones((n, n))


def _oracle_grid(rec):
    n = rec["n"]
    F = _speed(rec)
    i, j = rec["start"]
    res = cpu.solve_ifim((n, n), (1.0, 1.0), F, [j * n + i], [0.0])
    g = eik.new_grid(n, n, 1.0, 1.0, origin=(0.0, 0.0), speed=F)
    g.phi = res.phi.copy()
    g.state = res.state.copy()
    return g


@pytest.mark.parametrize("key", sorted(CASES))
def test_path_on_oracle_field_equals_reference(key):
    rec = CASES[key]
    g = _oracle_grid(rec)
    assert hashlib.sha256(np.ascontiguousarray(g.phi).tobytes()).hexdigest() == rec["phi_sha256"]
    path = pp.gradient_descent_path(g, tuple(rec["query"]), rec["step"])
    assert [list(p) for p in path.points] == rec["points"]
    assert path.phi == rec["phi"]


def test_synthetic_map_and_endpoints():
    for n in (16, 64, 97):
        m = pp.synthetic_barrier_map(n)
        rows = np.nonzero(m.blocked.any(axis=1))[0]
        assert len(rows) == 2
        gaps = [set(np.nonzero(~m.blocked[r])[0].tolist()) for r in rows]
        assert gaps[0] and gaps[1] and gaps[0].isdisjoint(gaps[1])
        s, gl = pp.synthetic_endpoints(n)
        assert s.j < rows[0] < rows[1] < gl.j and not m.blocked[s.j, s.i] and not m.blocked[gl.j, gl.i]
    with pytest.raises(ValueError):
        pp.synthetic_barrier_map(8)
    with pytest.raises(ValueError, match="does not match"):
        pp.BarrierMap(3, 2, np.zeros((3, 3), dtype=bool))


def test_validation_errors_match_reference():
    rec = CASES["single_n48_step0.5"]
    g = _oracle_grid(rec)
    with pytest.raises(ValueError, match="step"):
        pp.gradient_descent_path(g, (8.0, 0.0), 0.0)
    with pytest.raises(ValueError, match="step"):
        pp.gradient_descent_path(g, (8.0, 0.0), 10.0)
    with pytest.raises(ValueError, match="outside"):
        pp.gradient_descent_path(g, (55.0, 0.0), 0.1)
    one = pp.gradient_descent_path(g, g.cell_center(*rec["start"]), 0.1)  # starts in the source
    assert len(one) == 1
    # blocked start (T/test_pathplan.py:150-164)
    ex = CASES["example4_n64_step0.5"]
    gm = _oracle_grid(ex)
    wj = int(np.nonzero((gm.state == eik.CellState.BLOCKED).any(axis=1))[0][0])
    wi = int(np.nonzero(gm.state[wj] == eik.CellState.BLOCKED)[0][0])
    with pytest.raises(ValueError, match="blocked"):
        pp.gradient_descent_path(gm, gm.cell_center(wi, wj), 0.5)


def test_unreached_start_and_stalled_bowl():
    # an enclosed room the front never enters (T/test_pathplan.py:167-178)
    speed = np.ones((16, 16))
    speed[4:9, 4] = speed[4:9, 8] = speed[4, 4:9] = speed[8, 4:9] = 0.0
    res = cpu.solve_ifim((16, 16), (1.0, 1.0), speed, [0], [0.0])
    g = eik.new_grid(16, 16, 1.0, 1.0, speed=speed)
    g.phi, g.state = res.phi.copy(), res.state.copy()
    assert np.isinf(g.phi[6, 6])
    with pytest.raises(ValueError, match="unreached"):
        pp.gradient_descent_path(g, g.cell_center(6, 6), 0.5)
    # a bowl whose minimum is not a source (T/test_pathplan.py:204-213)
    b = eik.new_grid(17, 17, 1.0, 1.0)
    xx, yy = np.meshgrid(np.arange(17.0), np.arange(17.0))
    b.phi = (xx - 8.0) ** 2 + (yy - 8.0) ** 2
    b.state = np.zeros((17, 17), dtype=np.uint8)
    b.state[0, 0] = eik.CellState.SOURCE
    b.phi[0, 0] = -1.0
    with pytest.raises(RuntimeError, match="stalled"):
        pp.gradient_descent_path(b, (12.0, 9.0), 0.5)


def test_path_properties_and_csv(tmp_path):
    rec = CASES["example4_n96_step0.25"]
    g = _oracle_grid(rec)
    path = pp.gradient_descent_path(g, tuple(rec["query"]), rec["step"])
    assert np.all(np.diff(np.asarray(path.phi)) < 0.0)
    seg = np.hypot(*np.diff(np.asarray(path.points), axis=0).T)
    assert np.all(seg <= rec["step"] * (1 + 1e-12))
    blocked = g.state == eik.CellState.BLOCKED
    assert not any(blocked[round(y), round(x)] for x, y in path.points)
    out = tmp_path / "p.csv"
    path.to_csv(str(out))
    first = [float(t) for t in out.read_text().splitlines()[0].split(",")]
    assert first == [*rec["query"], rec["phi"][0]] and math.isfinite(first[2])


@pytest.mark.gpu
@pytest.mark.parametrize("key", [k for k in sorted(CASES) if CASES[k]["kind"] == "example4"])
def test_pipeline_on_gpu_field_equals_reference(key):
    """Barrier map -> GPU solve_ifim -> descent: the reference's path, bit for bit."""
    import torch

    rec = CASES[key]
    n = rec["n"]
    grid, result, path = pp.plan_path(pp.synthetic_barrier_map(n), eik.CellIndex(*rec["start"]),
                                      eik.CellIndex(*rec["goal"]), rec["step"], device="cuda:0")
    assert isinstance(grid.phi, torch.Tensor) and grid.phi.is_cuda
    assert eik.field_sha256(grid.phi) == rec["phi_sha256"]
    assert [list(p) for p in path.points] == rec["points"] and path.phi == rec["phi"]
