"""GPU fixpoint / residual vs the CPU restatement and the
reference's own fixpoint output, plus full-size properties of the iFIM field."""
import math

import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik
from oracle import cpu

pytestmark = pytest.mark.gpu


def test_fixpoint_matches_reference_golden(staged2d):
    """ex1 32^2 fixpoint produced by the live reference (E/oracle.py)."""
    Z = staged2d
    ny, nx = Z["stale_phi_in"].shape
    dx = float(Z["stale_dx"][0])
    g = eik.Grid(nx, ny, dx, dx, (-10.0, -10.0), np.full((ny, nx), np.inf), Z["stale_speed"].copy(),
                 np.where(Z["stale_speed"] == 0, 4, 0).astype(np.uint8))
    src = np.flatnonzero(Z["stale_state"].ravel() == eik.CellState.SOURCE)
    vals = Z["stale_fixpoint"].ravel()[src]
    bc = eik.BoundaryCondition(tuple((eik.CellIndex(int(c % nx), int(c // nx)), float(v)) for c, v in zip(src, vals)))
    res = eik.solve_fixpoint(g, bc)
    assert np.array_equal(res.phi.view(np.uint64), Z["stale_fixpoint"].view(np.uint64))


@pytest.mark.parametrize("kind", ["2d", "aniso", "3d"])
def test_fixpoint_bit_exact_vs_oracle(cases2d, cases3d, kind):
    if kind == "3d":
        meta, Z = cases3d
        names = list(meta)
    else:
        meta, Z = cases2d
        names = ["aniso_53x37", "sealed_40x20"] if kind == "aniso" else ["ex2_48", "ex5_48", "pocket_24", "checker_64"]
    for name in names:
        m = meta[name]
        if kind == "3d":
            shape, sp = (m["nz"], m["ny"], m["nx"]), m["h"]
            g = eik.new_grid_3d(m["nx"], m["ny"], m["nz"], m["h"], speed=Z[name + "__speed"].reshape(shape))
            cells = [eik.CellIndex3D(c % m["nx"], (c // m["nx"]) % m["ny"], c // (m["nx"] * m["ny"]))
                     for c in Z[name + "__seed_idx"].tolist()]
        else:
            shape, sp = (m["ny"], m["nx"]), (m["dx"], m["dy"])
            g = eik.new_grid(m["nx"], m["ny"], m["dx"], m["dy"], speed=Z[name + "__speed"])
            cells = [eik.CellIndex(c % m["nx"], c // m["nx"]) for c in Z[name + "__seed_idx"].tolist()]
        bc = eik.BoundaryCondition(tuple(zip(cells, Z[name + "__seed_val"].tolist())))
        res = eik.solve_fixpoint(g, bc)
        ref, st = cpu.solve_fixpoint(shape, sp, Z[name + "__speed"], Z[name + "__seed_idx"], Z[name + "__seed_val"])
        assert np.array_equal(res.phi.view(np.uint64), ref.view(np.uint64)), name
        assert (res.stats.iterations, res.stats.solver_calls) == (st["iterations"], st["solver_calls"]), name
        assert eik.max_residual(g) <= 1e-9


def test_max_residual_flags_a_stale_cell():
    g = eik.new_grid(32, 32, 1.0, 1.0)
    eik.solve_ifim(g, eik.seed_point(g, (3, 4), 0.0))
    assert eik.max_residual(g) <= 1e-12
    g.phi[20, 14] += 0.3
    assert abs(eik.max_residual(g) - 0.3) < 1e-9


@pytest.mark.slow
def test_full_size_ifim_equals_fixpoint_256():
    """cfg3-like: 3D 256^3, F=1, 16 random seeds -- iFIM vs the independent fixpoint
    (T/test_ifim.py:23-30 agreement <= 1e-9) and the residual gate."""
    n = 256
    rng = np.random.default_rng(2106)
    seeds = set()
    while len(seeds) < 16:
        seeds.add(tuple(int(v) for v in rng.integers(0, n, 3)))
    bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in sorted(seeds)))
    dev = torch.device("cuda:0")

    def grid():
        return eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=torch.float64, device=dev),
                          torch.ones((n, n, n), dtype=torch.float64, device=dev),
                          torch.zeros((n, n, n), dtype=torch.uint8, device=dev))

    g1, g2 = grid(), grid()
    r1 = eik.solve_ifim(g1, bc)
    r2 = eik.solve_fixpoint(g2, bc)
    assert torch.max(torch.abs(r1.phi - r2.phi)).item() <= 1e-9
    assert eik.max_residual(g1) <= 1e-9
    # exact-distance check: first-order error bounded like the 2D calibration (~0.3 h ln n per axis)
    z, y, x = torch.meshgrid(*(torch.arange(n, device=dev, dtype=torch.float64),) * 3, indexing="ij")
    exact = torch.full_like(r1.phi, np.inf)
    for s in seeds:
        exact = torch.minimum(exact, torch.sqrt((x - s[0]) ** 2 + (y - s[1]) ** 2 + (z - s[2]) ** 2))
    err = (r1.phi - exact).abs()
    assert err.max().item() <= 0.6 * np.log(n)  # first-order scheme: error ~ C h ln n (SURVEY.md §7 hard part 6)


def test_exact_distance_error_equals_oracle_64():
    """Constant-speed check against the exact distance: the GPU field's error equals
    the CPU oracle's error (SURVEY.md §8c/BASELINE.md parity gate)."""
    n = 64
    rng = np.random.default_rng(7)
    seeds = sorted({tuple(int(v) for v in rng.integers(0, n, 3)) for _ in range(16)})
    g = eik.new_grid_3d(n, n, n, 1.0)
    res = eik.solve_ifim(g, eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in seeds)))
    lin = [(k * n + j) * n + i for i, j, k in seeds]
    ref = cpu.solve_ifim((n, n, n), 1.0, np.ones((n, n, n)), lin, [0.0] * len(lin), threads=8)
    z, y, x = np.meshgrid(*(np.arange(n, dtype=np.float64),) * 3, indexing="ij")
    exact = np.min([np.sqrt((x - i) ** 2 + (y - j) ** 2 + (z - k) ** 2) for i, j, k in seeds], axis=0)
    e_gpu, e_cpu = np.abs(res.phi - exact), np.abs(ref.phi - exact)
    assert np.max(np.abs(e_gpu - e_cpu)) <= 1e-10
    assert e_gpu.max() <= 0.6 * np.log(n)


@pytest.mark.slow
def test_cfg5_full_size_ifim_equals_fixpoint():
    """cfg5 at its full 1024^3 (BASELINE.json configs[4] on one GPU): the iFIM field equals the
    GPU fixpoint ground truth (E/oracle.py) within 1e-9 (the reference's method-vs-fixpoint
    gate, T/test_fim.py:23 / T/test_ifim.py:30; measured 2.2e-10) and satisfies the equation."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    n = 1024
    dev = torch.device("cuda:0")
    w = bench.make_workload(torch, dev, "cfg5", n)
    bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in w.seeds))
    g = eik.Grid3D(n, n, n, w.h, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=torch.float64, device=dev),
                   w.F, torch.zeros((n, n, n), dtype=torch.uint8, device=dev))
    a = eik.solve_ifim(g, bc).phi
    assert eik.max_residual(g) <= 1e-9
    g.phi.fill_(np.inf)
    g.state.zero_()
    b = eik.solve_fixpoint(g, bc).phi
    assert eik.field_max_diff(a, b) <= 1e-9


def test_field_npy_streams_a_device_field(tmp_path):
    """export_field_npy / import_field_npy on a CUDA field (chunked D2H / H2D), bit-exact."""
    n = 96
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=torch.float64, device="cuda"),
                   torch.ones((n, n, n), dtype=torch.float64, device="cuda"),
                   torch.zeros((n, n, n), dtype=torch.uint8, device="cuda"))
    res = eik.solve_ifim(g, eik.seed_point(g, (10, 20, 30), 0.0))
    p = str(tmp_path / "phi.npy")
    eik.export_field_npy(g, p)
    h = eik.import_field_npy(p, device="cuda")
    assert torch.equal(h.phi, res.phi) and h.phi.is_cuda
    assert eik.field_sha256(np.load(p)) == eik.field_sha256(res.phi)


@pytest.mark.slow
def test_near_max_grid_1280_cubed():
    """Near the 2^31-cells-per-device limit (1280^3 = 2.1e9 cells, ~100 GB on the device): a
    corner source on a cubic grid gives a field that is bitwise symmetric under axis
    permutations (the solver sorts its three axis minima; Jacobi sets are order-free), finite
    everywhere, and within first-order error of the distance at the far corner."""
    n = 1280
    dev = torch.device("cuda:0")
    eik.clear_workspaces()  # earlier full-size tests may still hold cached workspaces / blocks
    torch.cuda.empty_cache()
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=torch.float64, device=dev),
                   torch.ones((n, n, n), dtype=torch.float64, device=dev),
                   torch.zeros((n, n, n), dtype=torch.uint8, device=dev))
    try:
        r = eik.solve_ifim(g, eik.seed_point(g, (0, 0, 0), 0.0))
        phi = g.phi
        del r
        assert bool(torch.isfinite(phi).all())
        for a, b in ((0, 2), (1, 2), (0, 1)):
            assert torch.equal(phi, phi.transpose(a, b)), (a, b)
        far = float(phi[n - 1, n - 1, n - 1])
        exact = math.sqrt(3.0) * (n - 1)
        assert exact <= far <= exact * 1.05
    finally:
        del g
        eik.clear_workspaces()
        torch.cuda.empty_cache()


def test_bench_json_contract_small():
    """bench.py's JSON line (the driver's contract) on a small grid: every required key present."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--size", "64", "--steps", "2",
                          "--warmup", "3", "--cpu-size", "16"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2 and d["dtype"] == "f64"
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.parametrize("extra,dtype,engine", [(["--dtype", "f32"], "f32", None),
                                                (["--config", "cfg5", "--size", "64"], "f64", "brick"),
                                                (["--config", "cfg1", "--size", "64"], "f64", None),
                                                (["--config", "cfg2", "--size", "128"], "f64", None),
                                                (["--config", "cfg3", "--size", "64"], "f64", None),
                                                (["--method", "fim"], "f64", None),
                                                (["--slabs"], "f64", None)])
def test_bench_variants_small(extra, dtype, engine):
    """bench.py's other modes end to end on small grids: the float32 perf mode, the brick remedy
    engine (forced), the 2D configs, cfg3, the FIM baseline and the one-GPU slab protocol; each
    prints a valid line (and names the remedy engine that ran when one is forced)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    if engine:
        env["EIK_REMEDY"] = engine
    args = [sys.executable, os.path.join(root, "bench.py"), "--steps", "1", "--warmup", "3", "--no-cpu", "--no-e2e"]
    if "--size" not in extra:
        args += ["--size", "64"]
    out = subprocess.run(args + extra, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["value"] > 0 and d["dtype"] == dtype
    if engine:
        assert d["config"]["remedy_engine"] == engine, d["config"]


def test_pinned_host_grid_result_copy():
    """A pinned CPU-tensor grid (the chunked download + overlapped host result copy of
    ifim._HostResult): grid.phi holds the solution in place, SolverResult.phi is a separate copy
    with the same bytes, both equal to the solve of the same problem on CUDA tensors."""
    n = 164  # > 2^22 cells: the large-field path
    k = np.arange(n) // 8
    F = np.where((k[:, None, None] + k[None, :, None] + k[None, None, :]) % 2 == 0, 1.0, 0.05)
    pin = lambda a: torch.as_tensor(a).pin_memory()  # noqa: E731
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), pin(np.full((n, n, n), np.inf)), pin(F),
                   pin(np.zeros((n, n, n), np.uint8)))
    res = eik.solve_ifim(g, eik.seed_point(g, eik.CellIndex3D(3, n // 2, n - 5), 0.0))
    dev = torch.device("cuda:0")
    g2 = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), float("inf"), dtype=torch.float64, device=dev),
                    torch.as_tensor(F, device=dev), torch.zeros((n, n, n), dtype=torch.uint8, device=dev))
    ref = eik.solve_ifim(g2, eik.seed_point(g2, eik.CellIndex3D(3, n // 2, n - 5), 0.0))
    assert res.phi.data_ptr() != g.phi.data_ptr()
    want = ref.phi.cpu().numpy().view(np.uint64)
    assert np.array_equal(g.phi.numpy().view(np.uint64), want)
    assert np.array_equal(res.phi.numpy().view(np.uint64), want)
    assert res.stats.solver_calls == ref.stats.solver_calls
