"""The reference's acceptance criteria that concern this path (T/test_acceptance.py),
run on the B200 engine: C01/C10 fields satisfy the equation, C03 no remedy on a smooth
single-source field, C05 first-order convergence to the exact distance, C06 result
invariance (workers, devices)."""
import math

import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik

pytestmark = pytest.mark.gpu
RESIDUAL_GATE = 1e-9  # T/test_acceptance.py:52


def _grid2d(m, Z, name):
    g = eik.Grid(m["nx"], m["ny"], m["dx"], m["dy"], (0.0, 0.0), np.full((m["ny"], m["nx"]), np.inf),
                 Z[name + "__speed"].copy(), Z[name + "__state0"].copy())
    nx = m["nx"]
    bc = eik.BoundaryCondition(tuple((eik.CellIndex(int(c) % nx, int(c) // nx), float(v))
                                     for c, v in zip(Z[name + "__seed_idx"], Z[name + "__seed_val"])))
    return g, bc


def test_c10_every_run_satisfies_the_equation(cases2d):
    """T/test_acceptance.py:342-351: max residual <= 1e-9 for every method run (ifim, fim, oracle)."""
    meta, Z = cases2d
    worst = 0.0
    for name, m in meta.items():
        for method in ("ifim", "fim", "oracle"):
            g, bc = _grid2d(m, Z, name)
            eik.run_method(method, g, bc)
            worst = max(worst, eik.max_residual(g))
    assert worst <= RESIDUAL_GATE, worst


def test_c03_no_remedy_on_smooth_single_source():
    """T/test_acceptance.py:197-212 (constant speed, one source): the remedy stage stays empty."""
    for n in (64, 128, 256):
        g = eik.new_grid(n, n, 1.0 / n, 1.0 / n)
        assert eik.solve_ifim(g, eik.seed_point(g, (n // 2, n // 3), 0.0)).stats.peak_remedy == 0
    for n in (32, 64):
        g = eik.new_grid_3d(n, n, n, 1.0)
        assert eik.solve_ifim(g, eik.seed_point(g, (n // 2, n // 3, n // 4), 0.0)).stats.peak_remedy == 0


def test_c05_first_order_convergence_3d():
    """T/test_acceptance.py:238-259 analogue on the GPU engine: Linf error of the point-source
    distance on the unit cube away from the source (|x - s| >= 0.25) halves with h."""
    errs = {}
    for n in (65, 129):
        h = 1.0 / (n - 1)
        dev = torch.device("cuda:0")
        g = eik.Grid3D(n, n, n, h, (0.0, 0.0, 0.0), torch.full((n, n, n), np.inf, dtype=torch.float64, device=dev),
                       torch.ones((n, n, n), dtype=torch.float64, device=dev),
                       torch.zeros((n, n, n), dtype=torch.uint8, device=dev))
        s = (n // 4, n // 2, n // 3)
        phi = eik.solve_ifim(g, eik.seed_point(g, s, 0.0)).phi
        ax = torch.arange(n, device=dev, dtype=torch.float64) * h
        d = torch.sqrt((ax[None, None, :] - s[0] * h) ** 2 + (ax[None, :, None] - s[1] * h) ** 2 +
                       (ax[:, None, None] - s[2] * h) ** 2)
        far = d >= 0.25
        errs[n] = float((phi - d).abs()[far].max())
    order = math.log2(errs[65] / errs[129])
    assert 0.7 <= order <= 1.3, (errs, order)


def test_c06_invariance_workers_and_devices(cases3d):
    """T/test_acceptance.py:262-274: identical digests whatever the worker count (ignored on the
    device) or the z-slab partition."""
    meta, Z = cases3d
    for name in ("checker_16", "smooth_13x11x9"):
        m = meta[name]
        nx, ny, nz = m["nx"], m["ny"], m["nz"]
        digests = set()
        for kw in ({"workers": 1}, {"workers": 2}, {"workers": 8}, {"devices": [0, 0]}, {"devices": [0, 0, 0]}):
            g = eik.Grid3D(nx, ny, nz, m["h"], (0.0, 0.0, 0.0), np.full((nz, ny, nx), np.inf),
                           Z[name + "__speed"].reshape(nz, ny, nx).copy(), Z[name + "__state0"].reshape(nz, ny, nx).copy())
            bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(int(c) % nx, (int(c) // nx) % ny, int(c) // (nx * ny)),
                                              float(v)) for c, v in zip(Z[name + "__seed_idx"], Z[name + "__seed_val"])))
            digests.add(eik.field_sha256(eik.solve_ifim(g, bc, **kw).phi))
        assert len(digests) == 1 and digests == {m["sha256"]}, name
