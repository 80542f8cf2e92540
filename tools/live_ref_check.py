"""Live-reference parity at a larger 2D size (one-off evidence run on the GPU box): the unmodified
reference from baseline/_ref solves the cfg2 sinusoid workload at n x n with its own solve_ifim
(pure Python / numpy, minutes at n = 1024), the B200 engine solves the same grid, and the phi bytes
and every RunStats field are compared.  python tools/live_ref_check.py [n]"""
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import numpy as np  # noqa: E402
from eikonal.grid import BoundaryCondition, CellIndex, new_grid  # noqa: E402  (the reference)
from eikonal.ifim import solve_ifim as ref_solve  # noqa: E402

import bench  # noqa: E402
import paper_2106_15869_b200 as eik  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
h, F, seeds = bench.workload_np("cfg2", n)
F = np.ascontiguousarray(F)


def grid():
    g = new_grid(n, n, h, h, origin=(0.0, 0.0), speed=F)
    return g, BoundaryCondition(tuple((CellIndex(i, j), 0.0) for i, j in seeds))


g, bc = grid()
t0 = time.perf_counter()
ref = ref_solve(g, bc, workers=1)
t_ref = time.perf_counter() - t0
g2, bc2 = grid()
t0 = time.perf_counter()
got = eik.solve_ifim(g2, bc2)
t_gpu = time.perf_counter() - t0
same_phi = np.array_equal(np.asarray(got.phi).view(np.uint64), np.asarray(ref.phi).view(np.uint64))
r, s = ref.stats, got.stats
fields = ("iterations", "solver_calls", "peak_active", "peak_remedy")
same_stats = all(getattr(r, k) == getattr(s, k) for k in fields) and list(r.active_history) == list(s.active_history)
print(f"cfg2 sinusoid {n}x{n}, 8 seeds: reference solve_ifim {t_ref:.1f} s, B200 {t_gpu * 1e3:.1f} ms (wall, incl. "
      f"host transfers); phi sha256 {hashlib.sha256(np.asarray(ref.phi).tobytes()).hexdigest()[:16]}; "
      f"stats {[getattr(r, k) for k in fields]}; bit-identical phi: {same_phi}; equal RunStats + active_history: "
      f"{same_stats}")
sys.exit(0 if same_phi and same_stats else 1)
