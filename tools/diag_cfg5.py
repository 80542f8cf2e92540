"""EIK_DIAG build on the cfg5 workload at n^3 (default 512): per-round / fill diagnostics."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["EIK_DIAG_PRINT"] = "1"
from paper_2106_15869_b200 import _native  # noqa: E402

_native.LIB = _native.LIB.replace("libeik_ifim.so", "libeik_ifim_diag.so")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2106_15869_b200 as eik  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
w = bench.make_workload(torch, torch.device("cuda"), "cfg5", n)
g = eik.Grid3D(n, n, n, w.h, (0.0, 0.0, 0.0), torch.full((n, n, n), float("inf"), dtype=torch.float64, device="cuda"),
               w.F, torch.zeros((n, n, n), dtype=torch.uint8, device="cuda"))
r = eik.solve_ifim(g, eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in w.seeds)))
print(r.stats.device_ms, r.stats.solver_calls, flush=True)
