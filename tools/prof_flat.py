"""One constant-speed 16-seed solve at n^3 (cfg3 family, default 256) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_15869_b200 as eik  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
rng = np.random.default_rng(2106)
seeds = []
while len(seeds) < 16:
    s = tuple(int(v) for v in rng.integers(0, n, 3))
    if s not in seeds:
        seeds.append(s)
g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), float("inf"), dtype=torch.float64, device="cuda"),
               torch.ones((n, n, n), dtype=torch.float64, device="cuda"), torch.zeros((n, n, n), dtype=torch.uint8, device="cuda"))
res = eik.solve_ifim(g, eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in seeds)))
torch.cuda.synchronize()
print("calls", res.stats.solver_calls, "iters", res.stats.iterations, "rem", res.stats.phases["remedy"], "dev", res.stats.device_ms)
