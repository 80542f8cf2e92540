"""One (or `reps`) solve_ifim of a bench.py workload on cuda:0, for ncu captures and quick timings.

    python tools/prof_solve.py cfg4 512 [reps]      (EIK_REMEDY=list|brick|auto selects the remedy engine)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2106_15869_b200 as eik  # noqa: E402
from paper_2106_15869_b200 import _native  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
dev = torch.device("cuda:0")
w = bench.make_workload(torch, dev, config, n)
for _ in range(reps):
    phi = torch.full(w.shape, float("inf"), dtype=torch.float64, device=dev)
    state = torch.zeros(w.shape, dtype=torch.uint8, device=dev)
    g = w.grid(eik, phi, w.F, state)
    res = eik.solve_ifim(g, w.bc(eik))
    torch.cuda.synchronize()
s = res.stats
print(f"{config}@{n}: calls {s.solver_calls} iters {s.iterations} peak_remedy {s.peak_remedy} "
      f"engine {_native.last_remedy_engine()} device_ms {s.device_ms}")
