"""One solve of a bench workload for ncu captures: python tools/prof_cfg.py cfg2 [n] [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2106_15869_b200 as eik  # noqa: E402

kind = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else {"cfg1": 256, "cfg2": 4096, "cfg3": 256, "cfg5": 1024}.get(kind, 512)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = bench.make_workload(torch, torch.device("cuda"), kind, n)
for _ in range(reps):
    g = w.grid(eik, torch.full(w.shape, float("inf"), dtype=torch.float64, device="cuda"), w.F,
               torch.zeros(w.shape, dtype=torch.uint8, device="cuda"))
    r = eik.solve_ifim(g, w.bc(eik))
    torch.cuda.synchronize()
print(kind, w.shape, r.stats.device_ms, r.stats.solver_calls)
