"""One checkerboard solve at n^3 (default 128) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_15869_b200 as eik

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
k = torch.arange(n, device="cuda") // max(1, n // 16)
F = torch.where(((k[None, None, :] + k[None, :, None] + k[:, None, None]) % 2) == 0, torch.tensor(1.0, dtype=torch.float64), torch.tensor(0.01, dtype=torch.float64))
for _ in range(reps):
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), float("inf"), dtype=torch.float64, device="cuda"),
                   F, torch.zeros((n, n, n), dtype=torch.uint8, device="cuda"))
    res = eik.solve_ifim(g, eik.seed_point(g, (n // 2, n // 2, n // 2), 0.0))
    torch.cuda.synchronize()
print("calls", res.stats.solver_calls, "dev", res.stats.device_ms)
