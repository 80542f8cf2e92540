"""cfg2 (2D 4096^2 sinusoid, 8 seeds) device time of solve_ifim / solve_fim."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_15869_b200 as eik  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
h = 1 / (n - 1)
x = h * np.arange(n)
xx, yy = np.meshgrid(x, x)
F = torch.as_tensor(1 + 0.5 * np.sin(2 * np.pi * xx) * np.sin(2 * np.pi * yy), device="cuda")
rng = np.random.default_rng(2106)
cells = []
while len(cells) < 8:
    c = tuple(int(v) for v in rng.integers(0, n, 2))
    if c not in cells:
        cells.append(c)
bc = eik.BoundaryCondition(tuple((eik.CellIndex(i, j), 0.0) for i, j in cells))
for method in ("ifim", "fim"):
    for rep in range(2):
        g = eik.Grid(n, n, h, h, (0.0, 0.0), torch.full((n, n), np.inf, dtype=torch.float64, device="cuda"), F,
                     torch.zeros((n, n), dtype=torch.uint8, device="cuda"))
        r = eik.run_method(method, g, bc)
    s = r.stats
    print(method, s.device_ms, "calls", s.solver_calls, "iters", s.iterations, "peakA", s.peak_active,
          "peakR", s.peak_remedy, f"{s.solver_calls / (s.device_ms['total'] * 1e-3) / 1e9:.2f} G/s", flush=True)
