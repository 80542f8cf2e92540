"""Device time of the peer-slab kernels emulated on one GPU (R rank groups in one launch)
against the single-device solve, cfg4 checkerboard at n^3."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_15869_b200 as eik  # noqa: E402
from paper_2106_15869_b200.slab_peer import EmulatedSlabs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = torch.arange(n, device="cuda") // (n // 16)
F = torch.where(((k[:, None, None] + k[None, :, None] + k[None, None, :]) % 2) == 0, torch.tensor(1.0, dtype=torch.float64), torch.tensor(0.01, dtype=torch.float64))
st0 = torch.zeros((n, n, n), dtype=torch.uint8, device="cuda")
c = n // 2
g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), float("inf"), dtype=torch.float64, device="cuda"),
               F, st0.clone())
for _ in range(2):
    g.phi.fill_(float("inf"))
    g.state.zero_()
    r = eik.solve_ifim(g, eik.seed_point(g, (c, c, c), 0.0))
print(f"single: {r.stats.device_ms}", flush=True)
for R in (1, 2, 4):
    em = EmulatedSlabs((n, n, n), 1.0, R, "cuda")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        phi, s, _ = em.solve(F, st0, [((c * n + c) * n + c, 0.0)])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"R={R}: wall {dt * 1e3:.1f} ms device {s.device_ms} identical={torch.equal(phi, r.phi)} "
          f"calls {s.solver_calls == r.stats.solver_calls}", flush=True)
    del em
