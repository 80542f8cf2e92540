"""Remedy throughput vs grid size (L2-resident vs DRAM-resident): python tools/scan_sizes.py [kind] n1 n2 ...
Prints remedy members, ms, ns/member and algorithmic GB/s for checkerboard (default) or cfg5 fields."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2106_15869_b200 as eik  # noqa: E402

args = sys.argv[1:]
kind = args.pop(0) if args and not args[0].isdigit() else "cfg4"
for n in map(int, args):
    w = bench.make_workload(torch, torch.device("cuda"), kind, n)
    best = None
    for _ in range(3):
        g = w.grid(eik, torch.full(w.shape, float("inf"), dtype=torch.float64, device="cuda"), w.F,
                   torch.zeros(w.shape, dtype=torch.uint8, device="cuda"))
        r = eik.solve_ifim(g, w.bc(eik))
        ms = r.stats.device_ms["remedy"]
        best = ms if best is None else min(best, ms)
    s = r.stats
    rc = s.phases["remedy"]["solver_calls"]
    upd_w = s.phases["update"]["solver_calls"] - s.phases["update"]["converged"]
    rw = s.phi_writes - upd_w
    print(f"{kind} n={n:5d} cells={w.cells:12d} rem_members={rc:13d} rounds={s.phases['remedy']['iterations']:5d} "
          f"rem_ms={best:9.2f} ns/member={best * 1e6 / max(rc, 1):7.3f} alg_GB/s={8 * (2 * rc + rw) / best / 1e6:8.1f}",
          flush=True)
