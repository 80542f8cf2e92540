"""EIK_DIAG build (tools/build_variant.py libeik_ifim_diag -DEIK_DIAG) on bench workloads: per-size-bucket
update iterations and remedy rounds with their phase B / A times.  python tools/diag_rounds.py cfg3 [n] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["EIK_DIAG_PRINT"] = "1"
from paper_2106_15869_b200 import _native  # noqa: E402

_native.LIB = _native.LIB.replace("libeik_ifim.so", os.environ.get("EIK_DIAG_LIB", "libeik_ifim_diag.so"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2106_15869_b200 as eik  # noqa: E402

args = sys.argv[1:]
while args:
    kind = args.pop(0)
    n = int(args.pop(0)) if args and args[0].isdigit() else None
    n = n or {"cfg1": 256, "cfg2": 4096, "cfg3": 256, "cfg5": 1024}.get(kind, 512)
    w = bench.make_workload(torch, torch.device("cuda"), kind, n)
    for rep in range(2):
        g = w.grid(eik, torch.full(w.shape, float("inf"), dtype=torch.float64, device="cuda"), w.F,
                   torch.zeros(w.shape, dtype=torch.uint8, device="cuda"))
        print(f"=== {kind} {w.shape} rep {rep}", file=sys.stderr, flush=True)
        r = eik.solve_ifim(g, w.bc(eik))
        print(kind, w.shape, r.stats.device_ms, r.stats.iterations, r.stats.solver_calls, file=sys.stderr, flush=True)
