"""Digest of the LIVE reference's own solve_ifim on a 2D BASELINE workload (CPU only; run in the
authoring container where /root/reference or baseline/_ref is importable):
python tools/live_ref_digest.py cfg2 4096.  Prints phi sha256 and the RunStats integers and compares
them with tests/golden/fullsize.json (the oracle digests the GPU is tested against), closing the
chain live reference == oracle == GPU at full size."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import numpy as np  # noqa: E402
from eikonal.grid import BoundaryCondition, CellIndex, new_grid  # noqa: E402  (the reference)
from eikonal.ifim import solve_ifim  # noqa: E402

import bench  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
h, F, seeds = bench.workload_np(config, n)
g = new_grid(n, n, h, h, origin=(0.0, 0.0), speed=np.ascontiguousarray(F))
bc = BoundaryCondition(tuple((CellIndex(i, j), 0.0) for i, j in seeds))
t0 = time.perf_counter()
res = solve_ifim(g, bc, workers=1)
secs = time.perf_counter() - t0
s = res.stats
out = {"config": config, "n": n, "seconds": round(secs, 1),
       "phi_sha256": hashlib.sha256(np.ascontiguousarray(res.phi).tobytes()).hexdigest(),
       "iterations": s.iterations, "solver_calls": s.solver_calls, "peak_active": s.peak_active,
       "peak_remedy": s.peak_remedy,
       "active_history_sha256": hashlib.sha256(np.asarray(s.active_history, dtype=np.int64).tobytes()).hexdigest()}
with open(os.path.join(ROOT, "tests", "golden", "fullsize.json")) as fh:
    rec = json.load(fh).get(f"{config}@{n}")
if rec:
    want = {"phi_sha256": rec["phi_sha256"], **{k: rec["stats"][k] for k in ("iterations", "solver_calls", "peak_active",
                                                                            "peak_remedy")},
            "active_history_sha256": rec["update"]["active_history_sha256"]}
    out["equals_oracle_digest"] = all(out[k] == v for k, v in want.items())
print(json.dumps(out), flush=True)
