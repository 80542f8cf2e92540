"""GPU cross-check digest of cfg5 at its BASELINE size (1024^3), where no oracle run is affordable
(the oracle port needs ~10 h on 8 cores; tests/golden/fullsize.json holds the oracle digests up to
512^3).  Three independent device implementations of the remedy must agree bit for bit -- the
member-list kernel (k_remedy), the TMA brick pipeline (k_remedy_b) and the multi-rank peer-slab
kernels with two ranks emulated on one GPU (k_update_mr / k_remedy_mr) -- on phi (chunked device
SHA-256, harness.field_digest) and every RunStats integer; the agreed digest is written to
tests/golden/fullsize_gpu.json.  Run on a B200:  python tools/make_gpu_crosscheck.py [n]
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2106_15869_b200 as eik  # noqa: E402
from paper_2106_15869_b200 import _native  # noqa: E402
from paper_2106_15869_b200.harness import field_digest  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dev = torch.device("cuda:0")
w = bench.make_workload(torch, dev, "cfg5", n)


def record(phi, s, how, secs):
    ph = s.phases
    return {"how": how, "seconds": round(secs, 3), "phi_field_digest": field_digest(phi),
            "iterations": s.iterations, "solver_calls": s.solver_calls, "peak_active": s.peak_active,
            "peak_remedy": s.peak_remedy, "phi_writes": s.phi_writes,
            "upd_iterations": ph["update"]["iterations"], "upd_calls": ph["update"]["solver_calls"],
            "frozen": ph["update"]["converged"], "build_calls": ph["build"]["solver_calls"],
            "remedy_size": ph["build"]["remedy_size"], "rem_iterations": ph["remedy"]["iterations"],
            "rem_calls": ph["remedy"]["solver_calls"],
            "active_history_sha256": hashlib.sha256(np.asarray(s.active_history, dtype=np.int64).tobytes()).hexdigest()}


runs = []
for engine in ("list", "brick"):
    os.environ["EIK_REMEDY"] = engine
    g = w.grid(eik, torch.full(w.shape, float("inf"), dtype=torch.float64, device=dev), w.F,
               torch.zeros(w.shape, dtype=torch.uint8, device=dev))
    t0 = time.perf_counter()
    res = eik.solve_ifim(g, w.bc(eik))
    torch.cuda.synchronize()
    assert _native.last_remedy_engine() == engine, _native.last_remedy_engine()
    runs.append(record(res.phi, res.stats, f"single device, remedy engine {engine}", time.perf_counter() - t0))
    print(runs[-1], flush=True)
    del g, res
    torch.cuda.empty_cache()
os.environ.pop("EIK_REMEDY")
eik.clear_workspaces()
torch.cuda.empty_cache()
from paper_2106_15869_b200.slab_peer import EmulatedSlabs  # noqa: E402

es = EmulatedSlabs(w.shape, w.h, 2, dev)
t0 = time.perf_counter()
phi, s, _ = es.solve(w.F, torch.zeros(w.shape, dtype=torch.uint8, device=dev), w.linear_seeds())
torch.cuda.synchronize()
runs.append(record(phi, s, "peer-slab kernels, 2 ranks emulated on one GPU", time.perf_counter() - t0))
print(runs[-1], flush=True)
keys = [k for k in runs[0] if k not in ("how", "seconds")]
for r in runs[1:]:
    bad = [k for k in keys if r[k] != runs[0][k]]
    assert not bad, (r["how"], bad)
out = os.path.join(ROOT, "tests", "golden", "fullsize_gpu.json")
db = json.load(open(out)) if os.path.exists(out) else {}
db[f"cfg5@{n}"] = {"config": "cfg5", "n": n, "speed_field_digest": field_digest(w.F), "agreed_by": [r["how"] for r in runs],
                   "seconds": {r["how"]: r["seconds"] for r in runs}, **{k: runs[0][k] for k in keys},
                   "note": "GPU cross-check (no oracle run at this size): three independent remedy "
                           "implementations agree bit for bit; tests/golden/fullsize.json pins the same "
                           "code paths to the oracle up to 512^3"}
with open(out, "w") as fh:
    json.dump(db, fh, indent=1, sort_keys=True)
print("agreed; wrote", out)
