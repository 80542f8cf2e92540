"""Full-size oracle digests for the BASELINE.json configs (TEST INFRASTRUCTURE ONLY).

Runs the C restatement of the reference engine (oracle/eik_oracle.c, OpenMP; E/ifim.py:75-235
staged exactly like solve_ifim, E/ifim.py:221-235) on the host, at the sizes BASELINE.json names,
and writes one record per config into tests/golden/fullsize.json:

* sha256 of the speed field (the GPU tests rebuild the field and check this first),
* the update step: every RunStats integer, sha256 + length of active_history, the frozen set
  (free cells with finite phi after the update step; its size is `converged`, its digest the
  sha256 of the finite-mask bytes), sha256 of phi after the update step,
* the build pass: calls, |R_0|, sha256 of the member mask (uint8 bytes, C order),
* the remedy step: rounds, calls, peak, writes,
* the composed stats (E/ifim.py:227-233) and sha256 of the final phi,
* the oracle's own wall time and thread count (the same-config CPU figure bench.py reports).

The oracle is pinned to the live reference by tests/test_oracle.py (golden fixtures made by
tests/golden/make_golden.py); this script extends that pin to full size.  Usage:

    python tests/golden/make_fullsize.py [cfg3 cfg2 cfg4 cfg5@512 ...] [--threads 8]

cfg4 (512^3, 14.2e9 solver calls) takes ~25 min on 8 cores; cfg5 is digested at 512^3 (the
1024^3 solve is ~3e11 calls, ~9 h here).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (workload_np: the host-built fields bench.py and the GPU tests use)
from oracle import cpu  # noqa: E402

OUT = os.path.join(HERE, "fullsize.json")
DEFAULT = ["cfg1@256", "cfg3@256", "cfg2@4096", "cfg4@512", "cfg5@512"]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def linear(seeds, n):
    if len(seeds[0]) == 2:
        return np.array([j * n + i for i, j in seeds], dtype=np.int64)
    return np.array([(k * n + j) * n + i for i, j, k in seeds], dtype=np.int64)


def digest(config: str, n: int, threads: int) -> dict:
    h, F, seeds = bench.workload_np(config, n)
    F = np.ascontiguousarray(F, dtype=np.float64)
    shape = F.shape
    spacing = (h, h) if F.ndim == 2 else h
    si = linear(seeds, n)
    sv = np.zeros(si.size)
    speed = F.ravel()
    state = np.where(speed == 0.0, 4, 0).astype(np.uint8)
    phi = np.full(speed.size, np.inf)
    t0 = time.perf_counter()
    up = cpu.update_step(shape, spacing, phi, speed, state, si, sv, threads=threads)
    t1 = time.perf_counter()
    hist = np.asarray(up.pop("active_history"), dtype=np.int64)
    free = (state != 4) & (state != 2)
    frozen = free & np.isfinite(phi)
    rec = {
        "config": config, "n": n, "shape": list(shape), "h": h, "seeds": [list(s) for s in seeds],
        "speed_sha256": sha(F),
        "update": {**up, "history_len": int(hist.size), "active_history_sha256": sha(hist),
                   "active_history_head": hist[:8].tolist(), "frozen": int(frozen.sum()),
                   "frozen_sha256": sha(frozen.astype(np.uint8)), "phi_sha256": sha(phi)},
    }
    member, bd = cpu.build_remedy(shape, spacing, phi, speed, state, threads=threads)
    t2 = time.perf_counter()
    rec["build"] = {"calls": bd["solver_calls"], "remedy_size": bd["remedy_size"], "member_sha256": sha(member)}
    rm = cpu.remedy_step(shape, spacing, phi, speed, state, member, threads=threads)
    t3 = time.perf_counter()
    rec["remedy"] = {"iterations": rm["iterations"], "solver_calls": rm["solver_calls"],
                     "peak_remedy": rm["peak_remedy"], "phi_writes": rm["phi_writes"]}
    rec["stats"] = {
        "iterations": up["iterations"] + rm["iterations"],
        "solver_calls": up["solver_calls"] + bd["solver_calls"] + rm["solver_calls"],
        "peak_active": up["peak_active"], "peak_remedy": rm["peak_remedy"],
        "phi_writes": up["phi_writes"] + rm["phi_writes"],
    }
    rec["phi_sha256"] = sha(phi)
    rec["phi_finite"] = int(np.isfinite(phi).sum())
    rec["phi_max_finite"] = float(phi[np.isfinite(phi)].max())
    rec["oracle"] = {"threads": threads, "seconds": {"update": t1 - t0, "build": t2 - t1, "remedy": t3 - t2,
                                                    "total": t3 - t0},
                     "calls_per_s": rec["stats"]["solver_calls"] / (t3 - t0),
                     "host": os.uname().nodename, "cpu_count": os.cpu_count()}
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=DEFAULT)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    cpu.build()
    db = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            db = json.load(fh)
    for spec in args.configs:
        config, n = spec.split("@")
        key = f"{config}@{n}"
        print(f"[fullsize] {key} ...", flush=True)
        rec = digest(config, int(n), args.threads)
        db[key] = rec
        with open(OUT + ".tmp", "w") as fh:
            json.dump(db, fh, indent=1, sort_keys=True)
        os.replace(OUT + ".tmp", OUT)
        print(f"[fullsize] {key}: calls {rec['stats']['solver_calls']} iterations {rec['stats']['iterations']} "
              f"peak_remedy {rec['stats']['peak_remedy']} in {rec['oracle']['seconds']['total']:.1f} s", flush=True)


if __name__ == "__main__":
    main()
