"""A/B timing of engine variants on bench workloads: python tools/ab_cfg.py cfg2,cfg3,cfg4 VARIANT.so[:ENV=V] ...
Each (variant, workload) runs in its own process (3 solves, min device ms per phase), alternating over 2
passes; the phi sha256 and solver calls must agree across variants."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, os, json, hashlib
sys.path.insert(0, sys.argv[1])
from paper_2106_15869_b200 import _native
_native.LIB = os.path.join(os.path.dirname(_native.LIB), sys.argv[2])
import torch, bench, paper_2106_15869_b200 as eik
kind = sys.argv[3]
n = {"cfg1": 256, "cfg2": 4096, "cfg3": 256, "cfg5": 1024}.get(kind, 512)
w = bench.make_workload(torch, torch.device("cuda"), kind, n)
best = None
for r in range(3):
    g = w.grid(eik, torch.full(w.shape, float("inf"), dtype=torch.float64, device="cuda"), w.F,
               torch.zeros(w.shape, dtype=torch.uint8, device="cuda"))
    res = eik.solve_ifim(g, w.bc(eik))
    d = res.stats.device_ms
    if best is None or d["total"] < best["total"]:
        best = dict(d)
phi = torch.as_tensor(res.phi).contiguous().view(torch.int64).cpu().numpy()
print("RESULT", json.dumps({"calls": res.stats.solver_calls, "sha": hashlib.sha256(phi.tobytes()).hexdigest()[:16], **best}))
'''

kinds = sys.argv[1].split(",")
variants = sys.argv[2:]
res = {}
for _ in range(2):
    for kind in kinds:
        for v in variants:
            so, _, env = v.partition(":")
            e = dict(os.environ)
            for kv in filter(None, env.split(",")):
                k, _, val = kv.partition("=")
                e[k] = val
            out = subprocess.run([sys.executable, "-c", CHILD, ROOT, so, kind], capture_output=True, text=True, env=e)
            line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
            if not line:
                print(v, kind, "FAILED", out.stderr[-2000:], flush=True)
                continue
            r = json.loads(line[0][7:])
            key = (kind, v)
            if key not in res or r["total"] < res[key]["total"]:
                res[key] = r
for kind in kinds:
    ref = None
    for v in variants:
        r = res.get((kind, v))
        if r is None:
            continue
        ref = ref or r
        same = r["sha"] == ref["sha"] and r["calls"] == ref["calls"]
        print(f"{kind:5s} {v:40s} update {r['update']:8.3f} build {r['build']:7.3f} remedy {r['remedy']:9.3f} "
              f"total {r['total']:9.3f}  {'same' if same else 'DIFFERENT'} {r['sha']}", flush=True)
