"""Where the e2e step's host-side time goes (design probe): cfg4 through solve_ifim with pinned host
tensors, timing the upload, the engine call, and the result commit separately."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2106_15869_b200 as eik  # noqa: E402
from paper_2106_15869_b200 import ifim  # noqa: E402

dev = torch.device("cuda:0")
w = bench.make_workload(torch, dev, "cfg4", 512)
speed = w.F.cpu().pin_memory()
phi = torch.empty(w.shape, dtype=torch.float64).pin_memory()
state = torch.empty(w.shape, dtype=torch.uint8).pin_memory()
bc = w.bc(eik)
T = {}
orig_dg, orig_commit = ifim._DeviceGrid.__init__, ifim._HostResult.commit


def dg_init(self, *a, **k):
    t0 = time.perf_counter()
    orig_dg(self, *a, **k)
    torch.cuda.synchronize()
    T["upload"] = time.perf_counter() - t0


def commit(self):
    t0 = time.perf_counter()
    r = orig_commit(self)
    T["commit"] = time.perf_counter() - t0
    return r


ifim._DeviceGrid.__init__ = dg_init
ifim._HostResult.commit = commit
for it in range(5):
    phi.fill_(float("inf"))
    state.zero_()
    g = w.grid(eik, phi, speed, state)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = eik.solve_ifim(g, bc)
    tot = time.perf_counter() - t0
    print(f"total {tot*1e3:.1f} ms  upload {T['upload']*1e3:.1f}  device {res.stats.device_ms['total']:.1f}  "
          f"commit {T['commit']*1e3:.1f}  other {(tot - T['upload'] - T['commit'])*1e3 - res.stats.device_ms['total']:.1f}")
