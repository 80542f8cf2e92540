"""Where the end-to-end (host buffers) time of one 512^3 solve goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_15869_b200 as eik  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = np.arange(n) // (n // 16)
F = np.where(((k[:, None, None] + k[None, :, None] + k[None, None, :]) % 2) == 0, 1.0, 0.01)
speed = torch.from_numpy(F).pin_memory()
phi = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
state = torch.empty((n, n, n), dtype=torch.uint8).pin_memory()
c = n // 2
bc = eik.BoundaryCondition(((eik.CellIndex3D(c, c, c), 0.0),))
print("torch threads", torch.get_num_threads(), "cpus", os.cpu_count())
for it in range(3):
    phi.fill_(float("inf"))
    state.zero_()
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), phi, speed, state)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = [x.to("cuda", non_blocking=True) for x in (phi, speed, state)]
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    phi.copy_(d[0], non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cl = phi.clone()
    t3 = time.perf_counter()
    res = eik.solve_ifim(g, bc)
    t4 = time.perf_counter()
    print(f"h2d {1e3 * (t1 - t0):.1f} ms  d2h {1e3 * (t2 - t1):.1f} ms  clone {1e3 * (t3 - t2):.1f} ms  "
          f"solve_ifim wall {1e3 * (t4 - t3):.1f} ms (device {res.stats.device_ms['total']:.1f})", flush=True)

# internal split of one host-grid solve_ifim
import ctypes as C  # noqa: E402
from paper_2106_15869_b200 import _native, ifim  # noqa: E402

for it in range(3):
    res = r = dg = out = None
    phi.fill_(float("inf"))
    state.zero_()
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), phi, speed, state)
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    idx, val = eik.seed_linear(g, bc)
    dg = ifim._DeviceGrid(g)
    geom = ifim.geometry(g)
    ws = ifim.workspace(geom, dg.device)
    si = torch.as_tensor(idx, dtype=torch.int64, device=dg.device)
    sv = torch.as_tensor(val, dtype=torch.float64, device=dg.device)
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    hcap = ifim._history_cap(geom)
    hist = np.zeros(hcap, dtype=np.int64)
    st = _native.Stats()
    out = ifim._HostResult(dg)
    rc = _native.lib().eik_ifim_solve(C.byref(geom), ifim._ptr(dg.phi), ifim._ptr(dg.speed), ifim._ptr(dg.state),
                                      ifim._ptr(si), ifim._ptr(sv), len(idx), 1e-12, ws.ptr, ws.nbytes,
                                      hist.ctypes.data_as(C.c_void_p), hcap, C.byref(st), dg.stream)
    T.append(time.perf_counter())
    out.thread.join()
    T.append(time.perf_counter())
    r = out.commit()
    T.append(time.perf_counter())
    print("upload+setup %.1f  engine call %.1f (device %.1f)  join %.1f  commit %.1f ms" % tuple(
        [1e3 * (T[1] - T[0]), 1e3 * (T[2] - T[1]), st.total_ms, 1e3 * (T[3] - T[2]), 1e3 * (T[4] - T[3])]))
