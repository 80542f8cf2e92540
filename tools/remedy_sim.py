"""Remedy-round statistics on the CPU (design tool, not a test): python tools/remedy_sim.py [config] n

Runs the oracle's update step and build pass, then replays the remedy rounds (E/ifim.py:191-216) in
numpy with the oracle's batched 3D solver, and reports per-round brick occupancy: how many bricks of
a given shape hold members, and the member density inside them.  Used to size the brick engine."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import cpu  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 2 else "cfg4"
n = int(sys.argv[-1])
h, F, seeds = bench.workload_np(config, n)
F = np.ascontiguousarray(F, dtype=np.float64)
shape = F.shape
phi = np.full(F.size, np.inf)
state = np.zeros(F.size, dtype=np.uint8)
si = [(k * n + j) * n + i for i, j, k in seeds]
cpu.update_step(shape, h, phi, F.reshape(-1), state, si, [0.0] * len(si), threads=os.cpu_count())
member, _ = cpu.build_remedy(shape, h, phi, F.reshape(-1), state, threads=os.cpu_count())
phi = phi.reshape(shape)
R = member.reshape(shape).astype(bool)
fixed = (state.reshape(shape) == 4) | (state.reshape(shape) == 2)
d = h / F
BR = [(8, 8, 32), (4, 4, 32), (16, 16, 32), (8, 16, 16)]


def shifted(a, axis, s, fill):
    out = np.full_like(a, fill)
    src = [slice(None)] * 3
    dst = [slice(None)] * 3
    if s > 0:
        src[axis], dst[axis] = slice(0, -s), slice(s, None)
    else:
        src[axis], dst[axis] = slice(-s, None), slice(0, s)
    out[tuple(dst)] = a[tuple(src)]
    return out


rounds = 0
tot = 0
stats = {b: [0, 0, 0] for b in BR}  # active bricks, members, brick-cells
big = {b: [0, 0, 0] for b in BR}
while R.any():
    idx = np.nonzero(R)
    m = idx[0].size
    tot += m
    P = np.pad(phi, 1, constant_values=np.inf)
    k, j, i = idx[0] + 1, idx[1] + 1, idx[2] + 1
    px = np.minimum(P[k, j, i - 1], P[k, j, i + 1])
    py = np.minimum(P[k, j - 1, i], P[k, j + 1, i])
    pz = np.minimum(P[k - 1, j, i], P[k + 1, j, i])
    v = cpu.local_3d_uniform(px, py, pz, F[idx], np.full(m, h))
    old = phi[idx]
    dec = v < old - 1e-12
    D = np.zeros(shape, dtype=bool)
    D[tuple(a[dec] for a in idx)] = True
    phi[tuple(a[dec] for a in idx)] = v[dec]
    for b in BR:
        bz, by, bx = b
        occ = R.reshape(n // bz, bz, n // by, by, n // bx, bx).sum(axis=(1, 3, 5))
        act = (occ > 0).sum()
        stats[b][0] += act
        stats[b][1] += m
        stats[b][2] += act * bz * by * bx
        if m >= n ** 3 // 8:
            big[b][0] += act
            big[b][1] += m
            big[b][2] += act * bz * by * bx
    N = D.copy()
    for ax in range(3):
        N |= shifted(D, ax, 1, False) | shifted(D, ax, -1, False)
    R = D | (N & ~fixed)
    rounds += 1
print(f"{config} n={n}: rounds={rounds} members={tot} ({tot / n ** 3:.1f} per cell)")
for b in BR:
    a, mm, c = stats[b]
    ab, mb, cb = big[b]
    print(f"  brick z{b[0]}y{b[1]}x{b[2]}: active-brick-rounds={a} density={mm / max(c, 1):.3f} "
          f"members/active brick={mm / max(a, 1):.0f}; big rounds (|R|>=N/8): density={mb / max(cb, 1):.3f} "
          f"share of members={mb / max(mm, 1):.2f}")
