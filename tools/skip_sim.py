"""Remedy solve-skip rule (design tool, not a test): python tools/skip_sim.py cfg4 128.
A member whose changed neighbours (D_{r-1}) leave every axis minimum unchanged cannot decrease
(its inputs equal those of its last evaluation); replays the rounds in numpy with the oracle's
solver, checks the rule never skips a decrease, and reports how often whole warps could skip."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from oracle import cpu
config = sys.argv[1]; n = int(sys.argv[2])
h, F, seeds = bench.workload_np(config, n)
F = np.ascontiguousarray(F, dtype=np.float64); shape = F.shape
phi = np.full(F.size, np.inf); state = np.zeros(F.size, dtype=np.uint8)
si = [(k * n + j) * n + i for i, j, k in seeds]
cpu.update_step(shape, h, phi, F.reshape(-1), state, si, [0.0] * len(si), threads=os.cpu_count())
member, _ = cpu.build_remedy(shape, h, phi, F.reshape(-1), state, threads=os.cpu_count())
phi = phi.reshape(shape); R = member.reshape(shape).astype(bool)
fixed = (state.reshape(shape) == 4) | (state.reshape(shape) == 2)
def sh(a, ax, s, fill):
    out = np.full_like(a, fill); src=[slice(None)]*3; dst=[slice(None)]*3
    if s > 0: src[ax], dst[ax] = slice(0, -s), slice(s, None)
    else: src[ax], dst[ax] = slice(-s, None), slice(0, s)
    out[tuple(dst)] = a[tuple(src)]; return out
Dprev = None; tot = 0; skp = 0; viol = 0; w32 = 0; w32all = 0; w32half = 0; rounds = 0
while R.any():
    idx = np.nonzero(R); m = idx[0].size; tot += m
    P = np.pad(phi, 1, constant_values=np.inf)
    k, j, i = idx[0] + 1, idx[1] + 1, idx[2] + 1
    px = np.minimum(P[k, j, i - 1], P[k, j, i + 1]); py = np.minimum(P[k, j - 1, i], P[k, j + 1, i]); pz = np.minimum(P[k - 1, j, i], P[k + 1, j, i])
    v = cpu.local_3d_uniform(px, py, pz, F[idx], np.full(m, h))
    old = phi[idx]; dec = v < old - 1e-12
    if Dprev is not None:
        Dp = np.pad(Dprev, 1, constant_values=False)
        clean = np.ones(m, dtype=bool)
        for (a, b) in [((k, j, i - 1), (k, j, i + 1)), ((k, j - 1, i), (k, j + 1, i)), ((k - 1, j, i), (k + 1, j, i))]:
            ca, cb = Dp[a], Dp[b]; va, vb = P[a], P[b]
            ok = (~ca & ~cb) | (ca & ~cb & (va >= vb)) | (cb & ~ca & (vb >= va))
            clean &= ok
        skp += clean.sum(); viol += (clean & dec).sum()
        order = np.argsort(np.ravel_multi_index(idx, shape))  # word order approx
        cl = clean[order]; g = cl[: (m // 32) * 32].reshape(-1, 32)
        w32 += g.shape[0]; w32all += g.all(axis=1).sum(); w32half += (g.sum(axis=1) >= 16).sum()
    D = np.zeros(shape, dtype=bool); D[tuple(a[dec] for a in idx)] = True
    phi[tuple(a[dec] for a in idx)] = v[dec]
    N = D.copy()
    for ax in range(3): N |= sh(D, ax, 1, False) | sh(D, ax, -1, False)
    R = D | (N & ~fixed); Dprev = D; rounds += 1
print(f"{config} n={n} rounds={rounds} members={tot} skippable={skp} ({skp/tot:.3f}) violations={viol} warps={w32} all-skip={w32all/max(w32,1):.3f} >=half={w32half/max(w32,1):.3f}")
