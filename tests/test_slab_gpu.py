"""Slab-sharded solves with the B200 engine in slab mode, R ranks emulated in
lockstep on one GPU (host threads + ThreadComm; no kernel waits on another),
bit-identical to the single-domain solve and to the oracle."""
import threading

import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik
from oracle import cpu
from paper_2106_15869_b200.slab import SlabSolver, ThreadComm
from paper_2106_15869_b200.slab_gpu import solve_ifim_slabs

pytestmark = pytest.mark.gpu


def problem(kind):
    rng = np.random.default_rng(11)
    if kind == "checker":
        nz, ny, nx = 24, 20, 40
        kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
        F = np.where(((ii // 4) + (jj // 4) + (kk // 4)) % 2 == 0, 1.0, 0.01)
    elif kind == "walls":
        nz, ny, nx = 13, 16, 37
        kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
        F = np.exp(0.5 * np.sin(0.5 * ii) * np.cos(0.3 * jj + 0.2 * kk))
        F[6, 3:14, 2:30] = 0.0
        F[3, 0:10, 10:12] = 0.0
    else:
        nz, ny, nx = 20, 18, 33
        F = np.ones((nz, ny, nx))
    free = np.flatnonzero(F.ravel() > 0)
    seeds = [(int(c), float(v)) for c, v in zip(rng.choice(free, 4, replace=False), (0.0, 0.3, 0.0, 1.0))]
    state = np.where(F == 0, 4, 0).astype(np.uint8)
    return (nz, ny, nx), 0.5, F, state, seeds


@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("kind", ["checker", "walls", "const"])
def test_slab_ranks_bit_identical(world, kind):
    shape, h, F, state, seeds = problem(kind)
    ref = cpu.solve_ifim(shape, h, F, [c for c, _ in seeds], [v for _, v in seeds], state=state, threads=8)
    shared = ThreadComm.make_shared(world)
    out, err = [None] * world, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            out[r] = solve_ifim_slabs(shape, h, F, state, seeds, ThreadComm(r, shared))
            torch.cuda.synchronize()
        except Exception as ex:  # pragma: no cover
            err.append(ex)
            shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not err, err
    phi = torch.cat([o[0] for o in out], dim=0).cpu().numpy()
    assert np.array_equal(phi.view(np.uint64), ref.phi.view(np.uint64))
    st = SlabSolver.combine(out[0][1])
    assert (st.iterations, st.solver_calls, st.peak_active, st.peak_remedy) == (
        ref.stats["iterations"], ref.stats["solver_calls"], ref.stats["peak_active"], ref.stats["peak_remedy"])
    assert st.active_history == ref.active_history
