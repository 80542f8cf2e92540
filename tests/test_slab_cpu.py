"""Slab decomposition protocol (paper_2106_15869_b200/slab.py) on the CPU:
sharded solves are bit-identical to the single-domain oracle, over gloo
(world_size 2, separate processes) and over the in-process ThreadComm."""
import os
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu
from paper_2106_15869_b200.slab import SlabPartition, SlabSolver, ThreadComm, TorchDistComm
from slab_cpu_engine import CpuSlabEngine


def problem(kind="checker"):
    rng = np.random.default_rng(7)
    nz, ny, nx = 9, 10, 12
    kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
    if kind == "checker":
        F = np.where(((ii // 3) + (jj // 3) + (kk // 3)) % 2 == 0, 1.0, 0.01)
    else:
        F = np.exp(0.5 * np.sin(0.7 * ii) * np.cos(0.4 * jj + 0.3 * kk))
        F[4, 2:8, 1:9] = 0.0
    free = np.flatnonzero(F.ravel() > 0)
    seeds = [(int(c), float(v)) for c, v in zip(rng.choice(free, 3, replace=False), (0.0, 0.5, 1.25))]
    state = np.where(F == 0, 4, 0).astype(np.uint8)
    return (nz, ny, nx), 0.7, F, state, seeds


def reference(shape, h, F, state, seeds):
    return cpu.solve_ifim(shape, h, F, [c for c, _ in seeds], [v for _, v in seeds], state=state)


def caps(shape):
    s = sum(shape)
    return 40 * s, 20 * s


def check(shape, ref, phi, stats):
    assert np.array_equal(phi.view(np.uint64), ref.phi.view(np.uint64))
    st = SlabSolver.combine(stats)
    assert (st.iterations, st.solver_calls, st.peak_active, st.peak_remedy) == (
        ref.stats["iterations"], ref.stats["solver_calls"], ref.stats["peak_active"], ref.stats["peak_remedy"])
    assert st.active_history == ref.active_history


def test_partition():
    p = SlabPartition(10, 3)
    assert [p.bounds(r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert p.owner(6) == 1 and p.owner(9) == 2
    with pytest.raises(ValueError):
        SlabPartition(2, 3).bounds(0)


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("kind", ["checker", "smooth"])
def test_thread_ranks_bit_identical(world, kind):
    shape, h, F, state, seeds = problem(kind)
    ref = reference(shape, h, F, state, seeds)
    part = SlabPartition(shape[0], world)
    shared = ThreadComm.make_shared(world)
    out = [None] * world
    err = []

    def run(r):
        try:
            z0, z1 = part.bounds(r)
            e = CpuSlabEngine(shape, h, F, state, z0, z1)
            st = SlabSolver(e, ThreadComm(r, shared), caps(shape)).solve(seeds)
            out[r] = (e.result(), st)
        except Exception as ex:  # pragma: no cover - surfaced below
            err.append(ex)
            shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not err, err
    phi = np.concatenate([o[0] for o in out], axis=0)
    check(shape, ref, phi, out[0][1])
    assert all(o[1] == out[0][1] for o in out)  # every rank agrees on the global stats


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape, h, F, state, seeds = problem("checker")
        z0, z1 = SlabPartition(shape[0], world).bounds(rank)
        e = CpuSlabEngine(shape, h, F, state, z0, z1)
        st = SlabSolver(e, TorchDistComm(), caps(shape)).solve(seeds)
        q.put((rank, e.result(), st))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bit_identical():
    import random

    world = 2
    port = 29500 + random.randint(0, 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    [p.join(timeout=60) for p in procs]
    shape, h, F, state, seeds = problem("checker")
    ref = reference(shape, h, F, state, seeds)
    phi = np.concatenate([r[1] for r in res], axis=0)
    check(shape, ref, phi, res[0][2])
