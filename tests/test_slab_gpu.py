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


class _GlooCudaComm:
    """TorchDistComm over gloo for CUDA planes: the exchange stages them through host memory."""

    def __init__(self):
        from paper_2106_15869_b200.slab import TorchDistComm

        self.c = TorchDistComm()
        self.rank, self.world = self.c.rank, self.c.world

    def exchange(self, send_lo, send_hi, like):
        dev = like.device
        cpu_ = lambda t: t.cpu() if t is not None else None  # noqa: E731
        lo, hi = self.c.exchange(cpu_(send_lo), cpu_(send_hi), like.cpu())
        return (lo.to(dev) if lo is not None else None), (hi.to(dev) if hi is not None else None)

    def allreduce_sum(self, values, device="cpu"):
        return self.c.allreduce_sum(values, "cpu")


def _gloo_gpu_worker(rank, world, port, kind, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        shape, h, F, state, seeds = problem(kind)
        phi, st = solve_ifim_slabs(shape, h, F, state, seeds, _GlooCudaComm())
        torch.cuda.synchronize()
        q.put((rank, phi.cpu().numpy(), SlabSolver.combine(st)))
    except Exception as ex:  # pragma: no cover
        q.put((rank, None, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["checker", "walls"])
def test_slab_two_processes_gloo(kind):
    """Two OS processes (torch.distributed, gloo), each running the B200 slab kernels for its
    z-slab and exchanging ghost planes / activation requests / decrease planes through the
    host-driven protocol: the multi-process path a multi-GPU run takes, with both ranks on one
    device (every step's kernels complete before the exchange, so no kernel waits on another)."""
    import multiprocessing as mp
    import random

    world = 2
    port = 31000 + random.randint(0, 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_gpu_worker, args=(r, world, port, kind, q)) for r in range(world)]
    [p.start() for p in procs]
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    [p.join(timeout=60) for p in procs]
    assert all(r[1] is not None for r in res), res
    shape, h, F, state, seeds = problem(kind)
    ref = cpu.solve_ifim(shape, h, F, [c for c, _ in seeds], [v for _, v in seeds], state=state, threads=8)
    phi = np.concatenate([r[1] for r in res], axis=0)
    assert np.array_equal(phi.view(np.uint64), ref.phi.view(np.uint64))
    for _, _, st in res:  # every rank holds the global stats
        assert (st.iterations, st.solver_calls, st.peak_active, st.peak_remedy) == (
            ref.stats["iterations"], ref.stats["solver_calls"], ref.stats["peak_active"], ref.stats["peak_remedy"])
        assert st.active_history == ref.active_history
