"""z-slab domain decomposition of the iFIM solve.

Rank q of R owns the planes ``[z0, z1)`` of a 3D grid (2D grids are split
along y, the slowest axis, the same way).  Each rank stores its planes plus one
ghost plane on each side; ghosts are never computed, only read.  The solve is
the reference's set-valued Jacobi iteration (E/ifim.py:75-218) executed in
bulk-synchronous steps, with exactly one exchange per update iteration /
remedy round:

update iteration k (E/ifim.py:107-132)
    local:    solve every owned active cell from the snapshot, write, decide
              converged/stay, activate owned +inf FAR neighbours; a converged
              cell whose neighbour lies in a ghost plane and reads +inf there
              records an *activation request* for that cell.
    exchange: (1) the owned boundary planes of phi (after the iteration) go to
              the neighbours' ghost planes; (2) activation requests go to the
              owner, which activates the cell iff it is still FAR and not
              blocked (the requester's +inf test used the same snapshot value
              the owner has).
    reduce:   |A_{k+1}| = sum over ranks  (termination + active_history).
build (E/ifim.py:137-161)
    local flags on owned free cells (ghosts current); reduce |R_0|, #free.
remedy round r (E/ifim.py:186-216)
    local:    R_r = D_{r-1} | (N(D_{r-1}) & ~fixed) using the neighbours'
              boundary D planes as ghost bits, then solve the members.
    exchange: boundary phi planes and boundary D_r planes.
    reduce:   |R_r|, |D_r|  (termination when the global |D_r| is 0).

Because every step reads an immutable snapshot, the sets, the field and every
RunStats integer are identical for any number of slabs.  ``SlabSolver`` drives
any per-rank engine implementing the ``SlabEngine`` methods over any
communicator with ``exchange`` / ``allreduce_sum``; ``TorchDistComm`` uses
torch.distributed (NCCL for CUDA tensors, gloo for CPU tensors).
"""
from __future__ import annotations

from dataclasses import dataclass, field


from .result import RunStats


@dataclass(frozen=True)
class SlabPartition:
    """Balanced contiguous split of ``n`` planes over ``world`` ranks."""

    n: int
    world: int

    def bounds(self, rank: int) -> tuple[int, int]:
        if not 0 <= rank < self.world:
            raise ValueError(f"rank {rank} outside world {self.world}")
        if self.world > self.n:
            raise ValueError(f"cannot split {self.n} planes over {self.world} ranks")
        base, extra = divmod(self.n, self.world)
        z0 = rank * base + min(rank, extra)
        return z0, z0 + base + (1 if rank < extra else 0)

    def owner(self, z: int) -> int:
        for r in range(self.world):
            z0, z1 = self.bounds(r)
            if z0 <= z < z1:
                return r
        raise ValueError(f"plane {z} outside 0..{self.n - 1}")


class SlabEngine:
    """Per-rank compute interface used by SlabSolver (see module docstring)."""

    def boundary_planes(self):  # -> (lo_phi, hi_phi): owned planes z0 and z1-1 (current values)
        raise NotImplementedError

    def set_ghosts(self, lo_phi, hi_phi):  # ghost planes z0-1, z1 (None at the global border)
        raise NotImplementedError

    def init_active(self, seeds) -> int:  # apply all seeds, activate owned neighbours; returns |A_1| local
        raise NotImplementedError

    def update_local(self):  # one iteration; returns (requests_lo, requests_hi) bit planes
        raise NotImplementedError

    def apply_requests(self, req_from_lo, req_from_hi) -> int:  # returns local |A_{k+1}|
        raise NotImplementedError

    def build_local(self) -> tuple[int, int]:  # (#free, |R_0|) local
        raise NotImplementedError

    def remedy_boundary_d(self):  # (lo_D, hi_D) bit planes of the last round
        raise NotImplementedError

    def remedy_local(self, ghost_d_lo, ghost_d_hi, first: bool) -> tuple[int, int]:  # (|R_r|, |D_r|) local
        raise NotImplementedError

    def result(self):  # owned phi planes
        raise NotImplementedError


class ThreadComm:
    """In-process communicator for R ranks driven by R host threads (lockstep
    emulation on one device or on the CPU; no kernel ever waits on another)."""

    def __init__(self, rank: int, shared: dict):
        self.rank = rank
        self.world = shared["world"]
        self.s = shared

    @staticmethod
    def make_shared(world: int) -> dict:
        import threading

        return {"world": world, "barrier": threading.Barrier(world), "slots": {}, "sums": [None] * world}

    def exchange(self, send_lo, send_hi, like):
        s, r = self.s, self.rank
        s["slots"][(r, "lo")] = send_lo  # travels to rank - 1
        s["slots"][(r, "hi")] = send_hi  # travels to rank + 1
        s["barrier"].wait()
        got_lo = s["slots"][(r - 1, "hi")] if r > 0 else None
        got_hi = s["slots"][(r + 1, "lo")] if r + 1 < self.world else None
        s["barrier"].wait()
        return got_lo, got_hi

    def allreduce_sum(self, values, device="cpu"):
        s = self.s
        s["sums"][self.rank] = list(values)
        s["barrier"].wait()
        out = [sum(v[i] for v in s["sums"]) for i in range(len(values))]
        s["barrier"].wait()
        return out


class TorchDistComm:
    """Neighbour exchange and sum-reduce over torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, send_lo, send_hi, like):
        """Send to rank-1 / rank+1, receive from them (None at the ends)."""
        import torch

        dist = self.dist
        ops, recv_lo, recv_hi = [], None, None
        if self.rank > 0:
            recv_lo = torch.empty_like(like)
            ops += [dist.P2POp(dist.isend, send_lo.contiguous(), self.rank - 1, self.group),
                    dist.P2POp(dist.irecv, recv_lo, self.rank - 1, self.group)]
        if self.rank + 1 < self.world:
            recv_hi = torch.empty_like(like)
            ops += [dist.P2POp(dist.isend, send_hi.contiguous(), self.rank + 1, self.group),
                    dist.P2POp(dist.irecv, recv_hi, self.rank + 1, self.group)]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return recv_lo, recv_hi

    def allreduce_sum(self, values, device="cpu"):
        import torch

        t = torch.tensor(values, dtype=torch.int64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return [int(v) for v in t.tolist()]


@dataclass
class SlabStats:
    update: RunStats = field(default_factory=lambda: RunStats(active_history=[]))
    build_calls: int = 0
    remedy_size: int = 0
    remedy: RunStats = field(default_factory=RunStats)


class SlabSolver:
    """Bulk-synchronous driver of the slab protocol (one exchange per step)."""

    def __init__(self, engine: SlabEngine, comm, caps: tuple[int, int], tensor_device="cpu"):
        self.e = engine
        self.c = comm
        self.cap_upd, self.cap_rem = caps
        self.dev = tensor_device

    def _refresh_ghosts(self):
        lo, hi = self.e.boundary_planes()
        got_lo, got_hi = self.c.exchange(lo, hi, lo)
        self.e.set_ghosts(got_lo, got_hi)

    def solve(self, seeds) -> SlabStats:
        st = SlabStats()
        n_local = self.e.init_active(seeds)  # applies the seeds (E/grid.py:212-215) first
        self._refresh_ghosts()
        n = self.c.allreduce_sum([n_local], self.dev)[0]
        up = st.update
        up.peak_active = n
        while n:
            up.iterations += 1
            if up.iterations > self.cap_upd:  # E/ifim.py:106-110
                raise RuntimeError(f"active list did not drain within {self.cap_upd} iterations")
            up.active_history.append(n)
            up.solver_calls += n
            req_lo, req_hi = self.e.update_local()
            self._refresh_ghosts()
            got_lo, got_hi = self.c.exchange(req_lo, req_hi, req_lo)
            n = self.c.allreduce_sum([self.e.apply_requests(got_lo, got_hi)], self.dev)[0]
            up.peak_active = max(up.peak_active, n)
        free, r0 = self.c.allreduce_sum(list(self.e.build_local()), self.dev)
        st.build_calls, st.remedy_size = free, r0
        rm = st.remedy
        rm.peak_remedy = r0
        first = True
        if r0:
            while True:
                rm.iterations += 1
                if rm.iterations > self.cap_rem:  # E/ifim.py:185-189
                    raise RuntimeError(f"remedy set did not drain within {self.cap_rem} rounds")
                d_lo, d_hi = self.e.remedy_boundary_d()
                g_lo, g_hi = self.c.exchange(d_lo, d_hi, d_lo)
                calls, decs = self.c.allreduce_sum(list(self.e.remedy_local(g_lo, g_hi, first)), self.dev)
                first = False
                rm.solver_calls += calls
                rm.peak_remedy = max(rm.peak_remedy, calls)
                self._refresh_ghosts()
                if decs == 0:
                    break
        return st

    @staticmethod
    def combine(st: SlabStats) -> RunStats:
        """solve_ifim's stats composition (E/ifim.py:227-233)."""
        return RunStats(
            iterations=st.update.iterations + st.remedy.iterations,
            solver_calls=st.update.solver_calls + st.build_calls + st.remedy.solver_calls,
            peak_active=st.update.peak_active,
            peak_remedy=st.remedy.peak_remedy,
            active_history=list(st.update.active_history),
        )
