#!/usr/bin/env python
"""Benchmark of the iFIM hot path (BASELINE.json metric: grid-node updates/s and
wall-clock to convergence, 3D 512^3).

Workload: 3D 512^3, h = 1, checkerboard speed of 32^3
blocks, F = 1 where (i//32 + j//32 + k//32) is even else 0.01 (the paper's 1:100
ratio), one point seed (value 0) at the centre (256, 256, 256).

A step = one complete solve_ifim (update step + build pass + remedy step) on a
fresh field: phi = +inf and state = FAR/BLOCKED are restored from resident
device copies at the start of every step (inside the timed region).
Node updates = RunStats.solver_calls (identical to the reference's count,
SURVEY.md §8d).  `value` = total node updates / device time over all ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--size 512] [--impl ours|reference]

N > 1 (torchrun): ONE 512^3 grid is z-slab sharded over the ranks (strong
scaling), by default in the fused peer-memory kernels
(paper_2106_15869_b200/slab_peer.py: neighbour planes read over NVLink inside
the persistent kernels, device-side cross-rank barrier); --host-slabs selects
the host-driven protocol (paper_2106_15869_b200/slab.py: one ghost-plane /
request / decrease-plane exchange per step over NCCL).  The time is the max
over ranks.  --slabs runs that protocol on one GPU.  --impl reference
times the CPU oracle port of the reference algorithm (oracle/eik_oracle.c,
OpenMP on all host cores) on a bounded sample of the same workload family.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
METRIC = "grid-node updates/sec (and wall-clock to convergence), 3D 512^3"
UNIT = "node-updates/s"


class Workload:
    """One BASELINE.json config: speed field (device tensor), spacing, point seeds ((i, j) or
    (i, j, k)); 2D configs are n^2, 3D configs n^3."""

    def __init__(self, name, n, h, F, seeds, desc):
        self.name, self.n, self.h, self.F, self.seeds, self.desc = name, n, h, F, seeds, desc
        self.ndim = F.dim()
        self.shape = tuple(F.shape)
        self.cells = int(np.prod(self.shape))

    def linear_seeds(self):
        n = self.n
        if self.ndim == 2:
            return [(j * n + i, 0.0) for i, j in self.seeds]
        return [((k * n + j) * n + i, 0.0) for i, j, k in self.seeds]

    def spacing(self):
        return (self.h, self.h) if self.ndim == 2 else self.h

    def grid(self, eik, phi, F, state):
        n = self.n
        if self.ndim == 2:
            return eik.Grid(n, n, self.h, self.h, (0.0, 0.0), phi, F, state)
        return eik.Grid3D(n, n, n, self.h, (0.0, 0.0, 0.0), phi, F, state)

    def bc(self, eik):
        idx = eik.CellIndex if self.ndim == 2 else eik.CellIndex3D
        return eik.BoundaryCondition(tuple((idx(*s), 0.0) for s in self.seeds))


def cfg5_modes(n):
    """cfg5 (SURVEY.md §8d / BASELINE.md): g = unit-variance sum of 32 Fourier modes with integer
    wavevectors 0 < |k| <= 4 and uniform phases, 16 distinct seeds; all from default_rng(2106)."""
    import itertools

    rng = np.random.default_rng(2106)
    ks = np.array([k for k in itertools.product(range(-4, 5), repeat=3) if 0 < sum(v * v for v in k) <= 16])
    K = ks[rng.choice(len(ks), 32, replace=False)]
    ph = rng.uniform(0.0, 2.0 * np.pi, 32)
    seeds = []
    while len(seeds) < 16:
        s = tuple(int(v) for v in rng.integers(0, n, 3))
        if s not in seeds:
            seeds.append(s)
    return K, ph, seeds


def cfg5_speed(torch, dev, n):
    """F = exp(0.5 g) on [0,1]^3 (h = 1/(n-1)), built plane-chunk by plane-chunk on the device."""
    K, ph, seeds = cfg5_modes(n)
    h = 1.0 / (n - 1)
    x = torch.arange(n, dtype=torch.float64, device=dev) * h
    F = torch.empty((n, n, n), dtype=torch.float64, device=dev)
    zc = max(1, (1 << 26) // (n * n))
    for z0 in range(0, n, zc):
        z1 = min(n, z0 + zc)
        g = torch.zeros((z1 - z0, n, n), dtype=torch.float64, device=dev)
        for (kx, ky, kz), p in zip(K.tolist(), ph.tolist()):
            a = 2 * np.pi * (kz * x[z0:z1])[:, None, None] + (2 * np.pi * ky * x)[None, :, None] + \
                (2 * np.pi * kx * x + p)[None, None, :]
            g += torch.cos(a)
        F[z0:z1] = torch.exp(0.5 * 0.25 * g)  # sqrt(2/32) = 0.25: unit variance
    return F, h, seeds


def workload_desc(config, n):
    if config == "cfg1":
        return f"cfg1: 2D {n}^2 F=1, h=1, centre seed"
    if config == "cfg2":
        return f"cfg2: 2D {n}^2 on [0,1]^2, F=1+0.5 sin(2 pi x) sin(2 pi y), 8 seeds (rng 2106)"
    if config == "cfg5":
        return f"cfg5: 3D {n}^3 on [0,1]^3, F=exp(0.5 g) (32 Fourier modes |k|<=4, rng 2106), 16 seeds"
    if config == "cfg3":
        return f"cfg3: 3D {n}^3 F=1, h=1, 16 random seeds (rng 2106)"
    return f"cfg4: 3D {n}^3 checkerboard 1:100 ({max(1, n // 16)}^3 blocks), h=1, seed (c,c,c)"


def _distinct_cells(rng, n, k, dim):
    out = []
    while len(out) < k:
        c = tuple(int(v) for v in rng.integers(0, n, dim))
        if c not in out:
            out.append(c)
    return out


def cfg5_speed_np(n):
    """cfg5's F = exp(0.5 g) on the host (numpy, plane chunks on a thread pool: the ufuncs
    release the GIL), same expression order as cfg5_speed."""
    from concurrent.futures import ThreadPoolExecutor

    K, ph, seeds = cfg5_modes(n)
    h = 1.0 / (n - 1)
    x = np.arange(n, dtype=np.float64) * h
    F = np.empty((n, n, n), dtype=np.float64)
    zc = max(1, (1 << 21) // (n * n))

    def chunk(z0):
        z1 = min(n, z0 + zc)
        g = np.zeros((z1 - z0, n, n), dtype=np.float64)
        for (kx, ky, kz), p in zip(K.tolist(), ph.tolist()):
            a = 2 * np.pi * (kz * x[z0:z1])[:, None, None] + (2 * np.pi * ky * x)[None, :, None] + \
                (2 * np.pi * kx * x + p)[None, None, :]
            g += np.cos(a)
        F[z0:z1] = np.exp(0.5 * 0.25 * g)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        list(ex.map(chunk, range(0, n, zc)))
    return F, h, seeds


# cfg5 fields up to this edge are built on the host with numpy (bit-identical to the field the
# full-size oracle digests in tests/golden/fullsize.json were computed on); larger ones on the
# device with torch (CUDA cos/exp may differ from numpy's in the last bit)
CFG5_HOST_MAX = 512


def workload_np(config, n):
    """(h, F, seeds) of one BASELINE.json config built on the host with numpy.  Every field here
    is bit-identical to what the oracle digests (tests/golden/make_fullsize.py) used."""
    if config == "cfg1":
        return 1.0, np.ones((n, n)), [(n // 2, n // 2)]
    if config == "cfg2":
        h = 1.0 / (n - 1)
        x = np.arange(n, dtype=np.float64) * h
        F = 1 + 0.5 * np.sin(2 * np.pi * x)[None, :] * np.sin(2 * np.pi * x)[:, None]
        return h, F, _distinct_cells(np.random.default_rng(2106), n, 8, 2)
    if config == "cfg3":
        return 1.0, np.ones((n, n, n)), _distinct_cells(np.random.default_rng(2106), n, 16, 3)
    if config == "cfg5":
        F, h, seeds = cfg5_speed_np(n)
        return h, F, seeds
    blk = max(1, n // 16)
    kk = np.arange(n) // blk
    F = np.where(((kk[:, None, None] + kk[None, :, None] + kk[None, None, :]) % 2) == 0, 1.0, 0.01)
    c = n // 2
    return 1.0, F, [(c, c, c)]


def make_workload(torch, dev, config, n):
    if config == "cfg5" and n > CFG5_HOST_MAX:
        F, h, seeds = cfg5_speed(torch, dev, n)
        return Workload("cfg5", n, h, F, seeds, workload_desc(config, n))
    h, F, seeds = workload_np(config, n)
    return Workload(config, n, h, torch.from_numpy(np.ascontiguousarray(F)).to(dev), seeds,
                    workload_desc(config, n))


def hbm_peak():
    try:
        with open(PEAKS_FILE) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_from_profiles(workload: str, kernel: str = "k_remedy"):
    """dram bytes per launch of the remedy kernel from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        for e in (d.get("kernels", {}).get(kernel, {}), *d.get("captures", {}).get(kernel, [])):
            if e.get("workload") == workload:
                return float(e["dram_bytes_read"]) + float(e["dram_bytes_write"])
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx.append(float(f[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# bounded CPU samples (~10-20 s of work on 8-16 host cores): the oracle port's edge per config, and
# the Python reference's (2D only, one core: the GIL) for the reference arm
CPU_SIZE = {"cfg1": 256, "cfg2": 2048, "cfg3": 256, "cfg4": 144, "cfg5": 128}
PYREF_SIZE = {"cfg1": 256, "cfg2": 512}
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def sample_label(config, n):
    return f"{n}^2" if config in ("cfg1", "cfg2") else f"{n}^3"


def cpu_sample(n: int, threads: int, config: str = "cfg4"):
    """Oracle port (C, OpenMP) on the same workload at edge n; returns (calls, seconds, threads)."""
    from oracle import cpu

    cpu.build()
    h, F, seeds = workload_np(config, n)
    F = np.ascontiguousarray(F)
    sd = Workload(config, n, h, _NpShape(F), seeds, "").linear_seeds()
    if F.size < (1 << 20):
        threads = 1  # small grids: per-iteration thread fan-out costs more than it saves
    t0 = time.perf_counter()
    res = cpu.solve_ifim(F.shape, (h, h) if F.ndim == 2 else h, F, [c for c, _ in sd], [v for _, v in sd],
                         threads=threads)
    dt = time.perf_counter() - t0
    return res.stats["solver_calls"], dt, threads


class _NpShape:
    """Just enough of a tensor for Workload's bookkeeping."""

    def __init__(self, a):
        self.shape = a.shape

    def dim(self):
        return len(self.shape)


def pyref_sample(n: int, config: str):
    """The reference's own solve_ifim (the unmodified package installed in baseline/_ref, its public
    API, workers=1) on a 2D config at edge n; returns (calls, seconds) or None if unavailable."""
    if config not in PYREF_SIZE or not os.path.isdir(os.path.join(REF_DIR, "eikonal")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from eikonal.grid import BoundaryCondition, CellIndex, new_grid
    from eikonal.ifim import solve_ifim

    h, F, seeds = workload_np(config, n)
    g = new_grid(n, n, h, h, origin=(0.0, 0.0), speed=np.ascontiguousarray(F))
    bc = BoundaryCondition(tuple((CellIndex(i, j), 0.0) for i, j in seeds))
    t0 = time.perf_counter()
    res = solve_ifim(g, bc, workers=1)
    return res.stats.solver_calls, time.perf_counter() - t0


def full_size_oracle(config, n):
    """The oracle port's full-size solve time recorded with the digests (tests/golden/fullsize.json)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "fullsize.json")) as fh:
            rec = json.load(fh).get(f"{config}@{n}")
    except OSError:
        return None
    if not rec:
        return None
    o = rec["oracle"]
    return {"size": sample_label(config, n), "seconds": round(o["seconds"]["total"], 2),
            "value": o["calls_per_s"], "unit": UNIT, "threads": o["threads"], "kind": "port",
            "where": f"authoring container ({o['cpu_count']} cores), tests/golden/make_fullsize.py"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    """The reference arm: the reference's own implementation timed on this host.  2D configs run
    the unmodified Python package from baseline/_ref (kind "reference", one core: the GIL);
    3D configs (the reference has no 3D engine) run the oracle port of its
    algorithm (kind "port", OpenMP on every host core).  Each step is one full solve of a bounded
    sample of the configured workload."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    py = args.config in PYREF_SIZE and os.path.isdir(os.path.join(REF_DIR, "eikonal"))
    n = args.cpu_size or (PYREF_SIZE[args.config] if py else CPU_SIZE[args.config])

    def one():
        if py:
            c, s = pyref_sample(n, args.config)
            return c, s, 1
        return cpu_sample(n, threads, args.config)

    for _ in range(args.warmup):
        one()
    calls, secs, used = 0, 0.0, 1
    for _ in range(args.steps):
        c, s, used = one()
        calls += c
        secs += s
    v = calls / secs
    impl = ("reference eikonal.solve_ifim (baseline/_ref, unmodified, workers=1)" if py
            else f"oracle/eik_oracle.c (port of E/ifim.py), OpenMP x{used}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(args.config, args.size), "size": args.size,
                   "parallelism": "host threads", "sample_size": n, "implementation": impl},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": used, "kind": "reference" if py else "port",
                         "sample": f"full solve_ifim of {workload_desc(args.config, n)} (a bounded "
                                   f"{sample_label(args.config, n)} sample of the {sample_label(args.config, args.size)} "
                                   f"workload) with {impl}",
                         "full_size": full_size_oracle(args.config, args.size)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class StepStats:
    def __init__(self, calls, iterations, peak_remedy, rem_calls, rem_writes, rem_ms, launches, phase_ms):
        self.calls, self.iterations, self.peak_remedy = calls, iterations, peak_remedy
        self.rem_calls, self.rem_writes, self.rem_ms = rem_calls, rem_writes, rem_ms
        self.launches, self.phase_ms = launches, phase_ms


def make_fim_step(eik, torch, dev, w, dtype):
    """One device-resident solve_fim (the paper's FIM baseline, E/fim.py) of the whole grid.
    Its whole persistent kernel stands in for the roofline kernel: bytes = 8 x (2 calls + writes)."""
    F = w.F.to(dtype)
    phi0 = torch.full(w.shape, float("inf"), dtype=dtype, device=dev)
    st0 = torch.zeros(w.shape, dtype=torch.uint8, device=dev)
    phi, st = torch.empty_like(phi0), torch.empty_like(st0)
    g = w.grid(eik, phi, F, st)
    bc = w.bc(eik)

    def step():
        phi.copy_(phi0)
        st.copy_(st0)
        s = eik.solve_fim(g, bc).stats
        return StepStats(s.solver_calls, s.iterations, 0, s.solver_calls, s.phi_writes, s.device_ms["total"],
                         s.gpu_launches, {"fim": round(s.device_ms["total"], 3)})

    return step


def make_single_step(eik, torch, dev, w, dtype):
    """One device-resident solve_ifim of the whole grid (inputs restored in the step)."""
    F = w.F.to(dtype)
    phi0 = torch.full(w.shape, float("inf"), dtype=dtype, device=dev)
    st0 = torch.zeros(w.shape, dtype=torch.uint8, device=dev)
    phi, st = torch.empty_like(phi0), torch.empty_like(st0)
    g = w.grid(eik, phi, F, st)
    bc = w.bc(eik)

    def step():
        phi.copy_(phi0)
        st.copy_(st0)
        r = eik.solve_ifim(g, bc)
        s = r.stats
        ph = s.phases
        upd_writes = ph["update"]["solver_calls"] - ph["update"]["converged"]
        rem_writes = s.phi_writes - upd_writes
        st_ = StepStats(s.solver_calls, s.iterations, s.peak_remedy, ph["remedy"]["solver_calls"], rem_writes,
                        s.device_ms["remedy"], s.gpu_launches, {k: round(v, 3) for k, v in s.device_ms.items()})
        st_.run_stats, st_.phi = s, phi
        # per-phase algorithmic bytes (8 B x (2 calls + writes); build: 2 x 8 B per free cell)
        rs = phi.element_size()
        st_.phase_bytes = {"update": rs * (2 * ph["update"]["solver_calls"] + upd_writes),
                           "build": rs * 2 * ph["build"]["solver_calls"],
                           "remedy": rs * (2 * ph["remedy"]["solver_calls"] + rem_writes)}
        return st_

    return step


def make_slab_step(torch, dev, w, world, rank):
    """This rank's share of ONE z-sharded solve (paper_2106_15869_b200/slab.py protocol)."""
    from paper_2106_15869_b200.slab import SlabPartition, SlabSolver, ThreadComm, TorchDistComm
    from paper_2106_15869_b200.slab_gpu import SlabGpuEngine

    n, F = w.n, w.F
    comm = TorchDistComm() if world > 1 else ThreadComm(0, ThreadComm.make_shared(1))
    z0, z1 = SlabPartition(n, world).bounds(rank)
    st0 = torch.zeros((n, n, n), dtype=torch.uint8, device=dev)
    e = SlabGpuEngine((n, n, n), w.h, F, st0, z0, z1, dev)
    clean_state = e.state.clone()
    seeds = w.linear_seeds()
    caps = (40 * 3 * n, 20 * 3 * n)

    def step():
        e.phi.fill_(float("inf"))
        e.state.copy_(clean_state)
        e.reset_counters()
        ss = SlabSolver(e, comm, caps, tensor_device=dev).solve(seeds)
        s = SlabSolver.combine(ss)
        return StepStats(s.solver_calls, s.iterations, s.peak_remedy, e.rem_calls_local, e.rem_decs_local,
                         e.rem_ms, e.launches, {"remedy_kernels_local": round(e.rem_ms, 3)})

    return step


def peer_slabs_possible(torch, dev, world, local):
    """Every rank can map every other rank's memory (NVLink / NVSwitch), agreed over all ranks."""
    import torch.distributed as dist

    ok = 1
    try:
        import torch.distributed._symmetric_memory  # noqa: F401

        for o in range(torch.cuda.device_count()):
            if o != local and o < world and not torch.cuda.can_device_access_peer(local, o):
                ok = 0
    except Exception:
        ok = 0
    t = torch.tensor([ok], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def peer_slabs_verify(torch, dev, world, rank):
    """Small multi-rank solve through DistributedSlabs compared bit for bit (phi, stats) with a
    single-device solve of the same problem on this rank: guards the cross-GPU memory ordering
    before the timed run trusts it."""
    import paper_2106_15869_b200 as eik
    from paper_2106_15869_b200.slab import SlabPartition
    from paper_2106_15869_b200.slab_peer import DistributedSlabs

    n = max(32, 8 * world)
    k = torch.arange(n, device=dev) // 4
    F = torch.where(((k[:, None, None] + k[None, :, None] + k[None, None, :]) % 2) == 0,
                    torch.tensor(1.0, dtype=torch.float64), torch.tensor(0.02, dtype=torch.float64))
    seeds = [(3, 5, 2), (n - 4, n // 2, n - 3)]
    g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), torch.full((n, n, n), float("inf"), dtype=torch.float64,
                                                             device=dev),
                   F, torch.zeros((n, n, n), dtype=torch.uint8, device=dev))
    ref = eik.solve_ifim(g, eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in seeds)))
    z0, z1 = SlabPartition(n, world).bounds(rank)
    ds = DistributedSlabs((n, n, n), 1.0)
    st = torch.zeros((z1 - z0, n, n), dtype=torch.uint8, device=dev)
    phi, s = ds.solve(F[z0:z1].contiguous(), st, [((kk * n + j) * n + i, 0.0) for i, j, kk in seeds])
    same = torch.equal(phi, ref.phi[z0:z1]) and s.solver_calls == ref.stats.solver_calls and \
        s.active_history == ref.stats.active_history
    del ds
    return same


def make_peer_step(torch, dev, w, world, rank):
    """This rank's share of ONE z-sharded solve in the fused peer-memory kernels
    (paper_2106_15869_b200/slab_peer.py): neighbour planes read over NVLink inside the
    persistent kernels, one device-side cross-rank barrier per iteration."""
    from paper_2106_15869_b200.slab import SlabPartition
    from paper_2106_15869_b200.slab_peer import DistributedSlabs

    n = w.n
    ds = DistributedSlabs((n, n, n), w.h)
    z0, z1 = SlabPartition(n, world).bounds(rank)
    sp = w.F[z0:z1].contiguous()
    st0 = torch.zeros((z1 - z0, n, n), dtype=torch.uint8, device=dev)
    st = torch.empty_like(st0)
    seeds = w.linear_seeds()

    def step():
        st.copy_(st0)
        phi_l, s = ds.solve(sp, st, seeds)
        ph = s.phases
        upd_writes = ph["update"]["solver_calls"] - ph["update"]["converged"]
        rem_writes = s.phi_writes - upd_writes
        st_ = StepStats(s.solver_calls, s.iterations, s.peak_remedy, ph["remedy"]["solver_calls"], rem_writes,
                        s.device_ms["remedy"], s.gpu_launches, {k: round(v, 3) for k, v in s.device_ms.items()})
        st_.run_stats, st_.phi = s, phi_l
        # per-phase algorithmic bytes (8 B x (2 calls + writes); build: 2 x 8 B per free cell);
        # the peer-slab engine is float64
        rs = 8
        st_.phase_bytes = {"update": rs * (2 * ph["update"]["solver_calls"] + upd_writes),
                           "build": rs * 2 * ph["build"]["solver_calls"],
                           "remedy": rs * (2 * ph["remedy"]["solver_calls"] + rem_writes)}
        return st_

    return step


def run_e2e_peer(torch, dev, w, world, rank, calls, args):
    """e2e at N>1 through DistributedSlabs: every step uploads this rank's slab of phi / speed /
    state from pinned host memory, solves, and downloads its phi slab; wall time max over ranks."""
    import torch.distributed as dist

    from paper_2106_15869_b200.slab import SlabPartition
    from paper_2106_15869_b200.slab_peer import DistributedSlabs

    n = w.n
    z0, z1 = SlabPartition(n, world).bounds(rank)
    ds = DistributedSlabs((n, n, n), w.h)
    sp_h = w.F[z0:z1].cpu().pin_memory()
    phi_h = torch.full((z1 - z0, n, n), float("inf"), dtype=torch.float64).pin_memory()
    st_h = torch.zeros((z1 - z0, n, n), dtype=torch.uint8).pin_memory()
    out_h = torch.empty_like(phi_h).pin_memory()
    sp = torch.empty(sp_h.shape, dtype=torch.float64, device=dev)
    st = torch.empty(st_h.shape, dtype=torch.uint8, device=dev)
    seeds = w.linear_seeds()
    steps = max(1, min(args.steps, 3))
    tot = 0.0
    for it in range(steps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sp.copy_(sp_h, non_blocking=True)
        st.copy_(st_h, non_blocking=True)
        phi, s = ds.solve(sp, st, seeds, phi_local=phi_h)
        out_h.copy_(phi, non_blocking=True)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        assert s.solver_calls == calls
        if it > 0:
            tot += float(dt.item())
    per = (z1 - z0) * n * n
    return {"value": calls * steps / tot, "unit": UNIT, "h2d_bytes_per_step": per * (8 + 8 + 1),
            "d2h_bytes_per_step": per * 8, "steps": steps, "ms_per_step": tot / steps * 1e3,
            "note": "per rank (rank 0's slab); wall time max over ranks"}


FULLSIZE = os.path.join(ROOT, "tests", "golden", "fullsize.json")


FULLSIZE_GPU = os.path.join(ROOT, "tests", "golden", "fullsize_gpu.json")


def parity_vs_crosscheck(w, r, world, s):
    """Sizes without an oracle run (cfg5 at 1024^3): the phi digest (chunked device SHA-256) and
    every RunStats integer against tests/golden/fullsize_gpu.json, the digest three independent
    device implementations of the remedy agreed on (tools/make_gpu_crosscheck.py)."""
    import hashlib

    try:
        with open(FULLSIZE_GPU) as fh:
            rec = json.load(fh).get(f"{w.name}@{w.n}")
    except OSError:
        rec = None
    if rec is None or world > 1:
        return "unpinned", f"no full-size digest for {w.name}@{w.n}"
    from paper_2106_15869_b200.harness import field_digest

    if field_digest(w.F) != rec["speed_field_digest"]:
        return "unpinned", "speed field differs from the digested one"
    ph = s.phases
    got = {"iterations": s.iterations, "solver_calls": s.solver_calls, "peak_active": s.peak_active,
           "peak_remedy": s.peak_remedy, "phi_writes": s.phi_writes, "upd_iterations": ph["update"]["iterations"],
           "upd_calls": ph["update"]["solver_calls"], "frozen": ph["update"]["converged"],
           "build_calls": ph["build"]["solver_calls"], "remedy_size": ph["build"]["remedy_size"],
           "rem_iterations": ph["remedy"]["iterations"], "rem_calls": ph["remedy"]["solver_calls"],
           "active_history_sha256": hashlib.sha256(np.asarray(s.active_history, dtype=np.int64).tobytes()).hexdigest(),
           "phi_field_digest": field_digest(r.phi)}
    bad = [k for k in got if got[k] != rec[k]]
    if bad:
        return "mismatch", "; ".join(f"{k}: {got[k]} != {rec[k]}" for k in bad)
    return "crosscheck-match", (f"phi digest + {len(got) - 1} RunStats fields equal the GPU cross-check digest "
                                f"({w.name}@{w.n}: {' == '.join(rec['agreed_by'])}; no oracle run at this size)")


def parity_vs_oracle(torch, w, r, world, rank, dtype):
    """After the timed steps: the last solve's phi sha256 and every RunStats integer against the
    full-size oracle digests (tests/golden/fullsize.json, made by tests/golden/make_fullsize.py
    from oracle/eik_oracle.c, which is pinned to the live reference).  Peer slabs: rank 0 hashes
    the slabs in z order (received over the process group).  Returns (status, detail)."""
    import hashlib

    if dtype != "f64":
        return "not-applicable", "float32 perf mode (checked against float64 at max-rel 1e-5 in tests)"
    s = getattr(r, "run_stats", None)
    if s is None:
        return "not-checked", "host-driven slab protocol"
    try:
        with open(FULLSIZE) as fh:
            rec = json.load(fh).get(f"{w.name}@{w.n}")
    except OSError:
        rec = None
    if rec is None:
        return parity_vs_crosscheck(w, r, world, s)
    h = hashlib.sha256()
    if world > 1:
        import torch.distributed as dist

        if rank == 0:
            h.update(r.phi.cpu().numpy().tobytes())
            for src in range(1, world):
                n = torch.zeros(1, dtype=torch.int64, device=r.phi.device)
                dist.recv(n, src)
                buf = torch.empty(int(n.item()), dtype=torch.float64, device=r.phi.device)
                dist.recv(buf, src)
                h.update(buf.cpu().numpy().tobytes())
        else:
            dist.send(torch.tensor([r.phi.numel()], dtype=torch.int64, device=r.phi.device), 0)
            dist.send(r.phi.reshape(-1).contiguous(), 0)
            return None, None
        speed_ok = True  # each rank's slab of the same host-built field
    else:
        h.update(r.phi.cpu().numpy().tobytes())
        speed_ok = hashlib.sha256(w.F.cpu().numpy().tobytes()).hexdigest() == rec["speed_sha256"]
    ph = s.phases
    got = {"iterations": s.iterations, "solver_calls": s.solver_calls, "peak_active": s.peak_active,
           "peak_remedy": s.peak_remedy, "phi_writes": s.phi_writes,
           "upd_iterations": ph["update"]["iterations"], "upd_calls": ph["update"]["solver_calls"],
           "frozen": ph["update"]["converged"], "build_calls": ph["build"]["solver_calls"],
           "remedy_size": ph["build"]["remedy_size"], "rem_iterations": ph["remedy"]["iterations"],
           "rem_calls": ph["remedy"]["solver_calls"],
           "active_history_sha256": hashlib.sha256(np.asarray(s.active_history, dtype=np.int64).tobytes()).hexdigest(),
           "phi_sha256": h.hexdigest()}
    u, b, m = rec["update"], rec["build"], rec["remedy"]
    want = {**{k: rec["stats"][k] for k in ("iterations", "solver_calls", "peak_active", "peak_remedy", "phi_writes")},
            "upd_iterations": u["iterations"], "upd_calls": u["solver_calls"], "frozen": u["frozen"],
            "build_calls": b["calls"], "remedy_size": b["remedy_size"], "rem_iterations": m["iterations"],
            "rem_calls": m["solver_calls"], "active_history_sha256": u["active_history_sha256"],
            "phi_sha256": rec["phi_sha256"]}
    bad = [k for k in want if got[k] != want[k]]
    if not speed_ok:
        return "unpinned", "speed field differs from the digested one"
    if bad:
        return "mismatch", "; ".join(f"{k}: {got[k]} != {want[k]}" for k in bad)
    return "digest-match", f"phi sha256 + {len(want) - 1} RunStats fields equal the oracle's ({w.name}@{w.n})"


def run_ours(args):
    import torch

    world, rank, local = dist_setup()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.force_peer:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    import paper_2106_15869_b200 as eik

    n = args.size
    w = make_workload(torch, dev, args.config, n)
    workload = w.desc
    rdt = torch.float32 if args.dtype == "f32" else torch.float64
    rsize = 4 if args.dtype == "f32" else 8
    if (args.dtype == "f32" or args.method == "fim" or w.ndim == 2) and (world > 1 or args.slabs):
        raise SystemExit("the float32 perf mode, the FIM baseline and the 2D configs are single-device")
    slabs = world > 1 or args.slabs or args.force_peer
    mode = "single"
    if (world > 1 or args.force_peer) and not args.host_slabs:
        # the fused peer-memory kernels; any failure is fatal (--host-slabs selects the NCCL protocol)
        import torch.distributed as dist

        if not peer_slabs_possible(torch, dev, world, local):
            raise SystemExit("peer-memory slabs need P2P mappings between every pair of ranks' GPUs; "
                             "pass --host-slabs for the host-driven NCCL protocol")
        ok = torch.tensor([int(peer_slabs_verify(torch, dev, world, rank))], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not ok.item():
            raise SystemExit("peer-memory slabs disagree with the single-device solve (small verification grid)")
        step, mode = make_peer_step(torch, dev, w, world, rank), "peer"
    elif slabs:
        step, mode = make_slab_step(torch, dev, w, world, rank), "host"
    elif args.method == "fim":
        step = make_fim_step(eik, torch, dev, w, rdt)
    else:
        step = make_single_step(eik, torch, dev, w, rdt)

    for _ in range(args.warmup):
        r = step()
    torch.cuda.synchronize()
    from paper_2106_15869_b200 import _native as _nat

    # which remedy engine ran (member list / TMA brick pipeline, chosen on the device from |R_0|)
    remedy_engine = _nat.last_remedy_engine(_nat.EIK_F32 if args.dtype == "f32" else _nat.EIK_F64) \
        if mode == "single" and args.method == "ifim" else ("list (peer slabs)" if mode != "single" else None)
    calls = r.calls
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rem_ms, launches = [], 0
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = step()
            rem_ms.append(r.rem_ms)
            launches += r.launches
            assert r.calls == calls
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    # slabs: ONE grid sharded over all ranks (strong scaling)
    value = calls * args.steps / (ms / 1e3)
    clocks = clk.summary()

    # roofline of the dominant kernel (k_remedy, this rank): algorithmic bytes (SURVEY.md §8d:
    # 8 B x (2 x solver_calls + phi_writes) of the remedy phase) / its CUDA-event duration.
    # Peer mode: the counts are global and the ranks run in lockstep, so the figure is the
    # aggregate over the ranks against the aggregate peak.
    alg_bytes = float(rsize) * (2 * r.rem_calls + r.rem_writes)
    rem_s = statistics.median(rem_ms) / 1e3
    peak, peak_src = hbm_peak()
    if mode == "peer":
        peak, peak_src = peak * world, peak_src + f" x {world} ranks"
    achieved = alg_bytes / rem_s / 1e9 if rem_s > 0 else None
    rem_kernel = "k_fim" if args.method == "fim" else ("k_remedy_b" if remedy_engine == "brick" else "k_remedy")
    traffic = traffic_from_profiles(workload, rem_kernel) if not slabs and args.dtype == "f64" and args.method == "ifim" \
        else None

    parity, parity_detail = parity_vs_oracle(torch, w, r, world, rank, args.dtype) if args.method == "ifim" \
        else ("not-checked", "FIM baseline (bit-exact vs the oracle in tests/test_gpu_fim.py)")
    out = None
    e2e_peer = None
    if mode == "peer" and not args.no_e2e:  # collective: every rank takes part
        try:
            e2e_peer = run_e2e_peer(torch, dev, w, world, rank, calls, args)
        except Exception as e:  # noqa: BLE001
            print(f"[bench] peer e2e failed on rank {rank}: {e!r}", file=sys.stderr, flush=True)
    if rank == 0:
        if e2e_peer is not None:
            e2e = e2e_peer
        elif not (slabs or args.no_e2e or args.method == "fim"):
            e2e = run_e2e(eik, torch, dev, w, calls, args, rdt)
        else:
            e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                   "note": "e2e is measured by the single-GPU run through solve_ifim"}
        cpu_n = args.cpu_size or CPU_SIZE[args.config]
        cpu_calls, cpu_s, cpu_threads = cpu_sample(cpu_n, os.cpu_count() or 1, args.config) if not args.no_cpu \
            else (0, 0.0, 0)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if slabs else "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": workload, "size": n, "method": args.method, "solver_calls_per_step": calls,
                       "iterations": r.iterations, "peak_remedy": r.peak_remedy, "remedy_engine": remedy_engine,
                       "parallelism": {"peer": f"z-slabs x{world} (peer-memory fused kernels)",
                                       "host": f"z-slabs x{world} (host-driven exchange)"}.get(mode, "single"),
                       "l2": (f"inputs larger than L2 (phi {w.cells * 8 / 2 ** 30:g} GiB fp64 per field)"
                              if w.cells * 8 > (126 << 20) else "inputs smaller than L2 (cfg1/cfg2-size 2D grid)"),
                       "phase_ms": r.phase_ms},
            "parity": parity, "parity_detail": parity_detail,
            "wall_clock_to_convergence_ms": ms / args.steps,
            "grid_cells_per_s": w.cells / (ms / args.steps * 1e-3),  # N / wall
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": rem_kernel, "alg_bytes_per_launch": alg_bytes,
                         "launch_ms": rem_s * 1e3,
                         "peak_source": peak_src},
            "phase_roofline": ({k: round(b / (r.phase_ms[k] * 1e-3) / 1e9 / hbm_peak()[0], 4)
                                for k, b in r.phase_bytes.items() if r.phase_ms.get(k)}
                               if getattr(r, "phase_bytes", None) else None),
            "cpu_baseline": {"value": (cpu_calls / cpu_s) if cpu_s else None, "unit": UNIT,
                             "cores": cpu_threads, "kind": "port",
                             "sample": f"full solve of {workload_desc(args.config, cpu_n)} (a bounded "
                                       f"{sample_label(args.config, cpu_n)} sample of the workload) with "
                                       f"oracle/eik_oracle.c, OpenMP x{cpu_threads}, {cpu_s:.1f} s",
                             "full_size": full_size_oracle(args.config, n)},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
    if world > 1 or args.force_peer:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)
        if out["parity"] == "mismatch":
            print(f"[bench] RESULT MISMATCH vs the oracle digests: {out['parity_detail']}", file=sys.stderr, flush=True)
            return 3
    return 0


def run_e2e(eik, torch, dev, w, calls, args, rdt):
    """Same metric through solve_ifim with host buffers: H2D of phi/speed/state from pinned
    memory and D2H of phi inside each timed step."""
    speed = w.F.to(rdt).cpu().pin_memory()
    phi = torch.empty(w.shape, dtype=rdt).pin_memory()
    state = torch.empty(w.shape, dtype=torch.uint8).pin_memory()
    bc = w.bc(eik)
    steps = max(1, min(args.steps, 3))
    warm = 2  # allocations: device grid, workspace, pinned result copies (cached by torch afterwards)
    tot = 0.0
    res = None
    for it in range(steps + warm):
        phi.fill_(float("inf"))
        state.zero_()
        g = w.grid(eik, phi, speed, state)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = eik.solve_ifim(g, bc)
        dt = time.perf_counter() - t0
        assert res.stats.solver_calls == calls
        if it >= warm:
            tot += dt
    N = w.cells
    # D2H: phi into the caller's array (the in-place API), in chunks; SolverResult.phi (the
    # reference returns grid.phi.copy()) takes some chunks by a second DMA and the others by host
    # copies of the landed chunks, overlapped with the remaining DMA (ifim._HostResult)
    from paper_2106_15869_b200.ifim import _HostResult

    rs = phi.element_size()
    dma2, hostcp = _HostResult.result_split(N * rs, rs)
    return {"value": calls * steps / tot, "unit": UNIT, "h2d_bytes_per_step": N * (rs + rs + 1),
            "d2h_bytes_per_step": N * rs + dma2, "steps": steps, "ms_per_step": tot / steps * 1e3,
            "host_copy_bytes_per_step": hostcp}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--size", type=int, default=None, help="grid edge (default 512; cfg5: 1024)")
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="BASELINE.json config (cfg4 = the headline 512^3 checkerboard)")
    ap.add_argument("--cpu-size", type=int, default=None,
                    help="edge of the bounded CPU sample (default per config: ~10-20 s of CPU work)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--method", default="ifim", choices=["ifim", "fim"],
                    help="ifim = the accelerated path (headline); fim = the paper's FIM baseline on the GPU")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                    help="f64 = parity mode (default, bit-exact); f32 = perf mode (max-rel 1e-5)")
    ap.add_argument("--slabs", action="store_true", help="use the z-slab protocol even on one GPU")
    ap.add_argument("--host-slabs", action="store_true", help="N>1: host-driven NCCL slabs instead of peer memory")
    ap.add_argument("--force-peer", action="store_true",
                    help="run the peer-memory slab kernels even at N=1 (under torchrun; a test of that path)")
    args = ap.parse_args()
    if args.size is None:
        args.size = {"cfg1": 256, "cfg2": 4096, "cfg3": 256, "cfg5": 1024}.get(args.config, 512)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
