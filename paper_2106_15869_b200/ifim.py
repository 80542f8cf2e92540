"""Drop-in iFIM entry points backed by the B200 engine.

Same names, signatures, argument meaning, return types and error behaviour as
the reference's E/ifim.py (E = /root/reference/pkg/src/eikonal):

    solve_ifim(grid, bc, tol=1e-12, workers=1) -> SolverResult     E/ifim.py:221-235
    ifim_update_step(grid, bc, tol=1e-12, workers=1) -> RunStats   E/ifim.py:75-134
    build_remedy_set(grid, tol=1e-12, workers=1) -> (RemedySet, int)  E/ifim.py:137-161
    ifim_remedy_step(grid, remedy, tol=1e-12, workers=1) -> RunStats  E/ifim.py:164-218
    RemedySet                                                      E/ifim.py:64-72

The solvers mutate ``grid.phi`` in place, mark seeds SOURCE in ``grid.state``
and start from whatever phi they are given.  ``workers`` is validated like
E/parallel.py:28-42 and otherwise ignored: the work runs on the GPU through
the C ABI in include/eik_ifim.h.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np
import torch

from . import _native
from .grid import CellState, seed_linear
from .result import RunStats, SolverResult


def resolve_workers(workers: int | None = None) -> int:
    """E/parallel.py:28-42 (validation only; the device engine ignores the count)."""
    if workers is None:
        env = os.environ.get("EIKONAL_WORKERS", "").strip()
        workers = int(env) if env else 1
    workers = int(workers)
    if workers == 0:
        return os.cpu_count() or 1
    if workers < 0:
        raise ValueError(f"worker count must be >= 0, got {workers}")
    return workers


def _check_tol(tol: float) -> None:
    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")


# ---------------------------------------------------------------------------
# device views of a grid
# ---------------------------------------------------------------------------

def _is_cuda_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def _pick_device(grid) -> torch.device:
    if _is_cuda_tensor(grid.phi):
        return grid.phi.device
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2106_15869_b200 needs a CUDA device (B200); no CPU fallback exists")
    dev = os.environ.get("EIKONAL_DEVICE", "cuda:0")
    return torch.device(dev)


def field_dtype(grid) -> int:
    """float32 phi selects the float32 perf-mode engine; anything else runs in float64."""
    d = getattr(grid.phi, "dtype", None)
    return _native.EIK_F32 if d in (torch.float32, np.float32) else _native.EIK_F64


def geometry(grid) -> _native.Geom:
    dt = field_dtype(grid)
    if getattr(grid, "ndim", 2) == 3:
        h = float(grid.h)
        return _native.Geom(int(grid.nx), int(grid.ny), int(grid.nz), h, h, h, 3, dt, 0, 0)
    return _native.Geom(int(grid.nx), int(grid.ny), 1, float(grid.dx), float(grid.dy), float(grid.dx), 2, dt, 0, 0)


class _DeviceGrid:
    """phi / speed / state of a grid as contiguous CUDA tensors.

    CUDA-tensor grids are used in place.  Host grids (numpy arrays or CPU
    tensors) are uploaded and ``commit`` writes phi (and state) back into the
    caller's arrays, which is what the in-place reference API promises.
    """

    def __init__(self, grid, need_phi=True, need_state=True):
        self.grid = grid
        self.device = _pick_device(grid)
        self.host = not _is_cuda_tensor(grid.phi)
        self.dtype = torch.float32 if field_dtype(grid) == _native.EIK_F32 else torch.float64
        self.phi = self._dev(grid.phi, self.dtype) if need_phi else None
        self.speed = self._dev(grid.speed, self.dtype)
        self.state = self._dev(grid.state, torch.uint8) if need_state else None

    def _dev(self, arr, dtype):
        if _is_cuda_tensor(arr):
            if arr.dtype != dtype or not arr.is_contiguous():
                raise ValueError(f"CUDA grid arrays must be contiguous {dtype}, got {arr.dtype}")
            if arr.device != self.device:
                raise ValueError("grid arrays live on different devices")
            return arr
        t = torch.as_tensor(np.ascontiguousarray(arr)) if isinstance(arr, np.ndarray) else arr
        pinned = isinstance(t, torch.Tensor) and t.is_pinned()
        return t.to(device=self.device, dtype=dtype, non_blocking=pinned).contiguous()

    @property
    def stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def commit(self, phi=True, state=False):
        if not self.host:
            return
        torch.cuda.synchronize(self.device)
        if phi:
            _copy_into(self.grid.phi, self.phi)
        if state:
            _copy_into(self.grid.state, self.state)


def _copy_into(host_arr, dev_t):
    if isinstance(host_arr, np.ndarray):
        torch.from_numpy(host_arr).copy_(dev_t.reshape(host_arr.shape))
    else:
        host_arr.copy_(dev_t.reshape(host_arr.shape), non_blocking=host_arr.is_pinned())
        if host_arr.is_pinned():
            torch.cuda.current_stream(dev_t.device).synchronize()


class _HostResult:
    """SolverResult.phi for host grids (the reference returns grid.phi.copy()).

    Large fields: the copy is allocated on a helper thread while the device
    solves (the engine call releases the GIL).  A pinned caller array gets a
    pinned copy (torch's caching host allocator reuses freed ones); the field is
    downloaded in chunks, and the result takes a quarter of the chunks by a second
    DMA and the rest by host copies of the landed chunks, overlapped with the
    remaining DMA.  A
    pageable caller array gets a first-touched pageable copy; the field is
    downloaded once into the caller's array and the copy is a host memcpy of it.
    """

    MIN_CELLS = 1 << 22
    CHUNK_BYTES = 1 << 27  # D2H chunk of the pinned path
    RESULT_DMA_FRAC = 0.25  # share of the result chunks taken by a second DMA instead of a host copy
    # (measured on the B200 hosts: a quarter balances the DMA engine against the host copy threads)

    @classmethod
    def result_split(cls, nbytes: int, elem: int) -> tuple[int, int]:
        """(second-DMA bytes, host-copy bytes) of a pinned result of ``nbytes`` (what commit does)."""
        frac = float(os.environ.get("EIK_RESULT_DMA_FRAC", cls.RESULT_DMA_FRAC))
        step = max(1, cls.CHUNK_BYTES // elem) * elem
        dma = host = 0
        for j, a in enumerate(range(0, nbytes, step)):
            b = min(nbytes, a + step)
            if int((j + 1) * frac) > int(j * frac):
                dma += b - a
            else:
                host += b - a
        return dma, host

    def __init__(self, dg):
        self.dg, self.buf, self.thread = dg, None, None
        phi = dg.grid.phi
        self.pinned = isinstance(phi, torch.Tensor) and phi.is_pinned()
        if dg.host and dg.phi.numel() >= self.MIN_CELLS:
            import threading

            def alloc():
                if self.pinned:
                    self.buf = torch.empty(tuple(phi.shape), dtype=dg.dtype, pin_memory=True)
                else:
                    b = torch.empty(tuple(phi.shape), dtype=dg.dtype)
                    b.zero_()  # first touch off the critical path
                    self.buf = b

            self.thread = threading.Thread(target=alloc, daemon=True)
            self.thread.start()

    def commit(self):
        """Device phi -> the caller's array and -> the result copy; returns the copy."""
        dg, gphi = self.dg, self.dg.grid.phi
        if self.thread is None:
            dg.commit(phi=True)
            return gphi.copy() if isinstance(gphi, np.ndarray) else gphi.clone()
        self.thread.join()
        buf = self.buf
        host = torch.from_numpy(gphi) if isinstance(gphi, np.ndarray) else gphi
        dev = dg.phi.reshape(host.shape)
        if self.pinned and not host.is_contiguous():
            host.copy_(dev, non_blocking=True)
            buf.copy_(dev, non_blocking=True)
            torch.cuda.current_stream(dg.device).synchronize()
        elif self.pinned:
            # one DMA into the caller's array, chunk by chunk; the result gets RESULT_DMA_FRAC of the
            # chunks by a second DMA and the others by host copies (torch's threaded copy) of the
            # landed chunks while the next chunks are in flight
            st = torch.cuda.current_stream(dg.device)
            hf, df, bf = host.reshape(-1), dev.reshape(-1), buf.reshape(-1)
            n = hf.numel()
            step = max(1, self.CHUNK_BYTES // hf.element_size())
            frac = float(os.environ.get("EIK_RESULT_DMA_FRAC", self.RESULT_DMA_FRAC))
            landed = []
            for j, a in enumerate(range(0, n, step)):
                b = min(n, a + step)
                hf[a:b].copy_(df[a:b], non_blocking=True)
                if int((j + 1) * frac) > int(j * frac):  # this chunk of the result: a second DMA
                    bf[a:b].copy_(df[a:b], non_blocking=True)
                    continue
                ev = torch.cuda.Event()
                ev.record(st)
                landed.append((a, b, ev))
            for a, b, ev in landed:
                ev.synchronize()
                bf[a:b].copy_(hf[a:b])
            st.synchronize()
        else:
            dg.commit(phi=True)
            buf.copy_(host)
        return buf.numpy() if isinstance(gphi, np.ndarray) else buf


def _host_mark_sources(grid, idx):
    """apply_boundary's state write (E/grid.py:215) on a host grid."""
    st = grid.state
    flat = st.reshape(-1)
    for c in idx:
        flat[c] = CellState.SOURCE


# ---------------------------------------------------------------------------
# workspace cache (the caller owns all device memory; the library allocates none)
# ---------------------------------------------------------------------------

class Workspace:
    def __init__(self, geom: _native.Geom, device: torch.device):
        n = C.c_size_t(0)
        _native.check(_native.lib(geom.dtype).eik_workspace_size(C.byref(geom), C.byref(n)), geom.dtype)
        self.nbytes = int(n.value)
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.gen = 0  # bumped by every call that rewrites the remedy set slots

    @property
    def ptr(self):
        return C.c_void_p(self.buf.data_ptr())


_WS: "dict" = {}  # (thread id, device, geometry) -> Workspace, least recently used first
_WS_LOCK = __import__("threading").RLock()
_TLS = __import__("threading").local()


class _ThreadReaper:
    """Lives in a thread's local storage: when the thread ends, its workspaces are released."""

    def __init__(self, ident):
        self.ident = ident

    def __del__(self):
        try:
            with _WS_LOCK:
                for k in [k for k in _WS if k[0] == self.ident]:
                    del _WS[k]
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass


def _ws_budget(device) -> int:
    """Bytes all cached workspaces of one device may hold (EIKONAL_WS_BUDGET, default half the
    device memory)."""
    env = os.environ.get("EIKONAL_WS_BUDGET", "").strip()
    if env:
        return int(float(env))
    return torch.cuda.get_device_properties(device).total_memory // 2


def workspace(geom: _native.Geom, device: torch.device) -> Workspace:
    """The calling thread's workspace for this geometry (kept between calls: the staged API
    leaves the remedy set in it).  Per thread, so concurrent solves on different grids of the
    same shape never share scratch memory (the reference's solvers are re-entrant).  A thread's
    workspaces are released when the thread ends, and the cache of a device is bounded by a byte
    budget (least recently used entries go first).  Evicting an entry only drops the cache's
    reference: a call (or a RemedySet) still holding the workspace keeps its memory alive."""
    import threading

    ident = threading.get_ident()
    if getattr(_TLS, "reaper", None) is None:
        _TLS.reaper = _ThreadReaper(ident)
    key = (ident, str(device), geom.nx, geom.ny, geom.nz, geom.ndim, geom.dtype)
    with _WS_LOCK:
        ws = _WS.pop(key, None)
        if ws is None:
            n = C.c_size_t(0)
            _native.check(_native.lib(geom.dtype).eik_workspace_size(C.byref(geom), C.byref(n)), geom.dtype)
            budget, need = _ws_budget(device), int(n.value)
            used = sum(w.nbytes for k, w in _WS.items() if k[1] == key[1])
            for k in [k for k in _WS if k[1] == key[1]]:  # least recently used first, before allocating
                if used + need <= budget:
                    break
                used -= _WS.pop(k).nbytes
            ws = Workspace(geom, device)
        _WS[key] = ws  # most recently used last
    return ws


def clear_workspaces() -> None:
    with _WS_LOCK:
        _WS.clear()


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _history_cap(g: _native.Geom) -> int:
    return 40 * (g.nx + g.ny + (g.nz if g.ndim == 3 else 0)) + 2


# ---------------------------------------------------------------------------
# RemedySet
# ---------------------------------------------------------------------------

class RemedySet:
    """Cells flagged for repair (E/ifim.py:64-72): ``member`` mask + ``cells`` work list.

    Sets produced by build_remedy_set live on the device; ``member`` and
    ``cells`` are materialised on first access (``cells`` = the members in
    ascending order, as E/ifim.py:158-161 builds it).  A RemedySet built by
    hand follows the reference's dataclass: ``cells`` defaults to an empty
    list, and the remedy step relaxes ``cells`` (E/ifim.py:184-193) while
    ``member`` only decides which neighbours get enqueued (E/ifim.py:211), so
    ``RemedySet(member=m)`` alone is an empty set and members outside ``cells``
    are never relaxed or enqueued.  The device engine works on sets, so
    ``cells`` must not repeat a cell and must be marked in ``member``
    (ValueError otherwise; the reference would process such a list with
    duplicates).
    """

    def __init__(self, member=None, cells=None, *, _device=None):
        self._member = member
        self._dev = _device  # dict(mask, count, ws, gen, host, shape)
        if cells is not None:
            self._cells = [int(c) for c in cells]
        else:
            self._cells = None if _device is not None else []

    def __len__(self) -> int:
        if self._dev is not None:
            return int(self._dev["count"])
        return len(self._cells)

    @property
    def member(self):
        if self._member is None and self._dev is not None:
            mask = self._dev["mask"].bool()  # flat (N,), like E/ifim.py:158
            self._member = mask.cpu().numpy() if self._dev["host"] else mask
        return self._member

    @member.setter
    def member(self, value):
        self.cells  # keep the work list of a device-backed set
        self._member = value
        self._dev = None

    @property
    def cells(self) -> list:
        if self._cells is None:
            m = self.member
            if isinstance(m, torch.Tensor):
                self._cells = torch.nonzero(m.reshape(-1)).reshape(-1).cpu().tolist()
            else:
                self._cells = np.flatnonzero(np.asarray(m).reshape(-1)).tolist()
        return self._cells

    @cells.setter
    def cells(self, value):
        self.member  # keep the membership mask of a device-backed set
        self._cells = [int(c) for c in value]
        self._dev = None

    def _drain(self):
        """After ifim_remedy_step the work list is empty and its members are cleared
        (E/ifim.py:186, :208); members outside the work list keep their mark."""
        if self._dev is not None:
            self._dev["count"] = 0
            self._dev["mask"].zero_()
        elif self._member is not None and self._cells:
            idx = self._cells
            if isinstance(self._member, torch.Tensor):
                flat = self._member.reshape(-1)
                flat[torch.as_tensor(idx, dtype=torch.int64, device=flat.device)] = False
            else:
                np.asarray(self._member).reshape(-1)[idx] = False
        self._cells = []

    def _device_masks(self, shape, device):
        """(work-list mask, member mask or None) as flat uint8 CUDA tensors."""
        if self._dev is not None:
            return self._dev["mask"], None
        n = int(np.prod(shape))
        cells = self._cells
        work = torch.zeros(n, dtype=torch.uint8, device=device)
        if cells:
            idx = torch.as_tensor(cells, dtype=torch.int64, device=device)
            if int(idx.min()) < 0 or int(idx.max()) >= n:
                raise ValueError(f"RemedySet.cells holds a cell outside the {n}-cell grid")
            work[idx] = 1
            if int(work.sum()) != len(cells):
                raise ValueError("RemedySet.cells repeats a cell (the device engine relaxes sets)")
        if self._member is None:
            return work, None
        m = self._member
        t = m if isinstance(m, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(m))
        mem = t.reshape(-1).to(device=device, dtype=torch.uint8).contiguous()
        if mem.numel() != n:
            raise ValueError(f"RemedySet.member has {mem.numel()} cells, the grid {n}")
        if cells and bool(((work != 0) & (mem == 0)).any()):
            raise ValueError("RemedySet.cells holds cells that RemedySet.member does not mark")
        return work, mem


# ---------------------------------------------------------------------------
# entry points
# ---------------------------------------------------------------------------

def _stats_from(s: _native.Stats) -> dict:
    return s.as_dict()


def ifim_update_step(grid, bc, tol: float = 1e-12, workers: int = 1) -> RunStats:
    """Drain the active list without neighbour convergence checks (E/ifim.py:75-134)."""
    _check_tol(tol)
    resolve_workers(workers)
    idx, val = seed_linear(grid, bc)
    dg = _DeviceGrid(grid)
    geom = geometry(grid)
    ws = workspace(geom, dg.device)
    ws.gen += 1
    si = torch.as_tensor(idx, dtype=torch.int64, device=dg.device)
    sv = torch.as_tensor(val, dtype=torch.float64, device=dg.device)
    hcap = _history_cap(geom)
    hist = np.zeros(hcap, dtype=np.int64)
    st = _native.Stats()
    rc = _native.lib(geom.dtype).eik_ifim_update_step(
        C.byref(geom), _ptr(dg.phi), _ptr(dg.speed), _ptr(dg.state), _ptr(si), _ptr(sv), len(idx), float(tol),
        ws.ptr, ws.nbytes, hist.ctypes.data_as(C.c_void_p), hcap, C.byref(st), dg.stream)
    if dg.host:
        _host_mark_sources(grid, idx)
        dg.commit(phi=True)
    _native.check(rc, geom.dtype)
    d = _stats_from(st)
    stats = RunStats(active_history=hist[: d["upd_iterations"]].tolist())
    stats.iterations = d["upd_iterations"]
    stats.solver_calls = d["upd_calls"]
    stats.peak_active = d["peak_active"]
    stats.phi_writes = d["phi_writes"]
    stats.phases = {"update": d}
    stats.device_ms = {"update": d["upd_ms"]}
    stats.gpu_launches = d["gpu_launches"]
    return stats


def build_remedy_set(grid, tol: float = 1e-12, workers: int = 1):
    """One full verification pass; returns (RemedySet, solver calls) (E/ifim.py:137-161)."""
    _check_tol(tol)
    resolve_workers(workers)
    dg = _DeviceGrid(grid)
    geom = geometry(grid)
    ws = workspace(geom, dg.device)
    ws.gen += 1
    st = _native.Stats()
    _native.check(_native.lib(geom.dtype).eik_build_remedy(
        C.byref(geom), _ptr(dg.phi), _ptr(dg.speed), _ptr(dg.state), float(tol), ws.ptr, ws.nbytes,
        C.byref(st), dg.stream))
    n = int(np.prod(tuple(int(s) for s in grid.phi.shape)))
    mask = torch.empty(n, dtype=torch.uint8, device=dg.device)
    _native.check(_native.lib(geom.dtype).eik_remedy_export(C.byref(geom), ws.ptr, ws.nbytes, _ptr(mask), dg.stream))
    remedy = RemedySet(_device={"mask": mask, "count": int(st.remedy_size), "ws": ws, "gen": ws.gen,
                                "host": dg.host, "shape": tuple(grid.phi.shape)})
    return remedy, int(st.build_calls)


def ifim_remedy_step(grid, remedy: RemedySet, tol: float = 1e-12, workers: int = 1) -> RunStats:
    """Relax the remedy set to quiescence, accepting only decreases (E/ifim.py:164-218)."""
    _check_tol(tol)
    resolve_workers(workers)
    dg = _DeviceGrid(grid)
    geom = geometry(grid)
    ws = workspace(geom, dg.device)
    fresh = (remedy._dev is not None and remedy._dev.get("ws") is ws and remedy._dev.get("gen") == ws.gen)
    if not fresh:
        work, member = remedy._device_masks(tuple(grid.phi.shape), dg.device)
        cnt = C.c_int64(0)
        _native.check(_native.lib(geom.dtype).eik_remedy_load_set(C.byref(geom), _ptr(work), _ptr(member),
                                                                  _ptr(dg.state), ws.ptr, ws.nbytes, C.byref(cnt),
                                                                  dg.stream))
    ws.gen += 1
    st = _native.Stats()
    rc = _native.lib(geom.dtype).eik_remedy_step(C.byref(geom), _ptr(dg.phi), _ptr(dg.speed), _ptr(dg.state), float(tol),
                                       ws.ptr, ws.nbytes, C.byref(st), dg.stream)
    dg.commit(phi=True)
    _native.check(rc, geom.dtype)
    remedy._drain()
    d = _stats_from(st)
    stats = RunStats()
    stats.iterations = d["rem_iterations"]
    stats.solver_calls = d["rem_calls"]
    stats.peak_remedy = d["peak_remedy"]
    stats.phi_writes = d["phi_writes"]
    stats.phases = {"remedy": d}
    stats.device_ms = {"remedy": d["rem_ms"]}
    stats.gpu_launches = d["gpu_launches"]
    return stats


def solve_ifim(grid, bc, tol: float = 1e-12, workers: int = 1, devices=None) -> SolverResult:
    """Update step + build + remedy, device-resident (E/ifim.py:221-235).

    ``devices`` (or EIKONAL_DEVICES): a GPU count or a list of CUDA indices; more than one
    shards a Grid3D into z-slabs solved by the peer-memory kernels (slab_peer.solve_multi),
    with results and statistics identical to the single-device solve.
    """
    t0 = time.perf_counter()
    _check_tol(tol)
    resolve_workers(workers)
    from .slab_peer import resolve_devices, solve_multi

    devs = resolve_devices(devices)
    idx, val = seed_linear(grid, bc)
    if devs is not None:
        if field_dtype(grid) == _native.EIK_F32:
            raise ValueError("the multi-device solve runs the float64 engine; pass float64 phi/speed")
        stats, phi = solve_multi(grid, idx, val, tol, devs)
        stats.wall_time = time.perf_counter() - t0
        return SolverResult(phi=phi, stats=stats)
    dg = _DeviceGrid(grid)
    geom = geometry(grid)
    ws = workspace(geom, dg.device)
    ws.gen += 1
    si = torch.as_tensor(idx, dtype=torch.int64, device=dg.device)
    sv = torch.as_tensor(val, dtype=torch.float64, device=dg.device)
    hcap = _history_cap(geom)
    hist = np.zeros(hcap, dtype=np.int64)
    st = _native.Stats()
    out = _HostResult(dg)
    rc = _native.lib(geom.dtype).eik_ifim_solve(
        C.byref(geom), _ptr(dg.phi), _ptr(dg.speed), _ptr(dg.state), _ptr(si), _ptr(sv), len(idx), float(tol),
        ws.ptr, ws.nbytes, hist.ctypes.data_as(C.c_void_p), hcap, C.byref(st), dg.stream)
    phi = None
    if dg.host:
        _host_mark_sources(grid, idx)
        phi = out.commit()
    _native.check(rc, geom.dtype)
    d = _stats_from(st)
    stats = RunStats(
        iterations=d["iterations"],
        solver_calls=d["solver_calls"],
        peak_active=d["peak_active"],
        peak_remedy=d["peak_remedy"],
        active_history=hist[: d["upd_iterations"]].tolist(),
    )
    stats.phi_writes = d["phi_writes"]
    stats.phases = {
        "update": {"iterations": d["upd_iterations"], "solver_calls": d["upd_calls"], "converged": d["converged"]},
        "build": {"solver_calls": d["build_calls"], "remedy_size": d["remedy_size"]},
        "remedy": {"iterations": d["rem_iterations"], "solver_calls": d["rem_calls"]},
    }
    stats.device_ms = {"update": d["upd_ms"], "build": d["build_ms"], "remedy": d["rem_ms"], "total": d["total_ms"]}
    stats.gpu_launches = d["gpu_launches"]
    if phi is None:
        phi = grid.phi.copy() if isinstance(grid.phi, np.ndarray) else grid.phi.clone()
    stats.wall_time = time.perf_counter() - t0
    return SolverResult(phi=phi, stats=stats)
