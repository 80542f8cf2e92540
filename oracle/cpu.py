"""ctypes wrapper over oracle/eik_oracle.c (TEST INFRASTRUCTURE ONLY).

Functions take flat numpy arrays in the reference's conventions
(E/grid.py:1-8: phi float64 with +inf unreached, speed float64 >= 0, state
uint8 CellState codes, linear index j*nx+i, or (k*ny+j)*nx+i in 3D).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "eik_oracle.c")
LIB = os.path.join(HERE, "libeik_oracle.so")

ORC_OK, ORC_EINVAL, ORC_ECAP = 0, 1, 2


class Geom(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("ndim", C.c_int32), ("pad", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("solver_calls", C.c_int64),
                ("peak_active", C.c_int64), ("peak_remedy", C.c_int64),
                ("phi_writes", C.c_int64), ("history_len", C.c_int64),
                ("remedy_size", C.c_int64), ("converged", C.c_int64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile the oracle (no FMA contraction, OpenMP) into oracle/libeik_oracle.so."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-o", LIB + ".tmp", SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        i64 = C.c_int64
        dbl = C.c_double
        GP = C.POINTER(Geom)
        SP = C.POINTER(Stats)
        L.orc_update_2d_uniform.restype = dbl
        L.orc_update_2d_uniform.argtypes = [dbl, dbl, dbl, dbl]
        L.orc_update_2d_aniso.restype = dbl
        L.orc_update_2d_aniso.argtypes = [dbl, dbl, dbl, dbl, dbl]
        L.orc_update_3d_uniform.restype = dbl
        L.orc_update_3d_uniform.argtypes = [dbl, dbl, dbl, dbl, dbl]
        L.orc_update_2d_uniform_batch.argtypes = [P, P, P, P, P, i64]
        L.orc_update_2d_aniso_batch.argtypes = [P, P, P, P, P, P, i64]
        L.orc_update_3d_uniform_batch.argtypes = [P, P, P, P, P, P, i64]
        L.orc_ifim_update_step.argtypes = [GP, P, P, P, P, P, i64, dbl, P, i64, SP, C.c_int]
        L.orc_build_remedy.argtypes = [GP, P, P, P, dbl, P, SP, C.c_int]
        L.orc_remedy_step.argtypes = [GP, P, P, P, P, dbl, P, i64, SP, C.c_int]
        L.orc_solve_ifim.argtypes = [GP, P, P, P, P, P, i64, dbl, P, i64, SP, P, C.c_int]
        L.orc_solve_fim.argtypes = [GP, P, P, P, P, P, i64, dbl, SP]
        L.orc_solve_fixpoint.argtypes = [GP, P, P, P, P, P, i64, dbl, i64, SP, C.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def geom(shape, spacing) -> Geom:
    """shape = (ny, nx) or (nz, ny, nx); spacing = (dx, dy) or h."""
    if len(shape) == 2:
        ny, nx = shape
        dx, dy = spacing
        return Geom(nx, ny, 1, dx, dy, dx, 2, 0)
    nz, ny, nx = shape
    h = float(spacing)
    return Geom(nx, ny, nz, h, h, h, 3, 0)


def _check(rc, what):
    if rc == ORC_EINVAL:
        raise ValueError(f"oracle {what}: invalid argument")
    if rc == ORC_ECAP:
        raise RuntimeError(f"oracle {what}: iteration cap exceeded")
    if rc != ORC_OK:
        raise RuntimeError(f"oracle {what}: error {rc}")


@dataclass
class OracleResult:
    phi: np.ndarray
    state: np.ndarray
    stats: dict
    phases: dict = field(default_factory=dict)
    active_history: list = field(default_factory=list)


def solve_ifim(shape, spacing, speed, seed_idx, seed_val, state=None, phi=None, tol=1e-12,
               threads=1) -> OracleResult:
    """Restatement of E/ifim.py:221-235 (2D) and its 3D generalisation."""
    g = geom(shape, spacing)
    speed = np.ascontiguousarray(speed, dtype=np.float64).ravel()
    n = speed.size
    if state is None:
        state = np.where(speed == 0.0, 4, 0).astype(np.uint8)
    state = np.ascontiguousarray(state, dtype=np.uint8).ravel().copy()
    phi = np.full(n, np.inf) if phi is None else np.ascontiguousarray(phi, dtype=np.float64).ravel().copy()
    si = np.ascontiguousarray(seed_idx, dtype=np.int64)
    sv = np.ascontiguousarray(seed_val, dtype=np.float64)
    hcap = 40 * (g.nx + g.ny + (g.nz if g.ndim == 3 else 0)) + 1
    hist = np.zeros(hcap, dtype=np.int64)
    st = Stats()
    phases = (Stats * 3)()
    rc = lib().orc_solve_ifim(C.byref(g), _ptr(phi), _ptr(speed), _ptr(state), _ptr(si), _ptr(sv), si.size,
                              tol, _ptr(hist), hcap, C.byref(st), C.cast(phases, C.c_void_p), threads)
    _check(rc, "solve_ifim")
    return OracleResult(phi=phi.reshape(shape), state=state.reshape(shape), stats=st.as_dict(),
                        phases={"update": phases[0].as_dict(), "build": phases[1].as_dict(),
                                "remedy": phases[2].as_dict()},
                        active_history=hist[: st.history_len].tolist())


def solve_fim(shape, spacing, speed, seed_idx, seed_val, state=None, phi=None, tol=1e-12) -> OracleResult:
    """Restatement of E/fim.py:62-144 (2D) and its 3D generalisation (serial)."""
    g = geom(shape, spacing)
    speed = np.ascontiguousarray(speed, dtype=np.float64).ravel()
    n = speed.size
    if state is None:
        state = np.where(speed == 0.0, 4, 0).astype(np.uint8)
    state = np.ascontiguousarray(state, dtype=np.uint8).ravel().copy()
    phi = np.full(n, np.inf) if phi is None else np.ascontiguousarray(phi, dtype=np.float64).ravel().copy()
    si = np.ascontiguousarray(seed_idx, dtype=np.int64)
    sv = np.ascontiguousarray(seed_val, dtype=np.float64)
    st = Stats()
    rc = lib().orc_solve_fim(C.byref(g), _ptr(phi), _ptr(speed), _ptr(state), _ptr(si), _ptr(sv), si.size, tol,
                             C.byref(st))
    _check(rc, "solve_fim")
    return OracleResult(phi=phi.reshape(shape), state=state.reshape(shape), stats=st.as_dict(), phases={},
                        active_history=[])


def update_step(shape, spacing, phi, speed, state, seed_idx, seed_val, tol=1e-12, threads=1):
    """E/ifim.py:75-134; phi/state are modified in place (flat views)."""
    g = geom(shape, spacing)
    hcap = 40 * (g.nx + g.ny + (g.nz if g.ndim == 3 else 0)) + 1
    hist = np.zeros(hcap, dtype=np.int64)
    st = Stats()
    si = np.ascontiguousarray(seed_idx, dtype=np.int64)
    sv = np.ascontiguousarray(seed_val, dtype=np.float64)
    rc = lib().orc_ifim_update_step(C.byref(g), _ptr(phi), _ptr(speed), _ptr(state), _ptr(si), _ptr(sv),
                                    si.size, tol, _ptr(hist), hcap, C.byref(st), threads)
    _check(rc, "update_step")
    d = st.as_dict()
    d["active_history"] = hist[: st.history_len].tolist()
    return d


def build_remedy(shape, spacing, phi, speed, state, tol=1e-12, threads=1):
    """E/ifim.py:137-161; returns (member uint8, stats)."""
    g = geom(shape, spacing)
    member = np.zeros(phi.size, dtype=np.uint8)
    st = Stats()
    rc = lib().orc_build_remedy(C.byref(g), _ptr(phi), _ptr(speed), _ptr(state), tol, _ptr(member),
                                C.byref(st), threads)
    _check(rc, "build_remedy")
    return member, st.as_dict()


def remedy_step(shape, spacing, phi, speed, state, member, tol=1e-12, threads=1):
    """E/ifim.py:164-218; phi and member modified in place."""
    g = geom(shape, spacing)
    st = Stats()
    hcap = 20 * (g.nx + g.ny + (g.nz if g.ndim == 3 else 0)) + 1
    hist = np.zeros(hcap, dtype=np.int64)
    rc = lib().orc_remedy_step(C.byref(g), _ptr(phi), _ptr(speed), _ptr(state), _ptr(member), tol,
                               _ptr(hist), hcap, C.byref(st), threads)
    _check(rc, "remedy_step")
    d = st.as_dict()
    d["remedy_history"] = hist[: min(st.history_len, hcap)].tolist()
    return d


def solve_fixpoint(shape, spacing, speed, seed_idx, seed_val, tol=1e-12, max_passes=0, threads=1):
    """E/oracle.py:22-70 (and its 3D generalisation)."""
    g = geom(shape, spacing)
    speed = np.ascontiguousarray(speed, dtype=np.float64).ravel()
    state = np.where(speed == 0.0, 4, 0).astype(np.uint8)
    phi = np.full(speed.size, np.inf)
    si = np.ascontiguousarray(seed_idx, dtype=np.int64)
    sv = np.ascontiguousarray(seed_val, dtype=np.float64)
    st = Stats()
    rc = lib().orc_solve_fixpoint(C.byref(g), _ptr(phi), _ptr(speed), _ptr(state), _ptr(si), _ptr(sv),
                                  si.size, tol, max_passes, C.byref(st), threads)
    _check(rc, "solve_fixpoint")
    return phi.reshape(shape), st.as_dict()


def _arrs(n, *xs):
    return [np.ascontiguousarray(np.broadcast_to(np.asarray(x, dtype=np.float64), (n,))) for x in xs]


def local_2d_uniform(a, b, f, delta):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b, f, d = _arrs(a.size, b, f, delta)
    out = np.empty_like(a)
    lib().orc_update_2d_uniform_batch(_ptr(a), _ptr(b), _ptr(f), _ptr(d), _ptr(out), a.size)
    return out


def local_2d_aniso(a, b, f, dx, dy):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b, f, x, y = _arrs(a.size, b, f, dx, dy)
    out = np.empty_like(a)
    lib().orc_update_2d_aniso_batch(_ptr(a), _ptr(b), _ptr(f), _ptr(x), _ptr(y), _ptr(out), a.size)
    return out


def local_3d_uniform(a, b, c, f, delta):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b, c, f, d = _arrs(a.size, b, c, f, delta)
    out = np.empty_like(a)
    lib().orc_update_3d_uniform_batch(_ptr(a), _ptr(b), _ptr(c), _ptr(f), _ptr(d), _ptr(out), a.size)
    return out
