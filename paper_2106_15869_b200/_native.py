"""Build and load the sm_100a engine (libeik_ifim.so) through its C ABI.

The library is compiled in-tree by ``build()`` (nvcc, -gencode
arch=compute_100a,code=sm_100a, -fmad=false for bit-exact float64) and loaded
with ctypes.  There is no fallback: if the library or a GPU is missing every
solver call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "eik_ifim.cu")
HDR = os.path.join(ROOT, "include", "eik_ifim.h")
LIB = os.path.join(HERE, "libeik_ifim.so")

EIK_OK, EIK_EINVAL, EIK_ECAP, EIK_ECUDA, EIK_ENCCL = 0, 1, 2, 3, 4

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",          # no FMA contraction: separately rounded IEEE ops like numpy
    "-Xcompiler", "-fPIC", "-shared",
]

EXPORTS = (
    "eik_workspace_size", "eik_ifim_update_step", "eik_build_remedy", "eik_remedy_load",
    "eik_remedy_export", "eik_remedy_step", "eik_ifim_solve", "eik_local_solve",
    "eik_last_error", "eik_version", "eik_workspace_offsets", "eik_slab_update_init", "eik_slab_update_iter",
    "eik_slab_apply_requests", "eik_slab_build", "eik_slab_remedy_round", "eik_solve_fixpoint",
    "eik_max_residual", "eik_mr_prepare", "eik_mr_run", "eik_peer_enable",
)


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/eik_ifim.cu into paper_2106_15869_b200/libeik_ifim.so."""
    stale = (not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)))
    if force or stale:
        cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp", SRC]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class Geom(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("ndim", C.c_int32), ("dtype", C.c_int32), ("flags", C.c_int32), ("reserved", C.c_int32)]


EIK_GEOM_SLAB = 1


class Rank(C.Structure):
    _fields_ = [("phi0", C.c_void_p), ("workspace", C.c_void_p), ("nz", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("solver_calls", C.c_int64),
                ("peak_active", C.c_int64), ("peak_remedy", C.c_int64),
                ("phi_writes", C.c_int64), ("history_len", C.c_int64),
                ("remedy_size", C.c_int64), ("converged", C.c_int64),
                ("upd_iterations", C.c_int64), ("upd_calls", C.c_int64),
                ("build_calls", C.c_int64), ("rem_iterations", C.c_int64),
                ("rem_calls", C.c_int64), ("gpu_launches", C.c_int64),
                ("upd_ms", C.c_float), ("build_ms", C.c_float),
                ("rem_ms", C.c_float), ("total_ms", C.c_float)]

    def as_dict(self) -> dict:
        return {k: (float(getattr(self, k)) if t is C.c_float else int(getattr(self, k)))
                for k, t in self._fields_}


_lib = None


def lib():
    """The loaded engine; raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise RuntimeError(
            f"B200 engine not built: {LIB} is missing (run `python -c 'import __graft_entry__ as g; g.build()'`)")
    L = C.CDLL(LIB)
    P, i64, dbl, vp = C.c_void_p, C.c_int64, C.c_double, C.c_void_p
    GP, SP = C.POINTER(Geom), C.POINTER(Stats)
    L.eik_workspace_size.argtypes = [GP, C.POINTER(C.c_size_t)]
    L.eik_ifim_update_step.argtypes = [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, P, i64, SP, vp]
    L.eik_build_remedy.argtypes = [GP, P, P, P, dbl, P, C.c_size_t, SP, vp]
    L.eik_remedy_load.argtypes = [GP, P, P, P, C.c_size_t, C.POINTER(i64), vp]
    L.eik_remedy_export.argtypes = [GP, P, C.c_size_t, P, vp]
    L.eik_remedy_step.argtypes = [GP, P, P, P, dbl, P, C.c_size_t, SP, vp]
    L.eik_ifim_solve.argtypes = [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, P, i64, SP, vp]
    L.eik_local_solve.argtypes = [C.c_int, P, P, P, P, dbl, dbl, P, i64, vp]
    L.eik_workspace_offsets.argtypes = [GP, P]
    L.eik_slab_update_init.argtypes = [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, C.POINTER(i64), vp]
    L.eik_slab_update_iter.argtypes = [GP, P, P, P, dbl, i64, P, C.c_size_t, vp]
    L.eik_slab_apply_requests.argtypes = [GP, P, P, i64, P, C.c_size_t, C.POINTER(i64), vp]
    L.eik_slab_build.argtypes = [GP, P, P, P, dbl, P, C.c_size_t, C.POINTER(i64), C.POINTER(i64), vp]
    L.eik_slab_remedy_round.argtypes = [GP, P, P, P, dbl, i64, P, C.c_size_t, C.POINTER(i64), C.POINTER(i64), vp]
    L.eik_solve_fixpoint.argtypes = [GP, P, P, P, P, P, i64, dbl, i64, P, C.c_size_t, SP, vp]
    L.eik_max_residual.argtypes = [GP, P, P, P, P, C.c_size_t, C.POINTER(dbl), vp]
    RP = C.POINTER(Rank)
    L.eik_mr_prepare.argtypes = [GP, C.c_int32, RP, C.c_int32, C.c_int32, P, P, P, P, i64, dbl, vp]
    L.eik_mr_run.argtypes = [GP, C.c_int32, RP, C.c_int32, C.c_int32, P, P, dbl, P, i64, SP, vp]
    L.eik_peer_enable.argtypes = [C.c_int32, C.c_int32]
    L.eik_last_error.restype = C.c_char_p
    L.eik_version.restype = C.c_char_p
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == EIK_OK:
        return
    msg = lib().eik_last_error().decode(errors="replace")
    if rc == EIK_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)
