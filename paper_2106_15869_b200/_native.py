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
DEPS = [os.path.join(HERE, "csrc", f) for f in ("eik_remedy_tma.cuh",)]
HDR = os.path.join(ROOT, "include", "eik_ifim.h")
LIB = os.path.join(HERE, "libeik_ifim.so")
LIB32 = os.path.join(HERE, "libeik_ifim_f32.so")  # float32 perf mode (-DEIK_SINGLE=1, names suffixed _f32)
EIK_F64, EIK_F32 = 0, 1

EIK_OK, EIK_EINVAL, EIK_ECAP, EIK_ECUDA, EIK_ENCCL = 0, 1, 2, 3, 4

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",          # no FMA contraction: separately rounded IEEE ops like numpy
    "-Xcompiler", "-fPIC", "-shared",
]

EXPORTS = (
    "eik_workspace_size", "eik_ifim_update_step", "eik_build_remedy", "eik_remedy_load", "eik_remedy_load_set",
    "eik_field_max_diff", "eik_chunk_sha256",
    "eik_remedy_export", "eik_remedy_step", "eik_ifim_solve", "eik_local_solve",
    "eik_last_error", "eik_version", "eik_last_remedy_engine", "eik_workspace_offsets", "eik_slab_update_init", "eik_slab_update_iter",
    "eik_slab_apply_requests", "eik_slab_build", "eik_slab_remedy_round", "eik_solve_fixpoint",
    "eik_max_residual", "eik_mr_prepare", "eik_mr_run", "eik_peer_enable", "eik_solve_fim",
)


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/eik_ifim.cu into paper_2106_15869_b200/libeik_ifim.so (float64) and
    libeik_ifim_f32.so (float32 perf mode)."""
    src_t = max(os.path.getmtime(f) for f in (SRC, HDR, *DEPS))
    for out, extra in ((LIB, []), (LIB32, ["-DEIK_SINGLE=1"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < src_t:
            cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp", SRC]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            subprocess.check_call(cmd)
            os.replace(out + ".tmp", out)
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


EXPORTS_F32 = (
    "eik_workspace_size_f32", "eik_ifim_update_step_f32", "eik_build_remedy_f32", "eik_remedy_load_f32",
    "eik_remedy_load_set_f32", "eik_field_max_diff_f32", "eik_chunk_sha256_f32",
    "eik_remedy_export_f32", "eik_remedy_step_f32", "eik_ifim_solve_f32", "eik_solve_fixpoint_f32",
    "eik_max_residual_f32", "eik_local_solve_f32", "eik_last_error_f32", "eik_version_f32", "eik_solve_fim_f32",
    "eik_last_remedy_engine_f32",
)

_lib = None
_lib32 = None
_last_dtype = EIK_F64


def _bind(L, name, argtypes):
    """Set a symbol's argtypes; a symbol missing from an older build stays unbound (calling it
    raises AttributeError) instead of breaking the whole library load."""
    try:
        getattr(L, name).argtypes = argtypes
    except AttributeError:
        pass


class _Suffixed:
    """The float32 library seen under the float64 entry-point names."""

    def __init__(self, cdll):
        self._l = cdll

    def __getattr__(self, name):
        return getattr(self._l, name + "_f32")


def lib(dtype: int = EIK_F64):
    """The loaded engine (float64, or the float32 perf-mode library for dtype EIK_F32);
    raises if it was not built (no CPU fallback)."""
    global _lib, _last_dtype
    _last_dtype = dtype  # check() reads the error text of the library used last
    if dtype == EIK_F32:
        return _lib_f32()
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise RuntimeError(
            f"B200 engine not built: {LIB} is missing (run `python -c 'import __graft_entry__ as g; g.build()'`)")
    L = C.CDLL(LIB)
    P, i64, dbl, vp = C.c_void_p, C.c_int64, C.c_double, C.c_void_p
    GP, SP = C.POINTER(Geom), C.POINTER(Stats)
    _bind(L, "eik_workspace_size", [GP, C.POINTER(C.c_size_t)])
    _bind(L, "eik_ifim_update_step", [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, P, i64, SP, vp])
    _bind(L, "eik_build_remedy", [GP, P, P, P, dbl, P, C.c_size_t, SP, vp])
    _bind(L, "eik_remedy_load", [GP, P, P, P, C.c_size_t, C.POINTER(i64), vp])
    _bind(L, "eik_remedy_load_set", [GP, P, P, P, P, C.c_size_t, C.POINTER(i64), vp])
    _bind(L, "eik_field_max_diff", [P, P, i64, P, C.POINTER(dbl), vp])
    _bind(L, "eik_chunk_sha256", [P, i64, i64, P, vp])
    _bind(L, "eik_remedy_export", [GP, P, C.c_size_t, P, vp])
    _bind(L, "eik_remedy_step", [GP, P, P, P, dbl, P, C.c_size_t, SP, vp])
    _bind(L, "eik_ifim_solve", [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, P, i64, SP, vp])
    _bind(L, "eik_local_solve", [C.c_int, P, P, P, P, dbl, dbl, P, i64, vp])
    _bind(L, "eik_workspace_offsets", [GP, P])
    _bind(L, "eik_slab_update_init", [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, C.POINTER(i64), vp])
    _bind(L, "eik_slab_update_iter", [GP, P, P, P, dbl, i64, P, C.c_size_t, vp])
    _bind(L, "eik_slab_apply_requests", [GP, P, P, i64, P, C.c_size_t, C.POINTER(i64), vp])
    _bind(L, "eik_slab_build", [GP, P, P, P, dbl, P, C.c_size_t, C.POINTER(i64), C.POINTER(i64), vp])
    _bind(L, "eik_slab_remedy_round", [GP, P, P, P, dbl, i64, P, C.c_size_t, C.POINTER(i64), C.POINTER(i64), vp])
    _bind(L, "eik_solve_fixpoint", [GP, P, P, P, P, P, i64, dbl, i64, P, C.c_size_t, SP, vp])
    _bind(L, "eik_max_residual", [GP, P, P, P, P, C.c_size_t, C.POINTER(dbl), vp])
    _bind(L, "eik_solve_fim", [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, SP, vp])
    RP = C.POINTER(Rank)
    _bind(L, "eik_mr_prepare", [GP, C.c_int32, RP, C.c_int32, C.c_int32, P, P, P, P, i64, dbl, vp])
    _bind(L, "eik_mr_run", [GP, C.c_int32, RP, C.c_int32, C.c_int32, P, P, dbl, P, i64, SP, vp])
    _bind(L, "eik_peer_enable", [C.c_int32, C.c_int32])
    L.eik_last_error.restype = C.c_char_p
    L.eik_version.restype = C.c_char_p
    _lib = L
    return L


def _lib_f32():
    global _lib32
    if _lib32 is not None:
        return _lib32
    if not os.path.exists(LIB32):
        raise RuntimeError(f"B200 float32 engine not built: {LIB32} is missing (run __graft_entry__.build())")
    L = C.CDLL(LIB32)
    P, i64, dbl, vp = C.c_void_p, C.c_int64, C.c_double, C.c_void_p
    GP, SP = C.POINTER(Geom), C.POINTER(Stats)
    _bind(L, "eik_workspace_size_f32", [GP, C.POINTER(C.c_size_t)])
    _bind(L, "eik_ifim_update_step_f32", [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, P, i64, SP, vp])
    _bind(L, "eik_build_remedy_f32", [GP, P, P, P, dbl, P, C.c_size_t, SP, vp])
    _bind(L, "eik_remedy_load_f32", [GP, P, P, P, C.c_size_t, C.POINTER(i64), vp])
    _bind(L, "eik_remedy_load_set_f32", [GP, P, P, P, P, C.c_size_t, C.POINTER(i64), vp])
    _bind(L, "eik_field_max_diff_f32", [P, P, i64, P, C.POINTER(dbl), vp])
    _bind(L, "eik_chunk_sha256_f32", [P, i64, i64, P, vp])
    _bind(L, "eik_remedy_export_f32", [GP, P, C.c_size_t, P, vp])
    _bind(L, "eik_remedy_step_f32", [GP, P, P, P, dbl, P, C.c_size_t, SP, vp])
    _bind(L, "eik_ifim_solve_f32", [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, P, i64, SP, vp])
    _bind(L, "eik_solve_fixpoint_f32", [GP, P, P, P, P, P, i64, dbl, i64, P, C.c_size_t, SP, vp])
    _bind(L, "eik_max_residual_f32", [GP, P, P, P, P, C.c_size_t, C.POINTER(dbl), vp])
    _bind(L, "eik_solve_fim_f32", [GP, P, P, P, P, P, i64, dbl, P, C.c_size_t, SP, vp])
    _bind(L, "eik_local_solve_f32", [C.c_int, P, P, P, P, dbl, dbl, P, i64, vp])
    L.eik_last_error_f32.restype = C.c_char_p
    L.eik_version_f32.restype = C.c_char_p
    _lib32 = _Suffixed(L)
    return _lib32


REMEDY_ENGINES = {0: "none", 1: "list", 2: "tile", 3: "brick"}


def last_remedy_engine(dtype: int = EIK_F64) -> str:
    """Engine of this thread's last remedy step (list / tile / brick, eik_last_remedy_engine)."""
    return REMEDY_ENGINES[int(lib(dtype).eik_last_remedy_engine())]  # the float32 library appends _f32 itself


def check(rc: int, dtype: int | None = None) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == EIK_OK:
        return
    msg = lib(_last_dtype if dtype is None else dtype).eik_last_error().decode(errors="replace")
    if rc == EIK_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)
