"""Dispatch and parity helpers for the iFIM path (E/harness.py:54-57, 121-179).

``run_method`` keeps the reference's string dispatch (the plugin point every
CLI command goes through, E/harness.py:121-144).  "ifim", "fim" (the paper's
baseline, E/fim.py) and "oracle" (the fixpoint ground truth, E/oracle.py) are
served by this package; fmm and fsm are out of scope and raise
like an unknown method would.
"""
from __future__ import annotations

import hashlib

import numpy as np
import torch

from .fim import solve_fim
from .fixpoint import max_residual, solve_fixpoint  # noqa: F401  (re-exported)
from .ifim import solve_ifim
from .result import SolverResult

METHOD_NAMES = ("fim", "ifim", "oracle")
PARALLEL_METHODS = frozenset({"fim", "ifim", "oracle"})


def run_method(method: str, grid, bc, tol: float = 1e-12, workers: int = 1) -> SolverResult:
    """E/harness.py:121-144 restricted to the accelerated method."""
    if method == "fim":
        return solve_fim(grid, bc, tol=tol, workers=workers)
    if method == "ifim":
        return solve_ifim(grid, bc, tol=tol, workers=workers)
    if method == "oracle":
        return solve_fixpoint(grid, bc, tol=tol, workers=workers)
    raise ValueError(f"unknown method {method!r}, expected one of {METHOD_NAMES}")


def _np(a):
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def _cuda(t) -> bool:
    return isinstance(t, torch.Tensor) and t.is_cuda


def _lib_for(t):
    from . import _native

    return _native.lib(_native.EIK_F32 if t.dtype == torch.float32 else _native.EIK_F64), _native


def _stream(t):
    import ctypes as C

    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def field_max_diff(a, b) -> float:
    """E/harness.py:165-174: max |a - b|, equal same-sign infinities count as 0.

    Two CUDA tensors of the same float dtype are reduced on the device (eik_field_max_diff, no
    host copy of either field); anything else goes through numpy like the reference."""
    if _cuda(a) and _cuda(b) and a.dtype == b.dtype and a.dtype in (torch.float64, torch.float32) \
            and a.device == b.device:
        import ctypes as C

        if tuple(a.shape) != tuple(b.shape):
            raise ValueError(f"field shapes differ: {tuple(a.shape)} vs {tuple(b.shape)}")
        a, b = a.contiguous(), b.contiguous()
        L, nat = _lib_for(a)
        scratch = torch.empty(2, dtype=torch.int64, device=a.device)
        out = C.c_double(0.0)
        nat.check(L.eik_field_max_diff(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), a.numel(),
                                       C.c_void_p(scratch.data_ptr()), C.byref(out), _stream(a)))
        return float(out.value)
    a, b = _np(a), _np(b)
    if a.shape != b.shape:
        raise ValueError(f"field shapes differ: {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    with np.errstate(invalid="ignore"):
        diff = np.abs(a - b)
    return float(np.where(both_inf, 0.0, diff).max())


_STREAM_BYTES = 1 << 26  # field_sha256 of a CUDA tensor: bytes per pinned staging buffer


def field_sha256(phi) -> str:
    """E/harness.py:177-179: digest of the raw field bytes (C order).

    A CUDA tensor is streamed to the host in 64 MiB pieces through two pinned buffers (the copy
    of the next piece overlaps the hashing of this one), so no full-size host copy is made; the
    digest is the reference's, byte for byte."""
    if _cuda(phi):
        h = hashlib.sha256()
        if phi.numel() == 0:
            return h.hexdigest()
        t = phi.detach().contiguous().reshape(-1).view(torch.uint8)
        n = t.numel()
        step = min(_STREAM_BYTES, n)
        bufs = [torch.empty(step, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        stream = torch.cuda.current_stream(t.device)
        events = [None, None]
        pieces = list(range(0, n, step))
        for k, off in enumerate(pieces[:2]):
            m = min(step, n - off)
            bufs[k][:m].copy_(t[off:off + m], non_blocking=True)
            events[k] = torch.cuda.Event()
            events[k].record(stream)
        for k, off in enumerate(pieces):
            m = min(step, n - off)
            events[k & 1].synchronize()
            h.update(bufs[k & 1][:m].numpy())
            nxt = k + 2
            if nxt < len(pieces):
                o2 = pieces[nxt]
                m2 = min(step, n - o2)
                bufs[k & 1][:m2].copy_(t[o2:o2 + m2], non_blocking=True)
                events[k & 1] = torch.cuda.Event()
                events[k & 1].record(stream)
        return h.hexdigest()
    return hashlib.sha256(np.ascontiguousarray(_np(phi)).tobytes()).hexdigest()


DIGEST_CHUNK = 1 << 16


def field_digest(phi, chunk: int = DIGEST_CHUNK) -> str:
    """Chunked field digest: sha256 over the concatenated sha256 digests of the raw field bytes
    (C order) cut into ``chunk``-byte pieces (the last may be short).  Equal fields have equal
    digests and any changed byte changes it, like field_sha256, but the piece digests of a CUDA
    tensor are computed on the device in parallel (eik_chunk_sha256): 32 bytes per 64 KiB leave
    the GPU.  Host arrays compute the same value with hashlib."""
    if chunk <= 0 or chunk % 64:
        raise ValueError("chunk must be a positive multiple of 64 bytes")
    if _cuda(phi):
        import ctypes as C

        if phi.numel() == 0:
            return hashlib.sha256(b"").hexdigest()
        t = phi.detach().contiguous().reshape(-1).view(torch.uint8)
        if t.data_ptr() % 16:
            t = t.clone()
        n = t.numel()
        pieces = (n + chunk - 1) // chunk
        dig = torch.empty(max(pieces, 1) * 32, dtype=torch.uint8, device=t.device)
        L, nat = _lib_for(phi)
        nat.check(L.eik_chunk_sha256(C.c_void_p(t.data_ptr()), n, chunk, C.c_void_p(dig.data_ptr()), _stream(t)))
        return hashlib.sha256(dig[: pieces * 32].cpu().numpy().tobytes()).hexdigest()
    b = np.ascontiguousarray(_np(phi)).tobytes()
    return hashlib.sha256(b"".join(hashlib.sha256(b[o:o + chunk]).digest()
                                   for o in range(0, len(b), chunk))).hexdigest()
