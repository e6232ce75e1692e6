"""Device plumbing: torch owns device memory and streams; the CUDA work is ours."""

from __future__ import annotations

import ctypes

import numpy as np
import torch


_cuda_ok: bool | None = None


def require_cuda() -> torch.device:
    global _cuda_ok
    if _cuda_ok is None:
        _cuda_ok = torch.cuda.is_available()
        if _cuda_ok:
            torch.cuda.init()  # the raw current-device / stream lookups below need torch's CUDA state
    if not _cuda_ok:
        raise RuntimeError("the nbnxn path runs on a CUDA device (sm_100a); none is visible")
    return torch.device("cuda", torch._C._cuda_getDevice())


def stream() -> ctypes.c_void_p:
    """torch's current stream on the current device (raw handle).  The
    public torch.cuda.current_stream() costs ~15 us of interpreter time per
    call -- several calls per MD step -- this lookup well under 1 us."""
    require_cuda()
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


def to_device(a, dtype: torch.dtype, shape=None) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA tensor (no copy when already there)."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=dtype)
    else:
        arr = np.ascontiguousarray(np.asarray(a, dtype=_np_dtype(dtype)))
        if not arr.flags.writeable:
            arr = arr.copy()
        t = torch.from_numpy(arr)
        t = t.to(device=dev, non_blocking=False)
    if shape is not None:
        t = t.reshape(shape)
    return t.contiguous()


def _np_dtype(dtype: torch.dtype):
    return {torch.float64: np.float64, torch.float32: np.float32, torch.int64: np.int64,
            torch.int32: np.int32}[dtype]


def is_device_tensor(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


# ---------------------------------------------------------------- drop-in host staging
# The numpy drop-in entry points (compute_nonbonded_original & co.) move whole
# arrays every call.  Pageable copies run at a fraction of the PCIe rate and
# need a host-side copy of read-only arrays first, so large arrays go through
# grow-only pinned staging buffers with asynchronous copies, and immutable
# (read-only) arrays -- a ParticleSystem's charges and types -- are uploaded
# once and recognised by identity afterwards.
_pinned: dict = {}
_devbuf: dict = {}
_ident: list = []  # [(array, probe, device tensor)], most recent first
_IDENT_MAX = 8


def _buffer(pool: dict, name: str, numel: int, dtype: torch.dtype, pinned: bool) -> torch.Tensor:
    t = pool.get(name)
    if t is None or t.numel() < numel or t.dtype != dtype:
        t = (torch.empty(max(numel, 1), dtype=dtype, pin_memory=True) if pinned
             else torch.empty(max(numel, 1), dtype=dtype, device=require_cuda()))
        pool[name] = t
    return t[:numel]


def _probe(arr: np.ndarray):
    flat = arr.reshape(-1)
    return flat[:16].copy(), flat[-16:].copy()


# Large uploads go in pieces: the host copy of piece k+1 into pinned memory
# overlaps the DMA of piece k (numpy copies run at ~18 GB/s, the link at ~45;
# 96k positions: 0.29 -> 0.18 ms).  Read-backs stay one copy: piecewise
# D2H measured no faster (the host copy into fresh memory dominates).
_PIECE = 1 << 17  # elements (1 MB of FP64)


def _h2d_pipelined(d: torch.Tensor, pin: torch.Tensor, src: np.ndarray) -> None:
    n = src.size
    pv = pin.numpy()
    for a in range(0, n, _PIECE):
        b = min(a + _PIECE, n)
        np.copyto(pv[a:b], src[a:b])
        d[a:b].copy_(pin[a:b], non_blocking=True)


def stage_in(a, dtype: torch.dtype, name: str) -> torch.Tensor:
    """numpy (or tensor) -> CUDA tensor valid until the next stage_in under
    ``name`` on this stream (callers use it within one API call)."""
    if isinstance(a, torch.Tensor):
        return to_device(a, dtype)
    arr = np.asarray(a)
    immutable = not arr.flags.writeable and arr.size > 0
    if immutable:
        for i, (ref, probe, d) in enumerate(_ident):
            if ref is arr and d.dtype == dtype:
                p0, p1 = _probe(arr)
                if np.array_equal(p0, probe[0]) and np.array_equal(p1, probe[1]):
                    if i:
                        _ident.insert(0, _ident.pop(i))
                    return d
                _ident.pop(i)
                break
    npdt = _np_dtype(dtype)
    src = np.ascontiguousarray(arr, dtype=npdt)
    n = src.size
    pin = _buffer(_pinned, name, n, dtype, pinned=True)
    if not immutable:
        d = _buffer(_devbuf, name, n, dtype, pinned=False)
        _h2d_pipelined(d, pin, src.reshape(-1))
        return d.reshape(src.shape)
    # immutable: an own device copy, kept while the array is cached
    d = torch.empty(n, dtype=dtype, device=require_cuda())
    _h2d_pipelined(d, pin, src.reshape(-1))
    d = d.reshape(src.shape)
    _ident.insert(0, (arr, _probe(arr), d))
    del _ident[_IDENT_MAX:]
    return d


def scratch(name: str, numel: int, dtype: torch.dtype) -> torch.Tensor:
    """Grow-only device buffer reused across calls under ``name``."""
    return _buffer(_devbuf, "scratch:" + name, numel, dtype, pinned=False)


def stage_out(t: torch.Tensor, name: str, copy: bool = True) -> np.ndarray:
    """CUDA tensor -> numpy through pinned memory (synchronises).  ``copy``
    False returns a view of the staging buffer, valid until the next
    stage_out under ``name`` (for callers that copy it anyway)."""
    pin = _buffer(_pinned, "out:" + name, t.numel(), t.dtype, pinned=True)
    pin.copy_(t.reshape(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    v = pin.numpy().reshape(tuple(t.shape))
    return v.copy() if copy else v
