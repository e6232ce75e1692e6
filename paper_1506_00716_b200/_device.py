"""Device plumbing: torch owns device memory and streams; the CUDA work is ours."""

from __future__ import annotations

import ctypes

import numpy as np
import torch


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the nbnxn path runs on a CUDA device (sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


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
