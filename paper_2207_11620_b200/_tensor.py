"""Host/device argument plumbing shared by the API modules.

The reference API takes and returns numpy arrays.  Here every public
function accepts numpy arrays or torch tensors: device tensors stay on the
device; numpy inputs are uploaded and the result is returned as numpy again
(the host<->device copies a drop-in caller would otherwise write by hand).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib

_NP2T = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
         np.dtype(np.int64): torch.int64, np.dtype(np.uint8): torch.uint8,
         np.dtype(np.int32): torch.int32}


def torch_dtype(dtype) -> torch.dtype:
    if isinstance(dtype, torch.dtype):
        return dtype
    return _NP2T[np.dtype(dtype)]


def np_dtype(dtype) -> np.dtype:
    if isinstance(dtype, torch.dtype):
        return {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64)}[dtype]
    return np.dtype(dtype)


def to_device(x, dtype=None) -> tuple[torch.Tensor, bool]:
    """(contiguous device tensor, came_from_host)."""
    if isinstance(x, torch.Tensor):
        t = x
        host = not t.is_cuda
        if dtype is not None and t.dtype != torch_dtype(dtype):
            t = t.to(torch_dtype(dtype))
        if host:
            t = t.to(_lib.device(), non_blocking=False)
        return t.contiguous(), host
    a = np.asarray(x)
    if dtype is not None:
        a = a.astype(np_dtype(dtype), copy=False)
    t = torch.from_numpy(np.ascontiguousarray(a)).to(_lib.device())
    return t, True


def out(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t
