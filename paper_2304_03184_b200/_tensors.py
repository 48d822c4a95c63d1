"""Host <-> device marshalling for the reference-shaped API.

The reference API takes and returns numpy float64 arrays; callers on the hot
path pass CUDA tensors instead and get CUDA tensors back (no host round trip).
"""
from __future__ import annotations

import numpy as np
import torch

from ._lib import require_cuda


def is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def dev(x, dtype=torch.float64, shape_last: int | None = None) -> torch.Tensor:
    """Contiguous CUDA tensor of `dtype` holding x (numpy, list or tensor)."""
    d = require_cuda()
    if isinstance(x, torch.Tensor):
        t = x.to(device=d, dtype=dtype)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=_np_dtype(dtype)))).to(d)
    t = t.contiguous()
    if shape_last is not None:
        t = t.reshape(-1, shape_last) if t.numel() else t.reshape(0, shape_last)
    return t


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def _np_dtype(dtype):
    return {
        torch.float64: np.float64,
        torch.float32: np.float32,
        torch.int32: np.int32,
        torch.int64: np.int64,
        torch.uint8: np.uint8,
        torch.float16: np.float16,
    }[dtype]
