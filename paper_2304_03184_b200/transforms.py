"""Dual-quaternion drop-ins of the reference's `capfields.transforms` hot path
(transforms.py:174-196) on the GPU: `dq_blend` (the DQB every ED warp runs per
sample) and `dq_apply`. Same packing ([w,x,y,z | w,x,y,z], real then dual), same
numpy evaluation order (bit-exact: csrc/dq.cuh), same errors: ValueError for a
negative weight, DegenerateWeightsError for a row whose weights sum to <= 0
(transforms.py:189-193). numpy in -> numpy out; CUDA tensors in -> CUDA tensors out.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import dev, host, is_device
from .errors import DegenerateWeightsError  # noqa: F401  (raised through _lib.check)

__all__ = ["dq_blend", "dq_apply", "DegenerateWeightsError"]


def dq_blend(weights, dqs):
    """Weighted dual-quaternion blend over the last-but-one axis (transforms.py:180):
    weights (..., k) non-negative with a positive sum per row, dqs (..., k, 8) ->
    (..., 8); real parts sign-aligned to each row's first entry, result unit-normalised."""
    on_dev = is_device(weights) or is_device(dqs)
    w = weights if is_device(weights) else np.asarray(weights, dtype=np.float64)
    q = dqs if is_device(dqs) else np.asarray(dqs, dtype=np.float64)
    if q.shape[-1] != 8 or tuple(q.shape[:-1]) != tuple(w.shape):
        raise ValueError("dq_blend: weights (..., k) and dqs (..., k, 8) must agree")
    lead = tuple(w.shape[:-1])
    k = int(w.shape[-1]) if len(w.shape) else 0
    n = int(np.prod(lead)) if lead else 1
    wd = dev(w).reshape(n, k)
    qd = dev(q).reshape(n, k, 8)
    out = torch.empty((n, 8), dtype=torch.float64, device=wd.device)
    err = torch.zeros(1, dtype=torch.int32, device=wd.device)
    s = _lib.stream_ptr()
    _lib.call("cf_dq_blend", wd.data_ptr() if k else None, qd.data_ptr() if k else None, n, k, out.data_ptr(),
              err.data_ptr(), s)
    _lib.call("cf_dq_status", err.data_ptr(), s)  # ValueError / DegenerateWeightsError as the reference
    out = out.reshape(*lead, 8)
    return out if on_dev else host(out)


def dq_apply(dq, p):
    """Apply unit dual quaternions (..., 8) to points (..., 3) (transforms.py:174),
    leading dimensions broadcast against each other."""
    on_dev = is_device(dq) or is_device(p)
    qs = tuple(dq.shape[:-1])
    ps = tuple(p.shape[:-1])
    if dq.shape[-1] != 8 or p.shape[-1] != 3:
        raise ValueError("dq_apply: dq (..., 8) and p (..., 3)")
    lead = np.broadcast_shapes(qs, ps)
    n = int(np.prod(lead)) if lead else 1
    qd, pd = dev(dq), dev(p)
    if qs != lead:
        qd = qd.expand(*lead, 8) if qd.numel() > 8 else qd.reshape(8)
    if ps != lead:
        pd = pd.expand(*lead, 3) if pd.numel() > 3 else pd.reshape(3)
    # one dq / one point for every row: stride 0; else materialised rows
    q_stride, p_stride = (0, 0)
    if qd.dim() > 1:
        qd, q_stride = qd.contiguous().reshape(n, 8), 8
    if pd.dim() > 1:
        pd, p_stride = pd.contiguous().reshape(n, 3), 3
    out = torch.empty((n, 3), dtype=torch.float64, device=qd.device)
    _lib.call("cf_dq_apply", qd.data_ptr(), q_stride, pd.data_ptr(), p_stride, n, out.data_ptr(), _lib.stream_ptr())
    out = out.reshape(*lead, 3)
    return out if on_dev else host(out)
