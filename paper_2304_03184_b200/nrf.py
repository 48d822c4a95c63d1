"""Radiance-field stages on the GPU — the SPEC `nrf` module:
multi-resolution hash encoding and the tiny density / colour / deformation MLPs.

HashGrid / hash_encode        SPEC.md:345-348, 363-371 (config.py:56-60)
FieldNetworks (E_g, E_c)
DeformNet                     SPEC.md:353-356, 419-420; PAPER.md:307
All math runs in csrc/hashgrid.cu and csrc/mlp.cu / field.cu (tcgen05).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import dev, host, is_device


# ----------------------------------------------------------------- hash grid

@dataclass
class HashGridConfig:
    n_levels: int = 16
    n_features: int = 2
    log2_table: int = 19
    base_resolution: int = 16
    max_resolution: int = 2048


class HashGrid:
    """Learnable multi-resolution hash tables: fp32 parameters (`table`, what
    training updates). With read_half=True the radiance-field kernels read an fp16
    copy (`table_f16`, refreshed by refresh_f16(); half the gather bytes — used for
    the F = 4 deformation grid). The standalone encode API reads the
    fp32 table."""

    def __init__(self, cfg: HashGridConfig | None = None, init_scale: float = 1e-4, seed: int = 0,
                 table: np.ndarray | torch.Tensor | None = None, read_half: bool = False):
        self.cfg = cfg = cfg or HashGridConfig()
        self.desc = _lib.HashGridDesc()
        _lib.call("cf_hashgrid_init", ctypes.byref(self.desc), cfg.n_levels, cfg.n_features, cfg.log2_table,
                  cfg.base_resolution, cfg.max_resolution)
        self.n_entries = int(self.desc.offset[_lib.CF_MAX_LEVELS])
        if table is None:
            g = np.random.default_rng(seed)
            table = g.uniform(-init_scale, init_scale, size=(self.n_entries, cfg.n_features)).astype(np.float32)
        self.table = dev(table, dtype=torch.float32, shape_last=cfg.n_features)
        if self.table.shape[0] != self.n_entries:
            raise ValueError(f"table must have {self.n_entries} entries")
        self.read_half = bool(read_half)
        self.table_f16 = self.table.to(torch.float16) if self.read_half else None

    def refresh_f16(self) -> None:
        """Re-round the fp16 copy after the fp32 table changed (stream-ordered)."""
        if self.read_half:
            self.table_f16.copy_(self.table)

    def table_for_kernels(self) -> torch.Tensor:
        """The tensor the field kernels read (fp16 copy or the fp32 table)."""
        return self.table_f16 if self.read_half else self.table

    def table_as_read(self) -> torch.Tensor:
        """The values the field kernels interpolate, as fp32."""
        return self.table_f16.float() if self.read_half else self.table

    @property
    def out_dim(self) -> int:
        return self.cfg.n_levels * self.cfg.n_features

    def levels(self):
        d = self.desc
        return [(int(d.resolution[l]), bool(d.dense[l]), int(d.offset[l])) for l in range(self.cfg.n_levels)]

    def encode(self, x_unit: torch.Tensor) -> torch.Tensor:
        n = x_unit.shape[0]
        out = torch.empty((n, self.out_dim), dtype=torch.float32, device=x_unit.device)
        _lib.call("cf_hashgrid_encode", ctypes.byref(self.desc), self.table.data_ptr(), x_unit.data_ptr(), int(n),
                  out.data_ptr(), _lib.stream_ptr())
        return out

    def encode_backward(self, x_unit: torch.Tensor, dfeat: torch.Tensor, grad: torch.Tensor) -> None:
        _lib.call("cf_hashgrid_encode_bwd", ctypes.byref(self.desc), x_unit.data_ptr(), dfeat.data_ptr(),
                  int(x_unit.shape[0]), grad.data_ptr(), _lib.stream_ptr())

    def indices(self, x_unit: torch.Tensor):
        n = x_unit.shape[0]
        L = self.cfg.n_levels
        idx = torch.empty((n, L, 8), dtype=torch.int32, device=x_unit.device)
        w = torch.empty((n, L, 8), dtype=torch.float32, device=x_unit.device)
        _lib.call("cf_hashgrid_indices", ctypes.byref(self.desc), x_unit.data_ptr(), int(n), idx.data_ptr(),
                  w.data_ptr(), _lib.stream_ptr())
        return idx, w


def hash_encode(grid: HashGrid, p):
    """SPEC hash_encode: points in [0,1]^3 (clamped) -> L*F features (fp32)."""
    on_dev = is_device(p)
    x = dev(p if on_dev else np.atleast_2d(np.asarray(p, dtype=np.float32)), dtype=torch.float32, shape_last=3)
    out = grid.encode(x)
    return out if on_dev else host(out)


# ----------------------------------------------------------------- MLPs

def pad16(n: int) -> int:
    return (n + 15) // 16 * 16


def pack_weight(W: np.ndarray, lo: bool = False) -> np.ndarray:
    """(N, K) float -> fp16 bytes in the UMMA canonical K-major layout
    [n/8][k/8][n%8][k%8] with N, K zero-padded to multiples of 16. lo=True packs
    the residual fp16(W - fp16(W)) instead (the "fp32" precision mode's B halves)."""
    W = np.asarray(W, dtype=np.float32)
    n, k = W.shape
    Np, Kp = pad16(n), pad16(k)
    P = np.zeros((Np, Kp), dtype=np.float16)
    h = W.astype(np.float16)
    P[:n, :k] = (W - h.astype(np.float32)).astype(np.float16) if lo else h
    return P.reshape(Np // 8, 8, Kp // 8, 8).transpose(0, 2, 1, 3).reshape(-1).view(np.uint8)


class MLP:
    """Bias-optional ReLU chain; weights stored fp16 (as the tensor cores read them)."""

    def __init__(self, widths, seed: int = 0, weights=None, biases=None, zero_last: bool = False):
        self.widths = [int(w) for w in widths]
        rng = np.random.default_rng(seed)
        if weights is None:
            weights = []
            for l in range(len(self.widths) - 1):
                fan_in = self.widths[l]
                bound = np.sqrt(6.0 / fan_in)  # Kaiming-uniform (ReLU)
                weights.append(rng.uniform(-bound, bound, size=(self.widths[l + 1], fan_in)))
            if zero_last:
                weights[-1] = np.zeros_like(weights[-1])
        self.weights = [np.asarray(w, dtype=np.float32).astype(np.float16).astype(np.float32) for w in weights]
        self.biases = biases  # list (None or (N,) array) per layer
        self.n_layers = len(self.weights)
        self._upload()

    def _upload(self):
        blob = np.concatenate([pack_weight(w) for w in self.weights])
        self.w_bytes = int(blob.size)
        self.blob = dev(blob.view(np.uint8).copy(), dtype=torch.uint8)
        b = np.zeros((self.n_layers, 128), dtype=np.float32)
        has = np.zeros(self.n_layers, dtype=np.int32)
        if self.biases is not None:
            for l, bl in enumerate(self.biases):
                if bl is not None:
                    b[l, :len(bl)] = bl
                    has[l] = 1
        self.bias = dev(b, dtype=torch.float32)
        self._has = (ctypes.c_int * self.n_layers)(*[int(v) for v in has])
        self._widths = (ctypes.c_int * (self.n_layers + 1))(*self.widths)

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        x = x.contiguous()
        n = x.shape[0]
        y = torch.empty((n, self.widths[-1]), dtype=torch.float32, device=x.device)
        _lib.call("cf_mlp_forward", self.n_layers, self._widths, self.blob.data_ptr(), self.w_bytes,
                  self.bias.data_ptr(), self._has, x.data_ptr(), int(n), y.data_ptr(), _lib.stream_ptr())
        return y
