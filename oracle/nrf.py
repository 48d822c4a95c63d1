"""ORACLE (test infrastructure only) — stages 2-4 on the CPU.

Restatement of SPEC.md's `nrf` module, which has no code and
no tests in the reference: parity UNPINNED by the reference; pinned only by the
SPEC's worked examples (tests/test_oracle_nrf.py). The hyper-parameter choices
the SPEC leaves open are frozen in DESIGN.md §4-§6 and restated here.

Precision modes: hash encoding is evaluated in float32 with the kernel's exact
operation order (indices bit-exact, features bit-equal). MLPs either in the
SPEC's 32-bit semantics (`mlp_forward_f32`: fp32 weights and inputs, float64
arithmetic — the reference the "fp32" device mode is held to), or in "kernel
precision" of the "fp16" device mode (`mlp_forward`: fp16-rounded operands per
layer, float64 accumulation).
"""
from __future__ import annotations

import math

import numpy as np

PRIMES = (np.uint32(1), np.uint32(2654435761), np.uint32(805459861))


def hash_levels(n_levels, log2_table, base_res, max_res):
    """(resolution, dense, offset) per level + total entries."""
    b = math.exp((math.log(max_res) - math.log(base_res)) / (n_levels - 1)) if n_levels > 1 else 1.0
    T = 1 << log2_table
    out, off = [], 0
    for l in range(n_levels):
        N = int(math.floor(base_res * math.pow(b, l) + 1e-9))
        dense = (N + 1) ** 3 <= T
        out.append((N, dense, off))
        off += ((N + 1) ** 3 + 7) // 8 * 8 if dense else T
    return out, off


def hash_corners(x_unit, level, log2_table):
    """Per-level corner indices (N, 8) uint32 and trilinear weights (N, 8) float32."""
    N, dense, _ = level
    x = np.clip(np.asarray(x_unit, dtype=np.float32), np.float32(0), np.float32(1))
    pos = x * np.float32(N)
    g = np.minimum(np.floor(pos), np.float32(N - 1)).astype(np.int64)
    fr = pos - g.astype(np.float32)
    idx = np.empty((len(x), 8), dtype=np.uint32)
    w = np.empty((len(x), 8), dtype=np.float32)
    one = np.float32(1)
    for c in range(8):
        bit = np.array([c & 1, (c >> 1) & 1, (c >> 2) & 1])
        xyz = (g + bit).astype(np.uint32)
        if dense:
            s = np.uint32(N + 1)
            idx[:, c] = xyz[:, 0] + xyz[:, 1] * s + xyz[:, 2] * s * s
        else:
            h = (xyz[:, 0] * PRIMES[0]) ^ (xyz[:, 1] * PRIMES[1]) ^ (xyz[:, 2] * PRIMES[2])
            idx[:, c] = h & np.uint32((1 << log2_table) - 1)
        wx = fr[:, 0] if bit[0] else one - fr[:, 0]
        wy = fr[:, 1] if bit[1] else one - fr[:, 1]
        wz = fr[:, 2] if bit[2] else one - fr[:, 2]
        w[:, c] = (wx * wy) * wz
    return idx, w


def hash_encode(table, x_unit, n_levels=16, n_features=2, log2_table=19, base_res=16, max_res=2048):
    """SPEC hash_encode, float32, fixed corner order."""
    levels, total = hash_levels(n_levels, log2_table, base_res, max_res)
    table = np.asarray(table, dtype=np.float32).reshape(total, n_features)
    out = np.empty((len(x_unit), n_levels * n_features), dtype=np.float32)
    with np.errstate(over="ignore"):
        for l, (N, dense, off) in enumerate(levels):
            idx, w = hash_corners(x_unit, (N, dense, off), log2_table)
            acc = w[:, 0:1] * table[off + idx[:, 0]]
            for c in range(1, 8):
                acc = acc + w[:, c:c + 1] * table[off + idx[:, c]]
            out[:, l * n_features:(l + 1) * n_features] = acc
    return out


def hash_encode_bwd(x_unit, dfeat, n_levels=16, n_features=2, log2_table=19, base_res=16, max_res=2048):
    """dL/dtable of hash_encode (float64 accumulation)."""
    levels, total = hash_levels(n_levels, log2_table, base_res, max_res)
    grad = np.zeros((total, n_features))
    with np.errstate(over="ignore"):
        for l, (N, dense, off) in enumerate(levels):
            idx, w = hash_corners(x_unit, (N, dense, off), log2_table)
            g = dfeat[:, l * n_features:(l + 1) * n_features].astype(np.float64)
            for c in range(8):
                np.add.at(grad, off + idx[:, c].astype(np.int64), w[:, c:c + 1].astype(np.float64) * g)
    return grad


def f16(x):
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float64)


def mlp_forward(weights, x, biases=None):
    """Kernel-precision MLP: fp16-rounded weights and layer inputs, float64
    accumulation, ReLU between layers, no output activation."""
    h = f16(x)
    n = len(weights)
    for l, W in enumerate(weights):
        y = h @ f16(W).T
        if biases is not None and biases[l] is not None:
            y = y + np.asarray(biases[l], dtype=np.float32).astype(np.float64)
        if l < n - 1:
            h = f16(np.maximum(y.astype(np.float32), 0.0))
        else:
            return y


def mlp_forward_f32(weights, x, biases=None):
    """SPEC 32-bit semantics: the fp32 weights and layer inputs
    exactly, float64 accumulation, ReLU between layers, no output activation."""
    h = np.asarray(x, dtype=np.float32).astype(np.float64)
    n = len(weights)
    for l, W in enumerate(weights):
        y = h @ np.asarray(W, dtype=np.float32).astype(np.float64).T
        if biases is not None and biases[l] is not None:
            y = y + np.asarray(biases[l], dtype=np.float32).astype(np.float64)
        if l < n - 1:
            h = np.maximum(y, 0.0)
        else:
            return y
