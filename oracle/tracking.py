"""CPU restatement of the tracker's PCG solve — TEST INFRASTRUCTURE ONLY.

pcg_solve (tracking.py:158-193): Jacobi-preconditioned CG on the damped normal
equations (J^T J + lambda diag(J^T J)) x = -J^T r, with J in CSR as
(val, col, rowptr, shape). Pinned against the reference's own outputs on its
tracker's systems (tests/golden/make_pcg.py -> tests/golden/pcg_ref.npz).
"""
from __future__ import annotations

import numpy as np


def _matvec(val, col, rowptr, v):
    out = np.zeros(len(rowptr) - 1)
    for i in range(len(out)):
        a, b = rowptr[i], rowptr[i + 1]
        out[i] = np.dot(val[a:b], v[col[a:b]])
    return out


def _rmatvec(val, col, rowptr, n_cols, w):
    out = np.zeros(n_cols)
    for i in range(len(rowptr) - 1):
        a, b = rowptr[i], rowptr[i + 1]
        np.add.at(out, col[a:b], val[a:b] * w[i])
    return out


def pcg_solve(val, col, rowptr, shape, r, lm_lambda, max_iters=32, tol=1e-6):
    n = int(shape[1])
    b = -_rmatvec(val, col, rowptr, n, r)
    if not np.any(b):
        return np.zeros(n)
    diag = _rmatvec(val * val, col, rowptr, n, np.ones(len(rowptr) - 1))
    damped = (1.0 + lm_lambda) * diag
    m_inv = np.where(damped > 1e-300, 1.0 / np.maximum(damped, 1e-300), 0.0)
    lam_d = lm_lambda * diag
    x = np.zeros(n)
    res = b.copy()
    z = m_inv * res
    p = z.copy()
    rz = float(res @ z)
    b_norm = np.linalg.norm(b)
    for _ in range(max_iters):
        Ap = _rmatvec(val, col, rowptr, n, _matvec(val, col, rowptr, p)) + lam_d * p
        pAp = float(p @ Ap)
        if pAp <= 0:
            break
        alpha = rz / pAp
        x += alpha * p
        res -= alpha * Ap
        if np.linalg.norm(res) <= tol * b_norm:
            break
        z = m_inv * res
        rz_new = float(res @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x


def pcg_solve_sparse(J, r, lm_lambda, max_iters=32, tol=1e-6):
    """The same algorithm with scipy.sparse products (the reference's formulation,
    tracking.py:158-193) — the CPU baseline bench.py times."""
    b = -(J.T @ r)
    if not np.any(b):
        return np.zeros(J.shape[1])
    diag = np.asarray(J.multiply(J).sum(axis=0)).reshape(-1)
    damped = (1.0 + lm_lambda) * diag
    m_inv = np.where(damped > 1e-300, 1.0 / np.maximum(damped, 1e-300), 0.0)
    lam_d = lm_lambda * diag
    x = np.zeros_like(b)
    res = b.copy()
    z = m_inv * res
    p = z.copy()
    rz = float(res @ z)
    b_norm = np.linalg.norm(b)
    for _ in range(max_iters):
        Ap = J.T @ (J @ p) + lam_d * p
        pAp = float(p @ Ap)
        if pAp <= 0:
            break
        alpha = rz / pAp
        x += alpha * p
        res -= alpha * Ap
        if np.linalg.norm(res) <= tol * b_norm:
            break
        z = m_inv * res
        rz_new = float(res @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x
