"""Non-rigid tracking solve: the cooperative-kernel PCG against the
reference's pcg_solve on its own tracker's Gauss-Newton system (tests/golden/
make_pcg.py; tracking.py:158-193, 358-508) and the oracle restatement.

Tolerance: the tracker's systems are ill-conditioned and 32 CG iterations do not
converge at small damping, so rounding differences are amplified: a 1e-15 relative
perturbation of r changes the REFERENCE's own x by 0.7 % at lambda = 1e-4 (measured in
make_pcg.py's setting). The comparison is therefore per regime: at lambda = 1 (well
conditioned) and for the converged tight-tolerance solve the iterates themselves match
(1e-10 / 1e-6 relative); for the unconverged solves the CG objective
q(x) = x^T A x / 2 - b^T x (what CG minimises over the Krylov space) and the damped
residual |A x - b| / |b| must lie inside the reference's own rounding envelope, measured
by re-running the reference with r perturbed by 1e-15 relative noise (8 draws):
lambda = 1e-4: q spread 4.1e-4, residual spread 8.4 %; lambda = 1e-2: q 2.3e-7,
residual 0.06 %. The bounds below are 5x / 3x those spreads.
"""
ENVELOPE = {0: (2e-3, 0.25), 1: (1.2e-6, 2e-3)}  # case -> (q rel, residual rel)
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import tracking as otr


@pytest.fixture(scope="module")
def ref():
    with np.load(os.path.join(GOLDEN, "pcg_ref.npz")) as z:
        return {k: z[k] for k in z.files}


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _objective(ref, lam, x):
    """CG objective and relative residual of the damped normal equations."""
    val, col, rowptr, shape = ref["val"], ref["col"], ref["rowptr"], ref["shape"]
    import scipy.sparse as sp
    J = sp.csr_matrix((val, col, rowptr), shape=tuple(shape))
    b = -(J.T @ ref["r"])
    d = np.asarray(J.multiply(J).sum(axis=0)).reshape(-1)
    Ax = J.T @ (J @ x) + lam * d * x
    return 0.5 * x @ Ax - b @ x, np.linalg.norm(Ax - b) / np.linalg.norm(b)


def _check(ref, i, x):
    lam, it, tol = ref["cases"][i]
    xr = ref[f"x{i}"]
    if lam >= 1.0:
        assert _rel(x, xr) <= 1e-10, (i, _rel(x, xr))
    elif it > 100:
        assert _rel(x, xr) <= 1e-6, (i, _rel(x, xr))
    else:
        q, res = _objective(ref, lam, x)
        qr, resr = _objective(ref, lam, xr)
        tq, tr = ENVELOPE[i]
        assert abs(q - qr) <= tq * abs(qr), (i, q, qr)
        assert abs(res - resr) <= tr * resr, (i, res, resr)


def test_oracle_matches_reference(ref):
    J = (ref["val"], ref["col"], ref["rowptr"], ref["shape"])
    for i, (lam, it, tol) in enumerate(ref["cases"]):
        if it > 100:
            continue  # the pure-Python oracle is slow at 400 iterations
        _check(ref, i, otr.pcg_solve(*J, ref["r"], lam, int(it), tol))


@pytest.mark.gpu
def test_gpu_pcg_matches_reference(ref):
    from paper_2304_03184_b200.tracking import GaussNewtonSystem, pcg_solve
    J = (ref["val"], ref["col"], ref["rowptr"], ref["shape"])
    sysm = GaussNewtonSystem(J, ref["r"])
    for i, (lam, it, tol) in enumerate(ref["cases"]):
        _check(ref, i, sysm.solve(lam, int(it), tol).cpu().numpy())
    _check(ref, 0, pcg_solve(J, ref["r"], 1e-4))


@pytest.mark.gpu
def test_gpu_pcg_edge_cases():
    from paper_2304_03184_b200.tracking import pcg_solve
    rng = np.random.default_rng(4)
    rows, cols = 300, 80
    dense = rng.normal(size=(rows, cols)) * (rng.random((rows, cols)) < 0.1)
    dense[:, 7] = 0.0  # an unconstrained unknown: zero diagonal, zero preconditioner
    nz = np.nonzero(dense)
    order = np.lexsort((nz[1], nz[0]))
    r_i, c_i = nz[0][order], nz[1][order]
    val = dense[r_i, c_i]
    rowptr = np.concatenate([[0], np.cumsum(np.bincount(r_i, minlength=rows))]).astype(np.int32)
    J = (val, c_i.astype(np.int32), rowptr, (rows, cols))
    r = rng.normal(size=rows)
    for lam, it, tol in ((1e-3, 32, 1e-6), (0.5, 5, 1e-6), (1e-6, 200, 1e-14)):
        x = pcg_solve(J, r, lam, it, tol)
        xo = otr.pcg_solve(*J, r, lam, it, tol)
        assert _rel(x, xo) <= 1e-7 and x[7] == 0.0  # well-conditioned random system
    assert not np.any(pcg_solve(J, np.zeros(rows), 1e-3))  # b = 0 -> x = 0
