"""Oracle for the dense symmetric pipeline (Fig. 3:
reduction to tridiagonal form, the tridiagonal eigensolver, back-transformation).

TEST INFRASTRUCTURE ONLY (same rule as oracle/__init__.py): only tests/, smoke() and bench.py's
cpu_baseline / --impl reference legs may import it; it shares no code with the CUDA path.

Plain, slow, textbook binary64 (numpy):
  householder_tridiag(A): for k = 0..n-3 the Householder reflector H_k = I - 2 u u^T (u a unit
      vector) that maps A[k+1:, k] onto a multiple of e_1 is applied from both sides,
      A <- H_k A H_k, and accumulated, Q <- Q H_k (Golub & Van Loan, "Householder
      tridiagonalization"); afterwards A is tridiagonal, A_in = Q T Q^T.  No blocking, no
      symmetric-update tricks: every reflector is applied to the full matrix as two rank-1
      updates, in the order the definition states.
  eig_dense(A, idx): T's eigenpairs from the binary128 tridiagonal oracle (bisection on T +
      inverse iteration, oracle.c), then z = Q y (the back-transformation).
The tridiagonal stage is binary128; the reduction is binary64, so the result is backward stable
to c n eps_x ||A|| (the accuracy the dense pipeline can have, whatever the tridiagonal solver).
"""
from __future__ import annotations

import numpy as np

from . import norm1, solve


def householder_tridiag(A):
    """Returns (d, e, Q) with A = Q T Q^T, T = tridiag(e, d, e)."""
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    n = A.shape[0]
    Q = np.eye(n)
    for k in range(n - 2):
        x = A[k + 1:, k].copy()
        nx = np.linalg.norm(x)
        if nx == 0.0:
            continue
        alpha = -nx if x[0] >= 0.0 else nx   # H x = alpha e_1, sign chosen against cancellation
        u = x.copy()
        u[0] -= alpha
        nu = np.linalg.norm(u)
        if nu == 0.0:
            continue
        u /= nu
        # A <- H A H with H = I - 2 u u^T acting on rows / columns k+1..n-1
        A[k + 1:, :] -= 2.0 * np.outer(u, u @ A[k + 1:, :])
        A[:, k + 1:] -= 2.0 * np.outer(A[:, k + 1:] @ u, u)
        Q[:, k + 1:] -= 2.0 * np.outer(Q[:, k + 1:] @ u, u)
    d = np.diag(A).copy()
    e = np.diag(A, -1).copy()
    return d, e, Q


def eig_dense(A, idx=None):
    """Eigenpairs of the dense symmetric A: (w, Z, (d, e, Q)); w binary64 (rounded from the
    binary128 eigenvalues of the reduced T), Z = Q y."""
    d, e, Q = householder_tridiag(A)
    n = d.shape[0]
    if idx is None:
        idx = np.arange(1, n + 1)
    lh, ll, Yh, Yl = solve(d, e, idx)
    Y = Yh + Yl
    return lh + ll, Q @ Y, (d, e, Q)


def dense_norm1(A) -> float:
    return float(np.max(np.sum(np.abs(A), axis=0)))


def residual_orth(A, w, Z):
    """max_j ||A z_j - w_j z_j||_2 / ||A||_1 and max |Z^T Z - I| (binary64 with the products
    accumulated by numpy; the dense stage's own error is far above their rounding)."""
    nrm = dense_norm1(A)
    R = A @ Z - Z * w[None, :]
    r = float(np.max(np.linalg.norm(R, axis=0))) / nrm
    G = Z.T @ Z - np.eye(Z.shape[1])
    return r, float(np.max(np.abs(G)))
