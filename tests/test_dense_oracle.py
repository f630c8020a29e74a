"""Pins of the dense-pipeline oracle (oracle/dense.py, PAPER.md
L1506-L1550) against things other than itself: LAPACK's dsyevd (numpy.linalg.eigvalsh, a
different algorithm), closed forms (1-2-1 under a random orthogonal similarity), exact special
cases (diagonal and already-tridiagonal input, n <= 2) and the defining identities
A = Q T Q^T, Q^T Q = I, A z = lambda z."""
import numpy as np
import pytest

import synth
from oracle import dense

EPS = 2.0 ** -53


def _tri(d, e):
    return np.diag(d) + np.diag(e, 1) + np.diag(e, -1)


@pytest.mark.parametrize("n,seed", [(7, 0), (50, 1), (120, 2)])
def test_reduction_identities(n, seed):
    p = synth.dense_from(synth.random_uniform(n, seed), seed)
    d, e, Q = dense.householder_tridiag(p.A)
    nrm = dense.dense_norm1(p.A)
    assert np.max(np.abs(Q.T @ Q - np.eye(n))) <= 8 * n * EPS
    assert np.max(np.abs(Q @ _tri(d, e) @ Q.T - p.A)) <= 8 * n * EPS * nrm
    # the reduced T keeps the spectrum of A (LAPACK dsyevd on both)
    assert np.max(np.abs(np.linalg.eigvalsh(_tri(d, e)) - np.linalg.eigvalsh(p.A))) <= 8 * n * EPS * nrm


@pytest.mark.parametrize("n,seed", [(40, 3), (150, 4)])
def test_eigenpairs_vs_lapack(n, seed):
    p = synth.dense_from(synth.random_uniform(n, seed), seed)
    w, Z, _ = dense.eig_dense(p.A)
    nrm = dense.dense_norm1(p.A)
    assert np.max(np.abs(w - np.linalg.eigvalsh(p.A))) <= 8 * n * EPS * nrm
    r, o = dense.residual_orth(p.A, w, Z)
    assert r <= 8 * n * EPS and o <= 8 * n * EPS, (r, o)


def test_closed_form_121_under_similarity():
    """A = Q0 tridiag(1, 2, 1) Q0^T: eigenvalues 2 - 2 cos(k pi / (n + 1)), eigenvectors
    +-Q0 s_k with s_k(j) = sqrt(2 / (n + 1)) sin(j (n + 1 - k) pi / (n + 1)) (T s = (2 + 2 cos) s
    for the sine vectors, so ascending order reverses their index)."""
    n = 64
    p = synth.dense_from(synth.one_two_one(n), 5)
    Q0 = synth.random_orthogonal(n, 5)
    w, Z, _ = dense.eig_dense(p.A)
    k = np.arange(1, n + 1)
    assert np.max(np.abs(w - (2 - 2 * np.cos(k * np.pi / (n + 1))))) <= 8 * n * EPS * 4
    j = np.arange(1, n + 1)
    S = np.sqrt(2.0 / (n + 1)) * np.sin(np.outer(j, n + 1 - k) * np.pi / (n + 1))
    ref = Q0 @ S
    sgn = np.sign(np.sum(ref * Z, axis=0))
    gaps = np.minimum(np.diff(np.r_[-np.inf, w]), np.diff(np.r_[w, np.inf]))
    err = np.linalg.norm(Z - ref * sgn[None, :], axis=0)
    assert np.all(err <= 8 * n * EPS * 4 / gaps + 1e-14), err.max()


def test_special_cases():
    # diagonal input: nothing to reduce
    a = np.array([3.0, -1.0, 2.0, 0.5])
    d, e, Q = dense.householder_tridiag(np.diag(a))
    assert np.array_equal(d, a) and np.all(e == 0) and np.array_equal(Q, np.eye(4))
    # already tridiagonal: the reflectors only flip signs (|e| and d kept)
    t = synth.random_small(9, 1)
    d, e, Q = dense.householder_tridiag(_tri(t.d, t.e))
    assert np.allclose(d, t.d, rtol=0, atol=4 * EPS) and np.allclose(np.abs(e), np.abs(t.e), atol=4 * EPS)
    assert np.allclose(np.abs(Q), np.eye(9), atol=4 * EPS)
    # n = 1, 2: T = A, Q = I
    for A in (np.array([[2.5]]), np.array([[1.0, 0.25], [0.25, -3.0]])):
        d, e, Q = dense.householder_tridiag(A)
        assert np.array_equal(_tri(d, e), A) and np.array_equal(Q, np.eye(A.shape[0]))
        w, Z, _ = dense.eig_dense(A)
        assert np.allclose(w, np.linalg.eigvalsh(A), atol=4 * EPS * 4)
