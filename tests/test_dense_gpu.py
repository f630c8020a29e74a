"""GPU parity of the dense symmetric pipeline (NEXT-4) through the C-ABI
(mr3_dsyevr_dd) against the dense oracle (oracle/dense.py: textbook Householder reduction +
binary128 tridiagonal oracle + back-transformation) and LAPACK dsyevd.

Tolerances (R23): a Householder reduction in binary64 is backward stable,
||dA|| <= c n eps ||A|| (c small), and so is the oracle's; eigenvalues of the two agree to
8 n eps ||A||_1, residuals max_j ||A z_j - w_j z_j||_2 / ||A||_1 and orthogonality
max |Z^T Z - I| are <= 8 n eps, and a column z_j with gap g_j to the rest of the spectrum
is within sin-angle 16 n eps ||A||_1 / g_j of the oracle's (Gap theorem on both residuals)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1304_1864_b200 as mr3
import synth
from oracle import dense

pytestmark = pytest.mark.gpu
EPS = 2.0 ** -53


def run(A, **kw):
    w, Z, st = mr3.mr3_dsyevr_dd(torch.from_numpy(np.ascontiguousarray(A)).cuda(), **kw)
    torch.cuda.synchronize()
    return w.cpu().numpy(), (Z.cpu().numpy() if Z is not None else None), st


def _check(A, w, Z, idx=None, oracle_vectors=True):
    n = A.shape[0]
    nrm = dense.dense_norm1(A)
    lap = np.linalg.eigvalsh(A)
    if idx is None:
        idx = np.arange(1, n + 1)
    assert np.max(np.abs(w - lap[idx - 1])) <= 8 * n * EPS * nrm
    r, o = dense.residual_orth(A, w, Z)
    assert r <= 8 * n * EPS and o <= 8 * n * EPS, (r, o)
    if oracle_vectors:
        wo, Zo, _ = dense.eig_dense(A, idx)
        assert np.max(np.abs(w - wo)) <= 8 * n * EPS * nrm
        full = lap
        gaps = []
        for k in idx:
            g = np.inf
            if k >= 2:
                g = min(g, full[k - 1] - full[k - 2])
            if k <= n - 1:
                g = min(g, full[k] - full[k - 1])
            gaps.append(g)
        gaps = np.array(gaps)
        sgn = np.where(np.sum(Z * Zo, axis=0) < 0, -1.0, 1.0)
        err = np.linalg.norm(Z - Zo * sgn[None, :], axis=0)
        bound = 16 * n * EPS * nrm / np.maximum(gaps, 1e-300) + 1e-13
        assert np.all(err <= bound), (err / bound).max()


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (3, 2), (37, 3), (200, 4), (515, 5)])
def test_dense_random(n, seed):
    p = synth.dense_from(synth.random_uniform(n, seed), seed)
    w, Z, st = run(p.A)
    _check(p.A, w, Z)


def test_dense_closed_form_121():
    n = 300
    p = synth.dense_from(synth.one_two_one(n), 6)
    w, Z, st = run(p.A)
    k = np.arange(1, n + 1)
    assert np.max(np.abs(w - (2 - 2 * np.cos(k * np.pi / (n + 1))))) <= 8 * n * EPS * 4
    _check(p.A, w, Z, oracle_vectors=False)


def test_dense_diagonal_and_subset():
    a = np.linspace(-2.0, 3.0, 64)
    w, Z, st = run(np.diag(a))
    assert np.array_equal(w, np.sort(a))
    assert np.max(np.abs(np.abs(Z) - np.eye(64))) <= 4 * EPS
    p = synth.dense_from(synth.glued_wilkinson(4, 21), 7)   # clustered spectrum, tree depth >= 1
    w, Z, st = run(p.A, range="I", il=20, iu=60)
    assert w.shape == (41,) and Z.shape == (p.n, 41)
    _check(p.A, w, Z, np.arange(20, 61), oracle_vectors=False)
    wn, Zn, _ = run(p.A, jobz="N")
    assert Zn is None and np.max(np.abs(wn - np.linalg.eigvalsh(p.A))) <= 8 * p.n * EPS * 12


@pytest.mark.slow
def test_dense_bench_size():
    """The bench workload's size (n = 4096): eigenvalues against LAPACK, residual and
    orthogonality of every column (GPU fp64 products)."""
    p = synth.dense_config(4096, 0)
    A = torch.from_numpy(np.ascontiguousarray(p.A)).cuda()
    w, Z, st = mr3.mr3_dsyevr_dd(A)
    n = p.n
    nrm = float(A.abs().sum(0).max())
    lap = np.linalg.eigvalsh(p.A)
    assert np.max(np.abs(w.cpu().numpy() - lap)) <= 8 * n * EPS * nrm
    R = A @ Z - Z * w[None, :]
    assert float(R.norm(dim=0).max()) / nrm <= 8 * n * EPS
    G = Z.T @ Z - torch.eye(n, dtype=torch.float64, device="cuda")
    assert float(G.abs().max()) <= 8 * n * EPS
    assert st["t_ms"]["reduce"] > 0 and st["t_ms"]["backtransform"] > 0


def test_dense_reduced_t_needs_no_rqi_fallback():
    """Regression (R9b): the extreme eigenvectors of a Householder-reduced T live in
    its first rows; the twist location once clamped the far rows' records and picked r = n - 1
    for them (bisection fallback).  n = 1024: every eigenpair converges in the RQI, and the
    solution keeps the dense parity bar."""
    p = synth.dense_config(1024, 3)
    w, Z, st = run(p.A)
    assert st["rqi_fallbacks"] == 0, st["rqi_fallbacks"]
    _check(p.A, w, Z, oracle_vectors=False)


@pytest.mark.parametrize("lg", [-660, 660])
def test_dense_extreme_scaling(lg):
    """Entries near 2^-660 / 2^660: the reflector norms square them (underflow / overflow) unless
    A is scaled by a power of 2 first (mr3_dsyevr_dd: k_dense_absmax, k_dense_scale; w scaled
    back).  Compared with the same problem at its natural scale: eigenvalues equal up to the
    exact factor, eigenvectors the same bits (found by tools/stress_dense.py)."""
    p = synth.dense_from(synth.random_uniform(150, 8), 8)
    w0, Z0, _ = run(p.A.copy())
    A = np.ldexp(p.A, lg)
    w, Z, st = run(A.copy())
    _check(p.A, np.ldexp(w, -lg), Z, oracle_vectors=False)
    # index subset and a value range given at the scaled magnitude
    w2, Z2, _ = run(A.copy(), range="I", il=10, iu=40)
    np.testing.assert_allclose(np.ldexp(w2, -lg), w0[9:40], rtol=0,
                               atol=8 * 150 * EPS * dense.dense_norm1(p.A))
    vl, vu = 0.5 * (w0[19] + w0[20]), 0.5 * (w0[59] + w0[60])
    w3, Z3, _ = run(A.copy(), range="V", vl=float(np.ldexp(vl, lg)), vu=float(np.ldexp(vu, lg)))
    assert w3.shape[0] == 40 and Z3.shape == (150, 40)
