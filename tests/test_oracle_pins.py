"""Pins for the binary128 oracle (oracle/), independent of the oracle itself.

Every check below ties the oracle to something it does not compute itself:
closed forms evaluated with mpmath at 50 digits, brute-force Jacobi, numpy's
LAPACK, invariants (trace, Frobenius norm, Sturm monotonicity), Weyl bounds and
Golub-Welsch quadrature weights. A dropped term, a wrong sign or index, or a
transposed operand anywhere in the oracle's Sturm recurrence, bisection, LU
solve or verifier fails at least one of them.
"""
import mpmath as mp
import numpy as np
import pytest

import oracle
import synth

mp.mp.dps = 50


def dd_split(x):
    """mpf -> (hi, lo) float64 pair with hi + lo = x to ~2^-106 relative."""
    hi = float(x)
    lo = float(x - mp.mpf(hi))
    return hi, lo


def as_mpf(hi, lo):
    return mp.mpf(float(hi)) + mp.mpf(float(lo))


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 129])
def test_121_eigenvalues_closed_form(n):
    """1-2-1: lambda_k = 2 - 2 cos(k pi/(n+1)) (BJ:5)."""
    p = synth.one_two_one(n)
    lh, ll = oracle.eigvals(p.d, p.e)
    for k in range(1, n + 1):
        ex = 2 - 2 * mp.cos(k * mp.pi / (n + 1))
        assert abs(as_mpf(lh[k - 1], ll[k - 1]) - ex) < mp.mpf("1e-30")


@pytest.mark.parametrize("n", [2, 5, 40])
def test_121_eigenvectors_closed_form(n):
    """z_j = (-1)^(j+1) sqrt(2/(n+1)) sin(j k pi/(n+1)), j*k reduced mod 2(n+1) (c18)."""
    p = synth.one_two_one(n)
    lh, ll, zh, zl = oracle.solve(p.d, p.e)
    for k in range(1, n + 1):
        ex = [(-1) ** (j + 1) * mp.sqrt(mp.mpf(2) / (n + 1)) *
              mp.sin(((j * k) % (2 * (n + 1))) * mp.pi / (n + 1)) for j in range(1, n + 1)]
        got = [as_mpf(zh[j, k - 1], zl[j, k - 1]) for j in range(n)]
        dot = mp.fsum(a * b for a, b in zip(ex, got))
        sgn = 1 if dot > 0 else -1
        err = max(abs(g - sgn * x) for g, x in zip(got, ex))
        assert err < mp.mpf("1e-28"), (k, err)


@pytest.mark.parametrize("n", [5, 6, 9, 30])
def test_clement_spectrum(n):
    """Clement/Kac: spectrum {-(n-1), -(n-3), ..., n-1}."""
    eh, el = zip(*[dd_split(mp.sqrt(k * (n - k))) for k in range(1, n)])
    d = np.zeros(n)
    lh, ll = oracle.eigvals(d, np.array(eh), d_lo=np.zeros(n), e_lo=np.array(el))
    for k in range(n):
        ex = -(n - 1) + 2 * k
        assert abs(as_mpf(lh[k], ll[k]) - ex) < mp.mpf("1e-28") * n


def test_clement_small_examples_fp64_inputs():
    """S:237 example: Kac n=5 -> {-4,-2,0,2,4} with fp64-rounded e (Weyl slack)."""
    p = synth.clement(5)
    lh, ll = oracle.eigvals(p.d, p.e)
    assert np.allclose(lh, [-4, -2, 0, 2, 4], atol=1e-14)


@pytest.mark.parametrize("n", [4, 20, 61])
def test_legendre_nodes_and_weights(n):
    """Jacobi matrix of Legendre polynomials: eigenvalues = Gauss nodes (roots of P_n),
    first eigenvector component^2 = w_k / 2 (Golub-Welsch).  Exact (dd) inputs."""
    eh, el = zip(*[dd_split(mp.mpf(k) / mp.sqrt(4 * k * k - 1)) for k in range(1, n)])
    d = np.zeros(n)
    lh, ll = oracle.eigvals(d, np.array(eh), d_lo=np.zeros(n), e_lo=np.array(el))
    x64, w64 = np.polynomial.legendre.leggauss(n)
    zh, zl = oracle.eigvecs(d, np.array(eh), lh, ll, d_lo=np.zeros(n), e_lo=np.array(el))
    for k in range(n):
        root = mp.findroot(lambda x: mp.legendre(n, x), x64[k])
        assert abs(as_mpf(lh[k], ll[k]) - root) < mp.mpf("1e-28")
        # Gauss weight from the derivative: w = 2 / ((1-x^2) P_n'(x)^2)
        dp = mp.diff(lambda x: mp.legendre(n, x), root)
        wk = 2 / ((1 - root ** 2) * dp ** 2)
        z1 = as_mpf(zh[0, k], zl[0, k])
        assert abs(z1 ** 2 - wk / 2) < mp.mpf("1e-26")
        assert abs(float(wk) - w64[k]) < 1e-13


# ---------------------------------------------------------------- brute force

@pytest.mark.parametrize("kind", ["uniform", "graded", "integer"])
@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("n", [1, 2, 3, 6, 12])
def test_vs_jacobi_bruteforce(n, seed, kind):
    p = synth.random_small(n, seed, kind)
    lh, ll = oracle.eigvals(p.d, p.e)
    jh, jl, vh, vl = oracle.jacobi(p.d, p.e)
    nrm = oracle.norm1(p.d, p.e)
    for k in range(n):
        assert abs(as_mpf(lh[k], ll[k]) - as_mpf(jh[k], jl[k])) <= mp.mpf("1e-30") * nrm
    # eigenvectors where eigenvalues are distinct enough to define them
    zh, zl = oracle.eigvecs(p.d, p.e, lh, ll)
    lam = lh + ll
    for k in range(n):
        gap = min([abs(lam[k] - lam[j]) for j in range(n) if j != k] or [np.inf])
        if gap < 1e-6 * max(nrm, 1e-300):
            continue
        s = oracle.sin_angles(zh[:, k:k + 1] + zl[:, k:k + 1], vh[:, k:k + 1], vl[:, k:k + 1])
        assert s[0] < 1e-15


@pytest.mark.parametrize("seed", range(3))
def test_vs_numpy_eigh(seed):
    p = synth.random_small(200, seed)
    lh, ll = oracle.eigvals(p.d, p.e)
    T = np.diag(p.d) + np.diag(p.e, 1) + np.diag(p.e, -1)
    ref = np.linalg.eigvalsh(T)
    assert np.max(np.abs(lh - ref)) < 1e-13 * oracle.norm1(p.d, p.e)


def test_split_matrix_union_of_blocks():
    """e_i = 0 splits T: spectrum = union of the block spectra (Jacobi per block)."""
    p = synth.split_matrix(12, 3, split_at=(4, 8))
    lh, ll = oracle.eigvals(p.d, p.e)
    blocks = [(0, 5), (5, 9), (9, 12)]
    ev = []
    for a, b in blocks:
        jh, jl, _, _ = oracle.jacobi(p.d[a:b], p.e[a:b - 1])
        ev += [as_mpf(h, l) for h, l in zip(jh, jl)]
    ev.sort()
    for k in range(12):
        assert abs(as_mpf(lh[k], ll[k]) - ev[k]) < mp.mpf("1e-30")


# ---------------------------------------------------------------- invariants

@pytest.mark.parametrize("make", [lambda: synth.random_uniform(300, 1),
                                  lambda: synth.glued_wilkinson(6, 21),
                                  lambda: synth.random_normal_f32(400, 2, 1, 400)])
def test_trace_and_frobenius(make):
    """sum lambda = sum d ; sum lambda^2 = sum d^2 + 2 sum e^2 (exact identities)."""
    p = make()
    lh, ll = oracle.eigvals(p.d, p.e)
    lam = [as_mpf(h, l) for h, l in zip(lh, ll)]
    tr = mp.fsum(mp.mpf(float(x)) for x in p.d)
    fr = mp.fsum(mp.mpf(float(x)) ** 2 for x in p.d) + 2 * mp.fsum(mp.mpf(float(x)) ** 2 for x in p.e)
    nrm = oracle.norm1(p.d, p.e)
    assert abs(mp.fsum(lam) - tr) < mp.mpf("1e-28") * nrm * p.n
    assert abs(mp.fsum(l * l for l in lam) - fr) < mp.mpf("1e-28") * nrm ** 2 * p.n


@pytest.mark.parametrize("make", [lambda: synth.random_uniform(150, 2),
                                  lambda: synth.one_two_one(100),
                                  lambda: synth.glued_wilkinson(3, 21)])
def test_sturm_monotone_and_endpoints(make):
    p = make()
    gl, gu = oracle.gershgorin(p.d, p.e)
    xs = np.linspace(gl, gu, 997)
    c = oracle.sturm_counts(p.d, p.e, xs)
    assert c[0] == 0 and c[-1] == p.n
    assert np.all(np.diff(c) >= 0)
    # counts agree with the oracle's own eigenvalues (and numpy's)
    lam = np.linalg.eigvalsh(np.diag(p.d) + np.diag(p.e, 1) + np.diag(p.e, -1))
    for x, cx in zip(xs[::37], c[::37]):
        if np.min(np.abs(lam - x)) > 1e-10:
            assert cx == np.sum(lam < x)


def test_glued_wilkinson_weyl():
    """Sorted eig(T) within ||glue||_2 = 2^-26 of sorted {eig(W21)} x copies (Weyl)."""
    copies = 5
    p = synth.glued_wilkinson(copies, 21)
    db, eb = synth.wilkinson_block(21)
    jh, jl, _, _ = oracle.jacobi(db, eb)
    ref = np.sort(np.repeat(jh + jl, copies))
    lh, ll = oracle.eigvals(p.d, p.e)
    assert np.max(np.abs((lh + ll) - ref)) <= 2.0 ** -26 * (1 + 1e-12)


def test_subset_indices_match_full():
    p = synth.random_uniform(120, 5)
    fh, fl = oracle.eigvals(p.d, p.e)
    idx = np.array([1, 7, 60, 119, 120])
    sh, sl = oracle.eigvals(p.d, p.e, idx)
    assert np.array_equal(sh, fh[idx - 1]) and np.array_equal(sl, fl[idx - 1])


def test_oracle_vectors_quad_residual_and_orthogonality():
    """The oracle's own (hi+lo) vectors: residual and orthogonality at binary128 level,
    evaluated independently in mpmath."""
    p = synth.random_small(10, 7)
    lh, ll, zh, zl = oracle.solve(p.d, p.e)
    n = p.n
    z = [[as_mpf(zh[i, k], zl[i, k]) for i in range(n)] for k in range(n)]
    for k in range(n):
        lam = as_mpf(lh[k], ll[k])
        for i in range(n):
            r = (mp.mpf(p.d[i]) - lam) * z[k][i]
            if i > 0:
                r += mp.mpf(p.e[i - 1]) * z[k][i - 1]
            if i < n - 1:
                r += mp.mpf(p.e[i]) * z[k][i + 1]
            assert abs(r) < mp.mpf("1e-29")
        for j in range(k + 1, n):
            assert abs(mp.fsum(a * b for a, b in zip(z[k], z[j]))) < mp.mpf("1e-29")


def test_degenerate_group_reorthogonalised():
    """Glued Wilkinson copies give near-degenerate groups: group reorthogonalisation
    must keep the oracle vectors orthonormal to ~1e-30."""
    p = synth.glued_wilkinson(4, 21)
    lh, ll, zh, zl = oracle.solve(p.d, p.e, group_tol_rel=1e-3)
    o, dd = oracle.orthogonality(zh + zl)
    assert o < 1e-15 and dd < 1e-15
    r1, r2, _ = oracle.residuals(p.d, p.e, lh, zh)
    assert r2.max() < 1e-16


# ---------------------------------------------------------------- verifier

def test_residual_verifier_hand_example():
    """T=[[2,1],[1,2]], w=1, z=(1,-1+t)/||.||: r = (t, 2t - ... ) evaluated in mpmath."""
    t = 2.0 ** -20
    z = np.array([1.0, -1.0 + t])
    z = z / np.linalg.norm(z)
    d, e = np.array([2.0, 2.0]), np.array([1.0])
    r1, r2, zn = oracle.residuals(d, e, np.array([1.0]), z[:, None])
    zm = [mp.mpf(float(x)) for x in z]
    r = [mp.mpf(1) * zm[0] + zm[1], zm[0] + zm[1]]
    assert abs(r1[0] - float((abs(r[0]) + abs(r[1])) / 3)) < 1e-20
    assert abs(r2[0] - float(mp.sqrt(r[0] ** 2 + r[1] ** 2) / 3)) < 1e-20


def test_orthogonality_verifier_known_dots():
    rng = np.random.default_rng(0)
    n = 50
    a = rng.standard_normal(n)
    a /= np.linalg.norm(a)
    b = rng.standard_normal(n)
    b -= (a @ b) * a
    b /= np.linalg.norm(b)
    c = np.cos(1e-3) * a + np.sin(1e-3) * b
    Z = np.stack([a, b, c], 1)
    o, dd = oracle.orthogonality(Z)
    zm = [[mp.mpf(float(x)) for x in Z[:, j]] for j in range(3)]
    ex = max(abs(mp.fsum(x * y for x, y in zip(zm[i], zm[j]))) for i in range(3) for j in range(3)
             if i != j)
    assert abs(o - float(ex)) < 1e-28


def test_sin_angle_verifier():
    th = 1e-9
    zo = np.zeros((3, 1))
    zo[0, 0] = 1.0
    zhat = np.array([[np.cos(th)], [np.sin(th)], [0.0]])
    s = oracle.sin_angles(zhat, zo, np.zeros_like(zo))
    assert abs(s[0] - np.sin(th)) < 1e-24
    s2 = oracle.sin_angles(-zhat, zo, np.zeros_like(zo))
    assert abs(s2[0] - np.sin(th)) < 1e-24
    sub = oracle.subspace_sin(zhat, zo, np.zeros_like(zo))
    assert abs(sub - np.sin(th)) < 1e-20


def test_norm1_and_gershgorin_rows_differ():
    """||T||_1 (Eq. (1.1)) and the Gershgorin bounds on matrices whose row sums
    differ, with the maximum in the first, a middle and the last row: against the dense
    matrix summed in mpmath (a plain definition, no tridiagonal shortcut)."""
    cases = [(np.array([9.0, 1.0, -2.0, 0.5]), np.array([-3.0, 0.25, 1.0])),      # first row
             (np.array([0.5, -1.0, 7.0, 0.25, 1.0]), np.array([0.5, -2.0, 3.0, 0.125])),  # middle
             (np.array([1.0, 2.0, -0.5, -6.0]), np.array([0.5, 0.75, -4.0]))]     # last row
    rng = np.random.default_rng(3)
    cases.append((rng.standard_normal(37) * np.exp2(rng.integers(-8, 9, 37)),
                   rng.standard_normal(36) * np.exp2(rng.integers(-8, 9, 36))))
    for d, e in cases:
        n = d.size
        T = [[mp.mpf(0)] * n for _ in range(n)]
        for i in range(n):
            T[i][i] = mp.mpf(float(d[i]))
        for i in range(n - 1):
            T[i][i + 1] = T[i + 1][i] = mp.mpf(float(e[i]))
        cols = [mp.fsum(abs(T[i][j]) for i in range(n)) for j in range(n)]
        assert abs(oracle.norm1(d, e) - float(max(cols))) <= 1e-30 * float(max(cols))
        radii = [mp.fsum(abs(T[i][j]) for j in range(n) if j != i) for i in range(n)]
        gl = min(T[i][i] - radii[i] for i in range(n))
        gu = max(T[i][i] + radii[i] for i in range(n))
        ogl, ogu = oracle.gershgorin(d, e)
        assert abs(ogl - float(gl)) <= 1e-28 * float(max(cols))
        assert abs(ogu - float(gu)) <= 1e-28 * float(max(cols))


@pytest.mark.parametrize("g", [2, 3, 5])
def test_subspace_sin_constructed_rotation(g):
    """Group subspace angles (oracle_subspace_residual) for g >= 2: the
    computed span Zhat is built with known principal angles theta_j to span(Z_G) and then
    mixed by a g x g rotation, so no column of Zhat lines up with a column of Z_G.  The
    largest principal angle's sine must come out as sin(max theta) and as the largest
    singular value of (I - Z_G Z_G^T) Zhat from an mpmath SVD: an index slip or a transposed
    operand in the g x g Gram matrix fails it."""
    rng = np.random.default_rng(100 + g)
    n = 40
    Q, _ = np.linalg.qr(rng.standard_normal((n, 2 * g)))
    U, V = Q[:, :g], Q[:, g:]                 # span(Z_G) and an orthogonal complement part
    A, _ = np.linalg.qr(rng.standard_normal((g, g)))  # basis of span(Z_G) given to the oracle
    B, _ = np.linalg.qr(rng.standard_normal((g, g)))  # rotation mixing the columns of Zhat
    theta = np.array([10.0 ** (-3 - 2 * j) for j in range(g)])
    rng.shuffle(theta)
    Zo = U @ A
    Zhat = (U * np.cos(theta) + V * np.sin(theta)) @ B
    s = oracle.subspace_sin(Zhat, Zo, np.zeros_like(Zo))
    assert abs(s - np.sin(theta.max())) <= 1e-14 * np.sin(theta.max()) + 1e-16
    # mpmath: singular values of the projection residual
    Zm = mp.matrix(Zhat.tolist())
    Om = mp.matrix(Zo.tolist())
    Pm = Zm - Om * (Om.T * Zm)
    sv = mp.svd_r(Pm, compute_uv=False)
    assert abs(s - float(max(sv))) <= 1e-14 * float(max(sv)) + 1e-18
