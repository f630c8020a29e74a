"""The binary128 oracle against the worked examples printed in SPEC.md (tests/golden/,
each file cites its source lines).  CPU only."""
import os

import mpmath
import numpy as np
import pytest

import oracle

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
mpmath.mp.prec = 240
EPS_Q = mpmath.mpf(2) ** -113  # binary128 unit roundoff: the oracle's bisection stops at ~2 eps_q


def _read(name):
    rows = {}
    with open(os.path.join(G, name)) as f:
        for ln in f:
            ln = ln.strip()
            if not ln or ln.startswith("#"):
                continue
            key, *vals = ln.split()
            rows.setdefault(key, []).append([float(v) for v in vals])
    return rows


def _q(hi, lo):
    return mpmath.mpf(float(hi)) + mpmath.mpf(float(lo))


def test_golden_kac5():
    g = _read("kac5.txt")
    n = int(g["n"][0][0])
    d = np.array(g["d"][0])
    k = np.array(g["e_sqrt_k(n-k)"][0])
    e = np.sqrt(k)  # fp64-rounded inputs
    lam = np.array(g["eigenvalues"][0])
    lh, ll = oracle.eigvals(d, e)
    slack = 2 * max(abs(float(mpmath.sqrt(mpmath.mpf(int(x)))) - mpmath.sqrt(mpmath.mpf(int(x))))
                    for x in k)
    assert n == d.size
    for i in range(n):
        assert abs(_q(lh[i], ll[i]) - lam[i]) <= slack + 1e-30


def test_golden_sturm_examples():
    with open(os.path.join(G, "sturm_examples.txt")) as f:
        for ln in f:
            if ln.startswith("#") or not ln.strip():
                continue
            name, d, e, x, c = [s.strip() for s in ln.split("|")]
            d = np.array(d.split(), dtype=float)
            e = np.array(e.split(), dtype=float)
            x = float(x)
            # an x that is itself an eigenvalue (one21_n3 at 2) meets a zero pivot, which
            # reading c14 (R6) counts as negative: count(x) = #{lambda <= x} there,
            # so the strict count of the example is checked just below x
            below = oracle.sturm_counts(d, e, np.array([np.nextafter(x, -np.inf)]))
            at = oracle.sturm_counts(d, e, np.array([x]))
            assert int(below[0]) == int(c), name
            assert int(at[0]) in (int(c), int(c) + 1), name


def test_golden_2x2_pairs():
    g = _read("pairs_2x2.txt")
    d, e = np.array(g["d"][0]), np.array(g["e"][0])
    lh, ll, zh, zl = oracle.solve(d, e)
    for j, (lam, z1, z2) in enumerate(g["pair"]):
        assert abs(_q(lh[j], ll[j]) - lam) <= 4 * EPS_Q * abs(lam)
        v = np.array([z1, z2])
        v = [mpmath.mpf(x) / mpmath.sqrt(2) for x in v]
        z = [_q(zh[i, j], zl[i, j]) for i in range(2)]
        s = 1 if z[0] * v[0] > 0 else -1
        assert max(abs(z[i] - s * v[i]) for i in range(2)) < 1e-30


def test_golden_diag123():
    g = _read("diag123.txt")
    d, e = np.array(g["d"][0]), np.array(g["e"][0])
    lh, ll, zh, zl = oracle.solve(d, e)
    for i, lam in enumerate(g["eigenvalues"][0]):
        assert abs(_q(lh[i], ll[i]) - lam) <= 4 * EPS_Q * abs(lam)
    for j in range(3):
        for i in range(3):
            assert abs(abs(_q(zh[i, j], zl[i, j])) - (1 if i == j else 0)) < 1e-30


def test_golden_121_n3():
    g = _read("one21_n3.txt")
    d, e = np.array(g["d"][0]), np.array(g["e"][0])
    lh, ll, zh, zl = oracle.solve(d, e)
    for i, c in enumerate(g["eigenvalues_2pm_sqrt2"][0]):
        assert abs(_q(lh[i], ll[i]) - (2 + c * mpmath.sqrt(2))) < 1e-30
    v = [mpmath.mpf(x) / mpmath.sqrt(2) for x in g["vector_of_2"][0]]
    z = [_q(zh[i, 1], zl[i, 1]) for i in range(3)]
    s = 1 if z[0] * v[0] > 0 else -1
    assert max(abs(z[i] - s * v[i]) for i in range(3)) < 1e-30


@pytest.mark.parametrize("name", sorted(os.listdir(G)))
def test_golden_files_cite_a_source(name):
    with open(os.path.join(G, name)) as f:
        head = f.read()
    assert "SPEC.md S:" in head or "PAPER.md L" in head, name
