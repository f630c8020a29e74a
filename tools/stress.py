#!/usr/bin/env python3
"""Robustness sweep (GPU): matrix families in the style of LAPACK's tridiagonal testers that the
BASELINE configs do not cover -- orthogonal-polynomial Jacobi matrices, graded and tightly clustered
spectra, single and glued Wilkinson matrices, zero diagonals, splits, repeated eigenvalues,
extreme scalings, tiny orders -- through mr3_dstemr_dd (all pairs) and mr3_sstemr_d.  Checked
with numpy/LAPACK in binary64 (this is a tool, not a parity test: no oracle):
  res  = max_j ||T z_j - w_j z_j|| / (||T||_1 n eps)
  orth = max |Z^T Z - I| / (n eps)
  eig  = max |w - w_lapack| / (||T||_1 n eps)
usage: python tools/stress.py [bound]   (prints one line per case, FAIL where a figure > bound)
"""
import sys

import numpy as np
import torch
from scipy.linalg import eigh_tridiagonal

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402

BOUND = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
rng = np.random.default_rng(1304)


def wilk(m):
    h = (m - 1) // 2
    return np.abs(np.arange(-h, h + 1)).astype(float), np.ones(m - 1)


def glued(copies, m, glue):
    d0, e0 = wilk(m)
    d = np.tile(d0, copies)
    e = np.concatenate([np.concatenate([e0, [glue]]) for _ in range(copies)])[:-1]
    return d, e


def cases():
    for n in (1, 2, 3, 5, 31, 33, 257, 1025):
        yield f"1-2-1 n={n}", np.full(n, 2.0), np.full(max(n - 1, 0), 1.0)
    for n in (200, 1500):
        i = np.arange(1, n)
        yield f"hermite n={n}", np.zeros(n), np.sqrt(i / 2.0)
        yield f"laguerre n={n}", 2.0 * np.arange(n) + 1.0, i.astype(float)
        yield f"chebyshev n={n}", np.zeros(n), np.concatenate([[np.sqrt(0.5)], np.full(n - 2, 0.5)])
        yield f"clement n={n}", np.zeros(n), np.sqrt(i * (n - i).astype(float))
    for n in (300, 1200):
        k = np.arange(n)
        yield f"graded-down 2^-k/4 n={n}", 2.0 ** (-k / 4.0), 2.0 ** (-(k[:-1] + 0.5) / 4.0) * 0.3
        yield f"graded-up n={n}", 2.0 ** ((k - n) / 4.0), 2.0 ** ((k[:-1] - n + 0.5) / 4.0) * 0.3
        yield f"graded 10^-k/20 strong n={n}", 10.0 ** (-k / 20.0), 10.0 ** (-k[:-1] / 20.0)
    for n in (400, 1600):
        d = 1.0 + 1e-10 * rng.standard_normal(n)
        yield f"near-identity e=1e-8 n={n}", d, np.full(n - 1, 1e-8)
        yield f"near-identity e=1e-14 n={n}", d, 1e-14 * rng.random(n - 1)
        yield f"constant d, e=0 n={n}", np.full(n, 3.0), np.zeros(n - 1)
        yield f"log-uniform e n={n}", rng.standard_normal(n), 10.0 ** rng.uniform(-12, 0, n - 1)
        yield f"zero diag random e n={n}", np.zeros(n), rng.random(n - 1) + 0.01
        e = rng.random(n - 1)
        e[rng.integers(0, n - 1, 7)] = 0.0
        yield f"7 exact splits n={n}", rng.standard_normal(n), e
        lam = np.concatenate([np.full(n // 2, 1.0), np.linspace(2, 3, n - n // 2)])
        yield f"half-cluster diag + tiny e n={n}", lam + 1e-13 * rng.standard_normal(n), np.full(n - 1, 1e-9)
    yield "wilkinson W101", *wilk(101)
    yield "wilkinson W401", *wilk(401)
    for glue in (1e-4, 1e-7, 1e-10, 1e-13):
        yield f"glued W21x50 glue={glue:g}", *glued(50, 21, glue)
    yield "glued W41x30 glue=1e-8", *glued(30, 41, 1e-8)
    for sc in (1e150, 1e-150, 1e300, 1e-290):
        d = rng.standard_normal(500)
        e = rng.standard_normal(499)
        yield f"random normal x{sc:g} n=500", d * sc, e * sc
    for n in (1000, 3000):
        yield f"random normal n={n}", rng.standard_normal(n), rng.standard_normal(n - 1)
        yield f"random uniform(0,1) n={n}", rng.random(n), rng.random(n - 1)


def check(name, d, e, io):
    n = d.size
    dt = torch.float64 if io == "f64" else torch.float32
    npdt = np.float64 if io == "f64" else np.float32
    d = d.astype(npdt)
    e = e.astype(npdt)
    if not (np.all(np.isfinite(d)) and np.all(np.isfinite(e))):
        return None
    fn = mr3.mr3_dstemr_dd if io == "f64" else mr3.mr3_sstemr_d
    try:
        w, Z, st = fn(torch.from_numpy(d).cuda().to(dt), torch.from_numpy(e).cuda().to(dt), "V", "A")
        torch.cuda.synchronize()
    except Exception as ex:  # noqa: BLE001
        return f"EXC {type(ex).__name__}: {ex}"
    w = w.cpu().numpy().astype(np.float64)
    Z = Z.cpu().numpy().astype(np.float64)
    d64, e64 = d.astype(np.float64), e.astype(np.float64)
    eps = 2.0 ** -53 if io == "f64" else 2.0 ** -24
    a = np.abs(d64)
    if n > 1:
        a[:-1] += np.abs(e64)
        a[1:] += np.abs(e64)
    nrm = max(a.max(), 1e-300)
    TZ = d64[:, None] * Z
    if n > 1:
        TZ[:-1] += e64[:, None] * Z[1:]
        TZ[1:] += e64[:, None] * Z[:-1]
    res = np.max(np.linalg.norm(TZ / nrm - (w / nrm)[None, :] * Z, axis=0)) / (n * eps)
    orth = np.max(np.abs(Z.T @ Z - np.eye(n))) / (n * eps)
    wl = eigh_tridiagonal(d64 / nrm, e64 / nrm, eigvals_only=True) if n > 1 else d64 / nrm
    eig = np.max(np.abs(np.sort(w) / nrm - wl)) / (n * eps)
    asc = bool(np.all(np.diff(w) >= 0))
    bad = (not np.isfinite(res + orth + eig)) or max(res, orth, eig) > BOUND or not asc
    return (f"{'FAIL' if bad else 'ok  '} res {res:8.3f} orth {orth:8.3f} eig {eig:8.3f} "
            f"asc {int(asc)} dmax {st['d_max']} clus {st['n_clusters']} rf {st['robustness_failures']} "
            f"fb {st['rqi_fallbacks']} blocks {st['n_blocks']}")


nfail = 0
for name, d, e in cases():
    for io in ("f64", "f32"):
        if io == "f32" and ("x1e" in name or "1e-13" in name or "1e-14" in name):
            continue
        r = check(name, np.asarray(d, float), np.asarray(e, float), io)
        if r is None:
            continue
        if r.startswith("FAIL") or r.startswith("EXC"):
            nfail += 1
        print(f"{io} {name:42s} {r}", flush=True)
print("failures:", nfail)
