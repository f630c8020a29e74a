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

BOUND = float(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 20.0
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


def check_subset(name, d, e, io, kind):
    """range 'I' / 'V' subsets against LAPACK's selection (binary64 reference values)."""
    n = d.size
    if n < 30:
        return None
    dt = torch.float64 if io == "f64" else torch.float32
    npdt = np.float64 if io == "f64" else np.float32
    d = d.astype(npdt)
    e = e.astype(npdt)
    if not (np.all(np.isfinite(d)) and np.all(np.isfinite(e))):
        return None
    d64, e64 = d.astype(np.float64), e.astype(np.float64)
    eps = 2.0 ** -53 if io == "f64" else 2.0 ** -24
    a = np.abs(d64)
    a[:-1] += np.abs(e64)
    a[1:] += np.abs(e64)
    nrm = max(a.max(), 1e-300)
    wl = eigh_tridiagonal(d64 / nrm, e64 / nrm, eigvals_only=True) * nrm
    il, iu = n // 3, n // 3 + min(50, n // 4)
    fn = mr3.mr3_dstemr_dd if io == "f64" else mr3.mr3_sstemr_d
    dd_, ee_ = torch.from_numpy(d).cuda().to(dt), torch.from_numpy(e).cuda().to(dt)
    try:
        if kind == "I":
            w, Z, st = fn(dd_, ee_, "V", "I", il, iu)
            ref = wl[il - 1:iu]
        else:
            # (vl, vu] between well separated neighbours where there are any
            gaps = np.diff(wl)
            lo = int(np.argmax(gaps[n // 4:n // 2])) + n // 4
            hi_ = int(np.argmax(gaps[n // 2 + 1:3 * n // 4])) + n // 2 + 1
            vl, vu = 0.5 * (wl[lo] + wl[lo + 1]), 0.5 * (wl[hi_] + wl[hi_ + 1])
            if not (gaps[lo] > 1e3 * n * eps * nrm and gaps[hi_] > 1e3 * n * eps * nrm):
                return None
            w, Z, st = fn(dd_, ee_, "V", "V", 1, 0, float(npdt(vl)), float(npdt(vu)))
            vl, vu = float(npdt(vl)), float(npdt(vu))
            ref = wl[(wl > vl) & (wl <= vu)]
        torch.cuda.synchronize()
    except Exception as ex:  # noqa: BLE001
        return f"EXC {type(ex).__name__}: {ex}"
    w = w.cpu().numpy().astype(np.float64)
    Z = Z.cpu().numpy().astype(np.float64)
    if w.size != ref.size or Z.shape != (n, ref.size):
        return f"FAIL count {w.size} (Z {Z.shape}) vs {ref.size}"
    if w.size == 0:
        return "ok   empty"
    TZ = d64[:, None] * Z
    TZ[:-1] += e64[:, None] * Z[1:]
    TZ[1:] += e64[:, None] * Z[:-1]
    res = np.max(np.linalg.norm(TZ / nrm - (w / nrm)[None, :] * Z, axis=0)) / (n * eps)
    orth = np.max(np.abs(Z.T @ Z - np.eye(w.size))) / (n * eps)
    eig = np.max(np.abs(w - ref)) / nrm / (n * eps)
    asc = bool(np.all(np.diff(w) >= 0))
    bad = (not np.isfinite(res + orth + eig)) or max(res, orth, eig) > BOUND or not asc
    return (f"{'FAIL' if bad else 'ok  '} m {w.size:4d} res {res:8.3f} orth {orth:8.3f} eig {eig:8.3f} "
            f"asc {int(asc)}")


def large_cases():
    n = 20000
    i = np.arange(1, n)
    k = np.arange(n)
    yield f"hermite n={n}", np.zeros(n), np.sqrt(i / 2.0)
    yield f"laguerre n={n}", 2.0 * k + 1.0, i.astype(float)
    yield f"graded-down 2^-k/4 (underflows) n={n}", 2.0 ** (-k / 4.0), 2.0 ** (-(k[:-1] + 0.5) / 4.0) * 0.3
    yield f"graded 10^-k/2000 n={n}", 10.0 ** (-k / 2000.0), 10.0 ** (-k[:-1] / 2000.0) * 0.5
    yield f"random normal n={n}", rng.standard_normal(n), rng.standard_normal(n - 1)
    yield f"zero diag random e n={n}", np.zeros(n), rng.random(n - 1) + 0.01
    yield "glued W21x900 glue=1e-9", *glued(900, 21, 1e-9)
    yield f"wilkinson W{n + 1}", *wilk(n + 1)
    yield f"clement n={n // 2}", np.zeros(n // 2), np.sqrt(np.arange(1, n // 2) * (n // 2 - np.arange(1, n // 2)).astype(float))


def check_large(name, d, e):
    """All pairs at n ~ 20000, checked on the GPU in binary64 torch (residual, Gram matrix) and
    against LAPACK's eigenvalues."""
    n = d.size
    dt_ = torch.from_numpy(d).cuda()
    et_ = torch.from_numpy(e).cuda()
    try:
        w, Z, st = mr3.mr3_dstemr_dd(dt_, et_, "V", "A")
        torch.cuda.synchronize()
    except Exception as ex:  # noqa: BLE001
        return f"EXC {type(ex).__name__}: {ex}"
    eps = 2.0 ** -53
    a = np.abs(d)
    a[:-1] += np.abs(e)
    a[1:] += np.abs(e)
    nrm = max(a.max(), 1e-300)
    TZ = dt_[:, None] * Z
    TZ[:-1] += et_[:, None] * Z[1:]
    TZ[1:] += et_[:, None] * Z[:-1]
    res = float(torch.linalg.vector_norm(TZ / nrm - (w / nrm)[None, :] * Z, dim=0).max()) / (n * eps)
    del TZ
    G = Z.T.contiguous() @ Z.T.contiguous().T
    G.diagonal().sub_(1.0)
    orth = float(G.abs().max()) / (n * eps)
    del G
    wl = eigh_tridiagonal(d / nrm, e / nrm, eigvals_only=True)
    wh = w.cpu().numpy()
    eig = np.max(np.abs(wh / nrm - wl)) / (n * eps)
    asc = bool(np.all(np.diff(wh) >= 0))
    bad = (not np.isfinite(res + orth + eig)) or max(res, orth, eig) > BOUND or not asc
    return (f"{'FAIL' if bad else 'ok  '} res {res:8.4f} orth {orth:8.4f} eig {eig:8.4f} asc {int(asc)} "
            f"dmax {st['d_max']} clus {st['n_clusters']} rf {st['robustness_failures']} "
            f"fb {st['rqi_fallbacks']} blocks {st['n_blocks']} ms {st['t_ms']['total']:.1f}")


nfail = 0
if "--large" in sys.argv:
    for name, d, e in large_cases():
        r = check_large(name, np.asarray(d, float), np.asarray(e, float))
        if r.startswith("FAIL") or r.startswith("EXC"):
            nfail += 1
        print(f"f64 {name:42s} {r}", flush=True)
        torch.cuda.empty_cache()
    print("failures:", nfail)
    sys.exit(0)
if "--subsets" in sys.argv:
    for name, d, e in cases():
        for io in ("f64", "f32"):
            if io == "f32" and ("x1e" in name or "1e-13" in name or "1e-14" in name):
                continue
            for kind in ("I", "V"):
                r = check_subset(name, np.asarray(d, float), np.asarray(e, float), io, kind)
                if r is None:
                    continue
                if r.startswith("FAIL") or r.startswith("EXC"):
                    nfail += 1
                print(f"{io} {kind} {name:42s} {r}", flush=True)
    print("failures:", nfail)
    sys.exit(0)
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
