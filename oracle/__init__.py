"""Python binding of the binary128 oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. The product path
(paper_1304_1864_b200/) never imports it and shares no code with it.

What the oracle computes (see oracle.c header for the PAPER.md citations):
eigenvalues of T by Sturm bisection on T itself in __float128, eigenvectors by
inverse iteration with group reorthogonalisation in __float128, and the
Eq. (1.1) metrics R and O. Results come back as (hi, lo) float64 pairs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, libquadmath, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC,
                               "-lquadmath", "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, dbl, u64, cint = ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int
        lib.oracle_norm1.argtypes = [i64, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.oracle_gershgorin.argtypes = [i64, _dp, _dp, _dp, _dp, _dp]
        lib.oracle_sturm_counts.argtypes = [i64, _dp, _dp, _dp, _dp, i64, _dp, _dp, _ip]
        lib.oracle_eigvals.argtypes = [i64, _dp, _dp, _dp, _dp, i64, _ip, _dp, _dp]
        lib.oracle_eigvals.restype = cint
        lib.oracle_eigvecs.argtypes = [i64, _dp, _dp, _dp, _dp, i64, _dp, _dp, dbl, u64, cint,
                                       _dp, _dp]
        lib.oracle_eigvecs.restype = cint
        lib.oracle_residuals.argtypes = [i64, _dp, _dp, i64, _dp, _dp, i64, _dp, _dp, _dp]
        lib.oracle_orthogonality.argtypes = [i64, i64, _dp, i64, _dp]
        lib.oracle_orthogonality.restype = dbl
        lib.oracle_sin_angles.argtypes = [i64, i64, _dp, i64, _dp, _dp, _dp]
        lib.oracle_subspace_residual.argtypes = [i64, i64, _dp, i64, _dp, _dp, _dp]
        lib.oracle_jacobi.argtypes = [i64, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.oracle_jacobi.restype = cint
        lib.oracle_num_threads.restype = cint
        _lib = lib
    return _lib


def _f64(a):
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _pe(e):
    # e may be empty (n == 1): pass a valid pointer anyway
    return _p(e if e.size else np.zeros(1))


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def norm1(d, e, d_lo=None, e_lo=None) -> float:
    lib = _load()
    d, e, d_lo, e_lo = _f64(d), _f64(e), _f64(d_lo), _f64(e_lo)
    hi, lo = ctypes.c_double(), ctypes.c_double()
    lib.oracle_norm1(d.size, _p(d), _p(d_lo), _pe(e), _p(e_lo), ctypes.byref(hi), ctypes.byref(lo))
    return hi.value + lo.value


def gershgorin(d, e):
    lib = _load()
    d, e = _f64(d), _f64(e)
    out = np.zeros(4)
    lib.oracle_gershgorin(d.size, _p(d), None, _pe(e), None, _p(out))
    return out[0] + out[1], out[2] + out[3]


def sturm_counts(d, e, x_hi, x_lo=None, d_lo=None, e_lo=None) -> np.ndarray:
    lib = _load()
    d, e, d_lo, e_lo = _f64(d), _f64(e), _f64(d_lo), _f64(e_lo)
    x_hi, x_lo = _f64(np.atleast_1d(x_hi)), _f64(x_lo)
    out = np.zeros(x_hi.size, dtype=np.int64)
    lib.oracle_sturm_counts(d.size, _p(d), _p(d_lo), _pe(e), _p(e_lo), x_hi.size, _p(x_hi),
                            _p(x_lo), out.ctypes.data_as(_ip))
    return out


def eigvals(d, e, idx=None, d_lo=None, e_lo=None):
    """Eigenvalues with 1-based indices idx (default all) as (hi, lo) float64 arrays."""
    lib = _load()
    d, e, d_lo, e_lo = _f64(d), _f64(e), _f64(d_lo), _f64(e_lo)
    n = d.size
    idx = np.arange(1, n + 1, dtype=np.int64) if idx is None else \
        np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    hi, lo = np.zeros(idx.size), np.zeros(idx.size)
    if idx.size:
        rc = lib.oracle_eigvals(n, _p(d), _p(d_lo), _pe(e), _p(e_lo), idx.size,
                                idx.ctypes.data_as(_ip), _p(hi), _p(lo))
        assert rc == 0
    return hi, lo


def eigvecs(d, e, lam_hi, lam_lo, group_tol: float | None = None, group_tol_rel: float = 1e-3,
            seed: int = 12345, iters: int = 3, d_lo=None, e_lo=None):
    """Unit eigenvectors (n x m, column-major hi/lo pairs) by inverse iteration.

    Groups: consecutive eigenvalues closer than group_tol (absolute; default
    group_tol_rel * ||T||_1) are reorthogonalised against each other (CGS2)."""
    lib = _load()
    d, e, d_lo, e_lo = _f64(d), _f64(e), _f64(d_lo), _f64(e_lo)
    lam_hi, lam_lo = _f64(lam_hi), _f64(lam_lo)
    n, m = d.size, lam_hi.size
    if group_tol is None:
        group_tol = group_tol_rel * norm1(d, e, d_lo, e_lo)
    zhi = np.zeros((m, n))  # row j = column j of Z (column-major storage)
    zlo = np.zeros((m, n))
    if m:
        rc = lib.oracle_eigvecs(n, _p(d), _p(d_lo), _pe(e), _p(e_lo), m, _p(lam_hi), _p(lam_lo),
                                float(group_tol), seed & (2**64 - 1), iters, _p(zhi), _p(zlo))
        assert rc == 0
    return zhi.T, zlo.T  # (n, m) views of column-major storage


def _colmajor(Z):
    Z = np.asarray(Z, dtype=np.float64)
    if Z.ndim == 1:
        Z = Z[:, None]
    return np.asfortranarray(Z)


def residuals(d, e, w, Z):
    """Per column: R1 = ||T z - w z||_1/||T||_1 (Eq. 1.1), R2 (2-norm), ||z||-1; quad."""
    lib = _load()
    d, e = _f64(d), _f64(e)
    Z = _colmajor(Z)
    w = _f64(w)
    n, m = Z.shape
    r1, r2, zn = np.zeros(m), np.zeros(m), np.zeros(m)
    if m:
        lib.oracle_residuals(n, _p(d), _pe(e), m, _p(w), Z.ctypes.data_as(_dp), n, _p(r1), _p(r2),
                             _p(zn))
    return r1, r2, zn


def orthogonality(Z):
    """O = max_{i!=j} |z_i^T z_j| (Eq. 1.1) with compensated dots; also max|z_i^T z_i - 1|."""
    lib = _load()
    Z = _colmajor(Z)
    n, m = Z.shape
    dd = ctypes.c_double()
    o = lib.oracle_orthogonality(n, m, Z.ctypes.data_as(_dp), n, ctypes.byref(dd))
    return o, dd.value


def sin_angles(Zhat, Zo_hi, Zo_lo):
    lib = _load()
    Zhat = _colmajor(Zhat)
    n, m = Zhat.shape
    zh, zl = _colmajor(Zo_hi), _colmajor(Zo_lo)
    out = np.zeros(m)
    if m:
        lib.oracle_sin_angles(n, m, Zhat.ctypes.data_as(_dp), n, zh.ctypes.data_as(_dp),
                              zl.ctypes.data_as(_dp), _p(out))
    return out


def subspace_sin(Zhat_G, Zo_hi_G, Zo_lo_G) -> float:
    """sin of the largest principal angle between span(Zhat_G) and span(Z_G)."""
    lib = _load()
    Zhat = _colmajor(Zhat_G)
    n, g = Zhat.shape
    zh, zl = _colmajor(Zo_hi_G), _colmajor(Zo_lo_G)
    P = np.zeros((g, n))
    lib.oracle_subspace_residual(n, g, Zhat.ctypes.data_as(_dp), n, zh.ctypes.data_as(_dp),
                                 zl.ctypes.data_as(_dp), _p(P))
    return float(np.linalg.norm(P.T, 2))


def jacobi(d, e, d_lo=None, e_lo=None):
    """Brute-force cyclic Jacobi (binary128) on the dense matrix; n <= 64."""
    lib = _load()
    d, e, d_lo, e_lo = _f64(d), _f64(e), _f64(d_lo), _f64(e_lo)
    n = d.size
    lh, ll = np.zeros(n), np.zeros(n)
    vh, vl = np.zeros((n, n)), np.zeros((n, n))
    rc = lib.oracle_jacobi(n, _p(d), _p(d_lo), _pe(e), _p(e_lo), _p(lh), _p(ll), _p(vh), _p(vl))
    assert rc == 0
    return lh, ll, vh.T, vl.T


def solve(d, e, idx=None, group_tol_rel: float = 1e-3, group_tol: float | None = None,
          seed: int = 12345):
    """Eigenpairs for the 1-based indices idx: (lam_hi, lam_lo, Z_hi, Z_lo)."""
    lh, ll = eigvals(d, e, idx)
    zh, zl = eigvecs(d, e, lh, ll, group_tol=group_tol, group_tol_rel=group_tol_rel, seed=seed)
    return lh, ll, zh, zl
