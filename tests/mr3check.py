"""Verification helpers for the GPU parity tests (test infrastructure).

Readings of the tolerances:
  fp64 I/O : |w - lambda_oracle| <= 4e-16 ||T||_1 ; R2 <= 1e-15 (2-norm numerator);
             R1 (Eq. 1.1) <= max(1e-15, 4 * R1 floor of the oracle's own rounded
             vectors) ; O <= 1e-14 ; per-column / per-group angles vs the oracle
             within the Gap-theorem bound (c5).
  fp32 I/O : |w - lambda| <= 4 eps_s ||T||_1 ; R1 <= 5e-7 ; O <= 5e-6.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle

EPS_S = 2.0 ** -24


def exact_orthogonality(Z: torch.Tensor):
    """O = max_{i!=j} |z_i^T z_j| and max |z_i^T z_i - 1| with error ~1e-19.

    Each column is split as z = h + l with h on a grid of 2^-b relative to the
    column's max, b = floor((52 - ceil(log2 n))/2): every product h_i h_j has at
    most 2b significant bits and n of them sum exactly in fp64, so H^T H is
    exact regardless of the GEMM's summation order; the small terms H^T L, L^T H,
    L^T L carry fp64 relative error on quantities below 2^-b.
    """
    Z = Z.to(torch.float64)
    n, m = Z.shape
    b = int((52 - int(np.ceil(np.log2(max(n, 2))))) // 2)
    mx = Z.abs().amax(dim=0).clamp_min(1e-300)
    e = torch.ceil(torch.log2(mx))
    scale = torch.pow(2.0, b - e)
    H = torch.round(Z * scale) / scale
    L = Z - H
    G = H.T @ H
    G += H.T @ L + L.T @ H + L.T @ L
    dg = torch.diagonal(G).clone()
    G.fill_diagonal_(0.0)
    return float(G.abs().max()) if m > 1 else 0.0, float((dg - 1).abs().max())


def exact_gram(A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """A^T B with the same exact-splitting scheme as exact_orthogonality."""
    A = A.to(torch.float64)
    B = B.to(torch.float64)
    n = A.shape[0]
    b = int((52 - int(np.ceil(np.log2(max(n, 2))))) // 2)

    def split(X):
        mx = X.abs().amax(dim=0).clamp_min(1e-300)
        sc = torch.pow(2.0, b - torch.ceil(torch.log2(mx)))
        H = torch.round(X * sc) / sc
        return H, X - H

    Ha, La = split(A)
    Hb, Lb = split(B)
    G = Ha.T @ Hb
    G += Ha.T @ Lb + La.T @ Hb + La.T @ Lb
    return G


def oracle_pairs(p, idx, need_vectors=True, group_tol=None):
    d = p.d.astype(np.float64)
    e = p.e.astype(np.float64)
    lh, ll = oracle.eigvals(d, e, idx)
    if not need_vectors:
        return lh, ll, None, None
    zh, zl = oracle.eigvecs(d, e, lh, ll, group_tol=group_tol,
                            group_tol_rel=1e-3 if len(idx) <= 1500 else 1e-9)
    return lh, ll, zh, zl


def check_solution(p, w, Z, idx, io="f64", oracle_vectors=True, gate_angles=True,
                   full_orth=True, verbose=False):
    """Compare GPU eigenpairs (w[j], Z[:, j]) for the 1-based indices idx with the oracle.

    w, Z are numpy (host) arrays for exactly these indices.  Returns a metrics dict.
    """
    d = p.d.astype(np.float64)
    e = p.e.astype(np.float64)
    n = p.n
    idx = np.asarray(idx, dtype=np.int64)
    nrm = oracle.norm1(d, e)
    w = np.asarray(w, dtype=np.float64)
    res = {"n": n, "m": int(idx.size)}
    # neighbours for gaps
    ext = np.unique(np.concatenate([idx, np.clip(idx - 1, 1, n), np.clip(idx + 1, 1, n)]))
    lh_all, ll_all = oracle.eigvals(d, e, ext)
    lam_ext = lh_all + ll_all
    pos = {int(k): i for i, k in enumerate(ext)}
    lam = np.array([lam_ext[pos[int(k)]] for k in idx])
    lam_hi = np.array([lh_all[pos[int(k)]] for k in idx])
    lam_lo = np.array([ll_all[pos[int(k)]] for k in idx])
    dl = np.abs(w - lam)
    res["eig_err"] = float(dl.max() / nrm) if idx.size else 0.0
    if Z is None:
        return res
    Zd = np.asarray(Z, dtype=np.float64)
    r1, r2, zn = oracle.residuals(d, e, w, Zd)
    res["R1"] = float(r1.max())
    res["R2"] = float(r2.max())
    res["norm_dev"] = float(np.abs(zn).max())
    if full_orth:
        if torch.cuda.is_available():
            o, dd = exact_orthogonality(torch.from_numpy(Zd).cuda())
        else:
            o, dd = oracle.orthogonality(Zd)
        res["O"] = o
        res["diag_dev"] = dd
    if oracle_vectors:
        zh, zl = oracle.eigvecs(d, e, lam_hi, lam_lo,
                                group_tol_rel=1e-3 if idx.size <= 1500 else 1e-9)
        # R1 floor: the oracle's own vectors rounded to the output format
        fl = np.float32 if io == "f32" else np.float64
        wz = (lam_hi + lam_lo).astype(fl).astype(np.float64)
        zf = (zh + zl).astype(fl).astype(np.float64)
        f1, f2, _ = oracle.residuals(d, e, wz, zf)
        res["R1_floor"] = float(f1.max())
        # gap-scaled angle rule
        rnorm = r2 * nrm
        theta = 2.0 * rnorm.max() / 1e-6
        ang = oracle.sin_angles(Zd, zh, zl)
        res["max_angle"] = float(ang.max())
        worst_ratio = 0.0
        n_group = 0
        # groups among consecutive requested indices (plus neighbour gaps)
        order = np.argsort(idx)
        i = 0
        while i < len(order):
            j = i
            while j + 1 < len(order) and idx[order[j + 1]] == idx[order[j]] + 1 and \
                    lam[order[j + 1]] - lam[order[j]] < theta:
                j += 1
            members = order[i:j + 1]
            kL, kR = idx[members[0]], idx[members[-1]]
            gl = lam_ext[pos[int(kL)]] - lam_ext[pos[int(max(kL - 1, 1))]] if kL > 1 else np.inf
            gr = lam_ext[pos[int(min(kR + 1, n))]] - lam_ext[pos[int(kR)]] if kR < n else np.inf
            gapout = min(gl, gr)
            if len(members) == 1:
                k = members[0]
                bound = max(1e-13, 2.0 * rnorm[k] / gapout)
                ratio = ang[k] / bound
            else:
                n_group += 1
                s = oracle.subspace_sin(Zd[:, members], zh[:, members], zl[:, members])
                bound = max(1e-13, 2.0 * np.sqrt(np.sum(rnorm[members] ** 2)) / gapout)
                ratio = s / bound
            worst_ratio = max(worst_ratio, ratio)
            i = j + 1
        res["angle_bound_ratio"] = float(worst_ratio)
        res["n_groups"] = n_group
        res["frac_cols_le_1e-13"] = float(np.mean(ang <= 1e-13))
    if verbose:
        print(res)
    return res


def assert_parity(res, io="f64", gate_angles=True):
    if io == "f64":
        assert res["eig_err"] <= 4e-16, res
        if "R2" in res:
            assert res["R2"] <= 1e-15, res
            if "R1_floor" in res:
                assert res["R1"] <= max(1e-15, 4 * res["R1_floor"]), res
        if "O" in res:
            assert res["O"] <= 1e-14 and res["diag_dev"] <= 1e-14, res
        if gate_angles and "angle_bound_ratio" in res:
            assert res["angle_bound_ratio"] <= 1.0, res
    else:
        assert res["eig_err"] <= 4 * EPS_S, res
        if "R1" in res:
            assert res["R1"] <= 5e-7, res
        if "O" in res:
            assert res["O"] <= 5e-6 and res["diag_dev"] <= 5e-6, res
