#!/usr/bin/env python3
"""Degenerate dense symmetric inputs through mr3_dsyevr_dd (GPU), checked with numpy in binary64:
zero, identity, diagonal, rank one, already tridiagonal, tiny orders, clustered spectra."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402

rng = np.random.default_rng(7)


def cases():
    yield "n=1", np.array([[2.5]])
    yield "n=2", np.array([[2.0, 1.0], [1.0, -1.0]])
    yield "n=3", np.array([[1.0, 2.0, 3.0], [2.0, 0.0, -1.0], [3.0, -1.0, 4.0]])
    for n in (64, 300):
        yield f"zero n={n}", np.zeros((n, n))
        yield f"identity n={n}", np.eye(n)
        yield f"diagonal n={n}", np.diag(rng.standard_normal(n))
        yield f"rank one n={n}", np.ones((n, n))
        t = np.diag(rng.standard_normal(n)) + np.diag(rng.random(n - 1), 1)
        yield f"tridiagonal n={n}", t + np.triu(t, 1).T
        q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = np.concatenate([np.full(n // 2, 1.0), np.linspace(2, 3, n - n // 2)])
        a = (q * lam) @ q.T
        yield f"half-cluster n={n}", 0.5 * (a + a.T)
        lam = 1.0 + 1e-14 * rng.standard_normal(n)
        a = (q * lam) @ q.T
        yield f"all clustered n={n}", 0.5 * (a + a.T)
        a = rng.standard_normal((n, n))
        yield f"random n={n}", 0.5 * (a + a.T)
        yield f"random x1e-200 n={n}", 0.5 * (a + a.T) * 1e-200


nfail = 0
for name, A in cases():
    n = A.shape[0]
    try:
        w, Z, st = mr3.mr3_dsyevr_dd(torch.from_numpy(np.ascontiguousarray(A)).cuda())
        torch.cuda.synchronize()
        w = w.cpu().numpy()
        Z = Z.cpu().numpy()
        nrm = max(np.abs(A).sum(1).max(), 1e-300)
        eps = 2.0 ** -53
        res = np.max(np.linalg.norm((A / nrm) @ Z - Z * (w / nrm)[None, :], axis=0)) / (n * eps)
        orth = np.max(np.abs(Z.T @ Z - np.eye(n))) / (n * eps)
        eig = np.max(np.abs(w / nrm - np.linalg.eigvalsh(A / nrm))) / (n * eps)
        asc = bool(np.all(np.diff(w) >= 0))
        bad = (not np.isfinite(res + orth + eig)) or max(res, orth, eig) > 20 or not asc
        r = f"{'FAIL' if bad else 'ok  '} res {res:7.3f} orth {orth:7.3f} eig {eig:7.3f} asc {int(asc)}"
    except Exception as ex:  # noqa: BLE001
        r = f"EXC {type(ex).__name__}: {ex}"
        bad = True
    nfail += bad
    print(f"{name:26s} {r}", flush=True)
print("failures:", nfail)
