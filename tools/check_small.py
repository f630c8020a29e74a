#!/usr/bin/env python3
"""Quick GPU sanity check: residuals, orthogonality and RQI fallbacks on representative matrices."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

for p in (synth.random_uniform(900, 11), synth.glued_wilkinson(12, 21), synth.legendre(3000),
          synth.random_uniform(4000, 3)):
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    T = np.diag(p.d) + np.diag(p.e, 1) + np.diag(p.e, -1)
    nT = np.abs(T).sum(axis=0).max()
    w, Z, st = mr3.mr3_dstemr_dd(d, e)
    w, Z = w.cpu().numpy(), Z.cpu().numpy()
    R = np.linalg.norm(T @ Z - Z * w[None, :], axis=0) / nT
    O = np.abs(Z.T @ Z - np.eye(p.n)).max()
    print(p.name, "iters_max", st["rqi_iters_max"], "fallbacks", st["rqi_fallbacks"], "maxR", R.max(),
          "O", O, flush=True)
