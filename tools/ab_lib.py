#!/usr/bin/env python3
"""Time one build of libmr3.so on a BASELINE config and compare its output with another's.

usage: tools/ab_lib.py <lib.so> <config> <reps> <out.npz> [<reference.npz>]
Prints per-kernel device times of every rep; saves w and a sample of Z columns to out.npz;
with a reference file prints max |dw| / ||T||_1 and the sampled column differences (up to sign).
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

lib, cfg, reps, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
ref = sys.argv[5] if len(sys.argv) > 5 else None
mr3.LIB_PATH = lib
p = synth.config(cfg)
il, iu = p.index_range()
fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
d = torch.from_numpy(p.d).cuda()
e = torch.from_numpy(p.e).cuda()
for r in range(reps):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    w, Z, st = fn(d, e, "V", p.range, il, iu)
    b.record()
    torch.cuda.synchronize()
    kt = {k: round(t, 2) for k, (t, _) in mr3.kernel_times().items()}
    print(f"{lib} cfg {cfg} rep {r}: {a.elapsed_time(b):8.2f} ms {kt} iters_max={st['rqi_iters_max']}"
          f" fallbacks={st['rqi_fallbacks']}", flush=True)
    if r < reps - 1:
        del w, Z
m = Z.shape[1]
cols = np.unique(np.linspace(0, m - 1, min(m, 64)).astype(np.int64))
wn = w.double().cpu().numpy()
Zs = Z[:, torch.from_numpy(cols).cuda()].double().cpu().numpy()
np.savez(out, w=wn, cols=cols, Z=Zs)
if ref:
    R = np.load(ref)
    tn = float(np.max(np.abs(p.d)) + 2 * np.max(np.abs(p.e)))
    dz = Zs - R["Z"]
    dz2 = Zs + R["Z"]
    dcol = np.minimum(np.abs(dz).max(axis=0), np.abs(dz2).max(axis=0))
    print(f"vs {ref}: max|dw|/|T| = {np.max(np.abs(wn - R['w'])) / tn:.3e}  "
          f"max sampled |dz| = {dcol.max():.3e}", flush=True)
