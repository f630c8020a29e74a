#!/usr/bin/env python3
"""Per-column residuals (binary128 oracle) of one solve under parameter settings.
usage: tools/dbg_resid.py "<synth expr>" PARAM=v ... ; prints the worst columns."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle  # noqa
import paper_1304_1864_b200 as mr3  # noqa
import synth  # noqa
p = eval("synth." + sys.argv[1])
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    mr3.set_param(k, float(v), 1 if p.io == "f32" else 0)
fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
il, iu = p.index_range()
w, Z, st = fn(torch.from_numpy(p.d).cuda(), torch.from_numpy(p.e).cuda(), "V", p.range, il, iu)
w, Z = w.cpu().numpy(), Z.cpu().numpy()
r1, r2, zn = oracle.residuals(p.d.astype(np.float64), p.e.astype(np.float64), w.astype(np.float64), Z.astype(np.float64))
o = np.argsort(-r2)[:12]
print(sys.argv[1:], "R2 max %.3g" % r2.max(), {k: st[k] for k in ("d_max", "n_clusters", "rqi_fallbacks", "rqi_iters_max")})
for j in o:
    print("  col %d w %.17g R2 %.3g |z|-1 %.2g" % (j, w[j], r2[j], zn[j]))
