#!/usr/bin/env python3
"""One solve of a BASELINE config (optionally an index subset) for ncu captures.

usage: tools/prof_case.py <config> [reps] [il iu] [jobz]
The subset form keeps Z small enough for ncu's kernel replay (which saves and
restores the memory a kernel writes); per-launch numbers scale with the columns.
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = synth.config(cfg)
il, iu = p.index_range()
rng = p.range
if len(sys.argv) > 4:
    il, iu, rng = int(sys.argv[3]), int(sys.argv[4]), "I"
jobz = sys.argv[5] if len(sys.argv) > 5 else "V"
d = torch.from_numpy(p.d).cuda()
e = torch.from_numpy(p.e).cuda()
fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
for _ in range(reps):
    w, Z, st = fn(d, e, jobz, rng, il, iu)
    torch.cuda.synchronize()
    print({k: round(v[0], 3) for k, v in mr3.kernel_times().items()}, st["rqi_iters_max"])
    del w, Z
