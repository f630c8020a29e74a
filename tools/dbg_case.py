#!/usr/bin/env python3
"""One config-5 style solve with MR3_DEBUG diagnostics (set MR3_DEBUG in the environment)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = synth.config(cfg)
il, iu = p.index_range()
d = torch.from_numpy(p.d).cuda()
e = torch.from_numpy(p.e).cuda()
fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
for r in range(reps):
    w, Z, st = fn(d, e, "V", p.range, il, iu)
    torch.cuda.synchronize()
    print({k: round(v[0], 3) for k, v in mr3.kernel_times().items()}, st["rqi_iters_max"], flush=True)
    del w, Z
