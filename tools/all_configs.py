#!/usr/bin/env python3
"""Time every BASELINE config (device API, inputs resident) and print the solver stats."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

for cfg in range(1, 6):
    p = synth.config(cfg)
    il, iu = p.index_range()
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
    ts = []
    for r in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        w, Z, st = fn(d, e, "V", p.range, il, iu)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
        del w, Z
    kt = {k: round(v[0], 2) for k, v in mr3.kernel_times().items()}
    print(f"config {cfg} ({p.name}, n={p.n}, io={p.io}): ms {[round(t, 2) for t in ts]} "
          f"iters_max={st['rqi_iters_max']} fallbacks={st['rqi_fallbacks']} clusters={st['n_clusters']} "
          f"levels={st['levels']} {kt}", flush=True)
