#!/usr/bin/env python3
"""A/B a solver parameter on one box: alternate the settings, print per-kernel device times.

usage: tools/ab_param.py <config> <PARAM> <v1> <v2> [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

cfg, name, v1, v2 = int(sys.argv[1]), sys.argv[2], float(sys.argv[3]), float(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
p = synth.config(cfg)
il, iu = p.index_range()
mode = 1 if p.io == "f32" else 0
fn = mr3.mr3_sstemr_d if mode else mr3.mr3_dstemr_dd
d = torch.from_numpy(p.d).cuda()
e = torch.from_numpy(p.e).cuda()
ref = None
for r in range(reps):
    for v in (v1, v2):
        mr3.set_param(name, v, mode)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        w, Z, st = fn(d, e, "V", p.range, il, iu)
        b.record()
        torch.cuda.synchronize()
        kt = {k: round(t, 2) for k, (t, _) in mr3.kernel_times().items()}
        if ref is None:
            ref = w.clone()
            refZ = Z.clone()
        dw = float((w - ref).abs().max())
        dz = float((Z - refZ).abs().max())
        print(f"{name}={v:g} rep {r}: {a.elapsed_time(b):8.2f} ms  {kt}  iters_max={st['rqi_iters_max']}"
              f" rows_x={st['bisect_rows_x']:.3g} rqi_rows={st['rqi_rows']:.4g} max|dw|={dw:.2e} max|dZ|={dz:.2e}",
              flush=True)
        del w, Z
mr3.set_param(name, -1, mode)
