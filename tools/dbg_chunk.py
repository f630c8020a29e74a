#!/usr/bin/env python3
"""Diagnostics: handoffs of the chunk-parallel RQI (MR3_DEBUG=1) on a config or a small case."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa
import synth  # noqa
cfg = sys.argv[1]
p = synth.config(int(cfg)) if cfg.isdigit() else eval("synth." + cfg)
il, iu = p.index_range()
mode = 1 if p.io == "f32" else 0
mr3.set_param("DEBUG", float(sys.argv[2]) if len(sys.argv) > 2 else 1, mode)
fn = mr3.mr3_sstemr_d if mode else mr3.mr3_dstemr_dd
w, Z, st = fn(torch.from_numpy(p.d).cuda(), torch.from_numpy(p.e).cuda(), "V", p.range, il, iu)
torch.cuda.synchronize()
print(st)
