"""Solve one config with MR3_DEBUG set in the environment (prints tree levels and
the RQI iteration histogram from the library) and print the stats."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

p = synth.config(int(sys.argv[1]))
d = torch.from_numpy(p.d).cuda()
e = torch.from_numpy(p.e).cuda()
il, iu = p.index_range()
fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
w, Z, st = fn(d, e, "V", p.range, il, iu)
print(st)
