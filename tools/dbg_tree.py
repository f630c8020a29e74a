import sys, numpy as np, torch
sys.path.insert(0,'.')
import synth, paper_1304_1864_b200 as mr3
p = synth.glued_wilkinson(2, 21)
d = torch.from_numpy(p.d).cuda(); e = torch.from_numpy(p.e).cuda()
w, Z, st = mr3.mr3_dstemr_dd(d, e)
print(st)
