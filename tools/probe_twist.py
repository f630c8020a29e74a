"""Located twists of the reduced dense T (DEBUG dump) -- diagnosis of the dense stragglers."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402

d = np.load(sys.argv[1])
e = np.load(sys.argv[2])
dt = torch.from_numpy(d).cuda()
et = torch.from_numpy(e).cuda()
mr3.set_param("DEBUG", 1)
w, Z, st = mr3.mr3_dstemr_dd(dt, et)
torch.cuda.synchronize()
mr3.set_param("DEBUG", -1)
print("fallbacks", st["rqi_fallbacks"])
