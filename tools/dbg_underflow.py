"""Bounded probe of the graded matrix that runs into subnormal / zero entries (tools/stress.py --large)."""
import faulthandler
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402

faulthandler.dump_traceback_later(int(sys.argv[2]) if len(sys.argv) > 2 else 60, exit=True)
n = int(sys.argv[1])
k0 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
k = np.arange(k0, k0 + n)
d = 2.0 ** (-k / 4.0)
e = 2.0 ** (-(k[:-1] + 0.5) / 4.0) * 0.3
print("n", n, "subnormal d", int(np.sum((d > 0) & (d < 2.3e-308))), "zero d", int(np.sum(d == 0)), flush=True)
mr3.set_param("DEBUG", 1, 0)
t0 = time.time()
w, Z, st = mr3.mr3_dstemr_dd(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), "V", "A")
torch.cuda.synchronize()
print("solve s", time.time() - t0, {k_: st[k_] for k_ in ("n_blocks", "d_max", "n_clusters", "rqi_fallbacks")}, flush=True)
print(st["t_ms"])
