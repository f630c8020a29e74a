"""Dense pipeline diagnosis 2: RQI stragglers on the reduced T under parameter changes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = synth.dense_config(n, 0)
A = torch.from_numpy(np.ascontiguousarray(p.A)).cuda()
Aw = A.clone()
mr3.mr3_dsyevr_dd(Aw, jobz="N", overwrite=True)
Ah = Aw.cpu().numpy()
d = np.diag(Ah).copy()
e = np.array([Ah[j, j + 1] for j in range(n - 1)])
np.save("gpurun_out/dense_T_d.npy", d)
np.save("gpurun_out/dense_T_e.npy", e)
dt = torch.from_numpy(d).cuda()
et = torch.from_numpy(e).cuda()
for params in ({}, {"RELAX": 0}, {"GRID": 0}, {"XPTS": 1}, {"GROUPS": 1}, {"TWISTW": 1e4}):
    for k, v in params.items():
        mr3.set_param(k, v)
    w2, Z2, st2 = mr3.mr3_dstemr_dd(dt, et)
    torch.cuda.synchronize()
    kt = {k: round(t, 2) for k, (t, _) in mr3.kernel_times().items()}
    print(params, "iters", st2["rqi_iters_max"], "fallbacks", st2["rqi_fallbacks"], kt, flush=True)
    for k in params:
        mr3.set_param(k, -1)
mr3.set_param("DEBUG", 1)
w2, Z2, st2 = mr3.mr3_dstemr_dd(dt, et)
torch.cuda.synchronize()
mr3.set_param("DEBUG", -1)
