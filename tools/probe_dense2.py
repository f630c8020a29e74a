"""Dense pipeline diagnosis: the tridiagonal stage's RQI path on the reduced T (RQI_CHUNK on/off)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = synth.dense_config(n, 0)
A = torch.from_numpy(np.ascontiguousarray(p.A)).cuda()
w, Z, st = mr3.mr3_dsyevr_dd(A)
# the reduced T: run the reduction again on a copy and read d, e back via the overwritten A
Aw = A.clone()
mr3.mr3_dsyevr_dd(Aw, jobz="N", overwrite=True)
Ah = Aw.cpu().numpy()  # row-major storage = column-major of A^T; T is symmetric
d = np.diag(Ah).copy()
e = np.array([Ah[j, j + 1] for j in range(n - 1)])  # row j col j+1 in row-major = A(j+1, j)
print("e stats: min|e|", np.abs(e).min(), "median", np.median(np.abs(e)), "max", np.abs(e).max())
print("e tail", np.abs(e[-8:]))
dt = torch.from_numpy(d).cuda()
et = torch.from_numpy(e).cuda()
for chunk in (8192, 0):
    mr3.set_param("RQI_CHUNK", chunk)
    for rep in range(2):
        w2, Z2, st2 = mr3.mr3_dstemr_dd(dt, et)
        torch.cuda.synchronize()
        kt = {k: round(t, 2) for k, (t, _) in mr3.kernel_times().items()}
        print("RQI_CHUNK", chunk, "iters", st2["rqi_iters_max"], "fallbacks", st2["rqi_fallbacks"],
              "d_max", st2["d_max"], "clusters", st2["n_clusters"], kt, flush=True)
mr3.set_param("RQI_CHUNK", -1)
w3, Z3, st3 = mr3.mr3_dstemr_dd(torch.from_numpy(synth.random_uniform(n, 0).d).cuda(),
                                torch.from_numpy(synth.random_uniform(n, 0).e).cuda())
print("config-2 recipe T directly:", {k: round(t, 2) for k, (t, _) in mr3.kernel_times().items()})
