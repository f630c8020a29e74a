"""Timing probe of the dense pipeline (GPU): per-phase device times at a few sizes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096]:
    p = synth.dense_config(n, 0)
    A = torch.from_numpy(np.ascontiguousarray(p.A)).cuda()
    for rep in range(3):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        w, Z, st = mr3.mr3_dsyevr_dd(A)
        b.record()
        torch.cuda.synchronize()
        kt = {k: round(t, 2) for k, (t, _) in mr3.kernel_times().items()}
        print(n, rep, f"{a.elapsed_time(b):.2f} ms", "reduce", round(st["t_ms"]["reduce"], 2),
              "back", round(st["t_ms"]["backtransform"], 2), kt, flush=True)
