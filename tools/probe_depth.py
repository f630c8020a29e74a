"""Probe: tree depth and backtracking statistics of glued Wilkinson matrices (GPU)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1304_1864_b200 as mr3  # noqa: E402
import synth  # noqa: E402

for copies in [int(c) for c in sys.argv[1:]] or [12, 30, 60, 100, 200]:
    p = synth.glued_wilkinson(copies, 21)
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    for bt in (1, 2):
        mr3.set_param("BACKTRACK", bt)
        t = time.time()
        w, Z, st = mr3.mr3_dstemr_dd(d, e)
        torch.cuda.synchronize()
        print(copies, "BT", bt, "d_max", st["d_max"], "clusters", st["n_clusters"], "fail",
              st["robustness_failures"], "bt", st["backtracks"], "tries", st["backtrack_tries"],
              "iters", st["rqi_iters_max"], "fallbacks", st["rqi_fallbacks"],
              f"{(time.time() - t) * 1e3:.1f} ms", flush=True)
    mr3.set_param("BACKTRACK", -1)
for cfg in (3, 4):
    p = synth.config(cfg)
    il, iu = p.index_range()
    mode = 1 if p.io == "f32" else 0
    fn = mr3.mr3_sstemr_d if mode else mr3.mr3_dstemr_dd
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    for rl in (0, 0.5):
        mr3.set_param("RELAX", rl, mode)
        w, Z, st = fn(d, e, "V", p.range, il, iu)
        torch.cuda.synchronize()
        kt = {k: round(t, 2) for k, (t, _) in mr3.kernel_times().items()}
        print("config", cfg, "RELAX", rl, "rows_y", st["bisect_rows"], "rows_x", st["bisect_rows_x"],
              kt, flush=True)
    mr3.set_param("RELAX", -1, mode)
