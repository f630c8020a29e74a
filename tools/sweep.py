"""Sweep a solver parameter on one config (GPU): k_bisect / k_rqi / total ms."""
import sys, time
import torch
sys.path.insert(0, ".")
import synth
import paper_1304_1864_b200 as mr3

cfg = int(sys.argv[1]); name = sys.argv[2]; vals = [float(v) for v in sys.argv[3:]]
p = synth.config(cfg)
d = torch.from_numpy(p.d).cuda(); e = torch.from_numpy(p.e).cuda()
il, iu = p.index_range()
fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
for v in vals:
    mr3.set_param(name, v, 1 if p.io == "f32" else 0)
    best = None
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        w, Z, st = fn(d, e, "V", p.range, il, iu)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        kt = mr3.kernel_times()
        if best is None or dt < best[0]:
            best = (dt, kt)
        del w, Z
    m = iu - il + 1
    print(f"{name}={v}: total {1e3*best[0]:.1f} ms", {k: round(x[0], 2) for k, x in best[1].items()},
          "rqi_rows/(n m)", round(st["rqi_rows"] / p.n / m, 3), "iters_max", st["rqi_iters_max"],
          "bisect_x/(n m)", round(st["bisect_rows_x"] / p.n / m, 2))
