"""Host vs device time of repeated solves (GPU): finds host overhead in the timed region."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1304_1864_b200 as mr3

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = synth.config(cfg)
d = torch.from_numpy(p.d).cuda(); e = torch.from_numpy(p.e).cuda()
il, iu = p.index_range()
fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
for xp in (1, 0):
    mr3.set_param("XPHASE", xp)
    for it in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        w, Z, st = fn(d, e, "V", p.range, il, iu)
        b.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        kt = mr3.kernel_times()
        print(f"xphase={xp} it={it} host={1e3*(t1-t0):.2f} ms events={a.elapsed_time(b):.2f} ms "
              f"kernels={sum(v[0] for v in kt.values()):.2f} {dict((k, round(v[0],2)) for k,v in kt.items())}")
        del w, Z
