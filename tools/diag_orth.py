"""Diagnose the worst orthogonality pair of a solve (GPU)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle, synth
import paper_1304_1864_b200 as mr3
from mr3check import exact_gram

def main(copies=2, seed=None):
    p = synth.glued_wilkinson(copies, 21)
    if seed is not None:
        mr3.set_param("SEED", seed)
    d = torch.from_numpy(p.d).cuda(); e = torch.from_numpy(p.e).cuda()
    w, Z, st = mr3.mr3_dstemr_dd(d, e)
    print(st)
    G = exact_gram(Z, Z) - torch.eye(p.n, dtype=torch.float64, device="cuda")
    Gc = G.abs().cpu().numpy()
    wc = w.cpu().numpy(); Zc = Z.cpu().numpy()
    lh, ll, zh, zl = oracle.solve(p.d, p.e)
    r1, r2, _ = oracle.residuals(p.d, p.e, wc, Zc)
    ang = oracle.sin_angles(Zc, zh, zl)
    order = np.dstack(np.unravel_index(np.argsort(-Gc.ravel()), Gc.shape))[0][:12]
    for i, j in order:
        if i < j:
            print(f"pair {i},{j}: |zi.zj|={Gc[i,j]:.3e} w={wc[i]:.17g},{wc[j]:.17g} gap={wc[j]-wc[i]:.3e} "
                  f"lam_or={lh[i]+ll[i]:.17g} r2={r2[i]:.2e},{r2[j]:.2e} ang={ang[i]:.2e},{ang[j]:.2e}")
    # oracle gaps
    lam = lh + ll
    print("min oracle gap", np.min(np.diff(lam)))

if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
