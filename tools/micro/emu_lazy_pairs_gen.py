import sys, struct, numpy as np
sys.path.insert(0, '/root/repo'); import synth
from scipy.linalg import eigh_tridiagonal
p = synth.config(int(sys.argv[1])); j = int(sys.argv[2])
a, b = p.d.astype(np.float64), p.e.astype(np.float64); n = len(a)
gl = np.min(a - np.abs(np.r_[0, b]) - np.abs(np.r_[b, 0]))
mu = gl - 1e-3 * abs(gl) - 1e-3
d = np.zeros(n); l = np.zeros(n)
d[0] = a[0] - mu
for i in range(n - 1):
    l[i] = b[i] / d[i]; d[i + 1] = a[i + 1] - mu - l[i] * b[i]
assert np.all(d > 0)
w, V = eigh_tridiagonal(a - mu, b, select='i', select_range=(j, j))
lam = w[0]; r = int(np.argmax(np.abs(V[:, 0])))
def two_prod(x, y):
    h = x * y; return h, np.fma(x, y, -h) if hasattr(np, 'fma') else 0.0
import math
with open('/tmp/emu/in.bin', 'wb') as f:
    f.write(struct.pack('<idd q', n, lam, 0.0, r))
    for i in range(n):
        from fractions import Fraction as Fr
        ex = Fr(d[i]) * Fr(l[i]); ld = float(ex); ldl = float(ex - Fr(ld))
        ex2 = ex * Fr(l[i]); lld = float(ex2); lldl = float(ex2 - Fr(lld))
        f.write(struct.pack('<6d', d[i], 0.0, ld, ldl, lld, lldl))
print('n', n, 'lam', lam, 'r', r)
