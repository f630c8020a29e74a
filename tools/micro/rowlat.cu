// Microbenchmark (tools only): latency of one projective fixed-twist F row in pair
// arithmetic (k_rqi / k_rqi_fb), one thread, rows read from shared memory; variants:
//   0: D = d q + p ; p' = lld p - lam D              (current form)
//   1: the same + the l+ norm chain (rcp, W)          (current kernel row)
//   2: dot2 form p' = (lld - lam) p - (lam d) q
//   3: two independent chains interleaved (form 0)
// prints cycles per row (clock64)
#include <cstdio>
#include "../../paper_1304_1864_b200/csrc/dd.cuh"
using namespace mr3;
constexpr int NR = 512;
__global__ void k(int variant, int reps, double *out, long long *cyc) {
    __shared__ double rows[NR * 8];
    for (int i = threadIdx.x; i < NR * 8; i += blockDim.x)
        rows[i] = (i % 8 == 1 || i % 8 == 3 || i % 8 == 5 || i % 8 == 7) ? 1e-18 * (i % 13) : 0.5 + 0.001 * (i % 97);
    __syncthreads();
    if (threadIdx.x != 0) return;
    dd lam = mkdd(0.3, 1e-18), mlam = neg(lam);
    dd p = mlam, q = mkdd(1.0, 0.0), p2 = mlam, q2 = mkdd(1.0, 0.0);
    double W = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
#pragma unroll 8
        for (int k = 0; k < NR; k++) {
            const double2 *rp = reinterpret_cast<const double2 *>(rows + 8 * k);
            double2 a = rp[0], b = rp[1], dd4 = rp[3];
            dd d = mkdd(a.x, a.y), lld = mkdd(b.x, b.y), ld = mkdd(dd4.x, dd4.y);

            if (variant == 0 || variant == 1) {
                dd D = fma_dd(d, q, p);
                if (variant == 1) {
                    double lpx = hi(ld) * hi(q) * rcp(hi(D));
                    double l2 = lpx * lpx;
                    W = fmin(fma(l2, W, l2), 1e250);
                }
                p = fma_dd(mlam, D, mul(lld, p));
                q = D;
            } else if (variant == 2) {
                dd D = fma_dd(d, q, p);
                p = dot2_dd(add(lld, mlam), p, mul(mlam, d), q);
                q = D;
            } else {
                dd D = fma_dd(d, q, p);
                dd D2 = fma_dd(d, q2, p2);
                p = fma_dd(mlam, D, mul(lld, p));
                p2 = fma_dd(mlam, D2, mul(lld, p2));
                q = D;
                q2 = D2;
            }
            if ((k & 7) == 7) {  // rescale as the kernels do
                const unsigned ex = (unsigned)__double2hiint(hi(p)) & 0x7ff00000u;
                const unsigned ey = (unsigned)__double2hiint(hi(q)) & 0x7ff00000u;
                const unsigned em = ex > ey ? ex : ey;
                if (em != 0x7ff00000u && em != 0u) {
                    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                    p = scale_pow2(p, sc);
                    q = scale_pow2(q, sc);
                    p2 = scale_pow2(p2, sc);
                    q2 = scale_pow2(q2, sc);
                }
            }
        }
    }
    long long t1 = clock64();
    out[0] = hi(p) + hi(q) + W + hi(p2) + hi(q2);
    cyc[0] = t1 - t0;
}
int main() {
    double *o;
    long long *c;
    cudaMalloc(&o, 8);
    cudaMalloc(&c, 8);
    const int reps = 20;
    for (int v = 0; v < 4; v++) {
        k<<<1, 32>>>(v, 1, o, c);
        k<<<1, 32>>>(v, reps, o, c);
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("variant %d: %.1f cycles per row\n", v, (double)h / (reps * NR));
    }
    return 0;
}
