// dd_probe.cu -- TEST INFRASTRUCTURE: exposes the product's pair-arithmetic layer
// (paper_1304_1864_b200/csrc/dd.cuh, binary_y of PAPER.md §3.1) through a tiny
// C-ABI so tests/test_dd.py can check every operation against exact rational arithmetic
// (Python fractions) on the host and on the device.  Nothing here is on the solve path.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_1304_1864_b200/csrc/dd.cuh"

using namespace mr3;

// op: 0 add (sloppy), 1 add_ieee, 2 sub, 3 mul, 4 div, 5 fma_dd (a*b+c), 6 dot2_dd (a*b+c*d
// with d = (c_hi, c_lo) reused: a*b + c*c), 7 sqrt_r(a), 8 mul(dd, double b.hi), 9 add(dd, double b.hi)
MR3_HD void dd_apply(int op, dd a, dd b, dd c, dd &r) {
    switch (op) {
        case 0: r = add(a, b); break;
        case 1: r = add_ieee(a, b); break;
        case 2: r = sub(a, b); break;
        case 3: r = mul(a, b); break;
        case 4: r = div(a, b); break;
        case 5: r = fma_dd(a, b, c); break;
        case 6: r = dot2_dd(a, b, c, c); break;
        case 7: r = sqrt_r(a); break;
        case 8: r = mul(a, b.hi); break;
        case 9: r = add(a, b.hi); break;
        default: r = mkdd(0.0, 0.0);
    }
}

__global__ void k_dd_probe(int op, int64_t n, const double *a, const double *b, const double *c,
                           double *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    dd r;
    dd_apply(op, mkdd(a[2 * i], a[2 * i + 1]), mkdd(b[2 * i], b[2 * i + 1]),
             mkdd(c[2 * i], c[2 * i + 1]), r);
    out[2 * i] = r.hi;
    out[2 * i + 1] = r.lo;
}

extern "C" {
// a, b, c, out: n interleaved (hi, lo) pairs in HOST memory
void ddp_host(int op, int64_t n, const double *a, const double *b, const double *c, double *out) {
    for (int64_t i = 0; i < n; i++) {
        dd r;
        dd_apply(op, mkdd(a[2 * i], a[2 * i + 1]), mkdd(b[2 * i], b[2 * i + 1]),
                 mkdd(c[2 * i], c[2 * i + 1]), r);
        out[2 * i] = r.hi;
        out[2 * i + 1] = r.lo;
    }
}
// the same with DEVICE pointers; returns a cudaError_t
int ddp_device(int op, int64_t n, const double *a, const double *b, const double *c, double *out) {
    if (n <= 0) return 0;
    k_dd_probe<<<(unsigned)((n + 255) / 256), 256>>>(op, n, a, b, c, out);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}
}
