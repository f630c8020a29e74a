// FP64 dependent-chain latencies (cycles) on one thread: DFMA, DADD, DMUL
#include <cstdio>
__global__ void k(double *out, long long *cyc, double a, double b, int n) {
    double x = a, y = b, z = a;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) x = fma(x, b, a);
    }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) y = y + a;
    }
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) z = z * b;
    }
    long long t3 = clock64();
    out[0] = x + y + z;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
    double *o; long long *c; cudaMalloc(&o, 8); cudaMalloc(&c, 24);
    int n = 100000;
    k<<<1, 1>>>(o, c, 1e-9, 0.999999, n);
    k<<<1, 1>>>(o, c, 1e-9, 0.999999, n);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("DFMA %.2f DADD %.2f DMUL %.2f cycles\n", h[0] / (16.0 * n), h[1] / (16.0 * n), h[2] / (16.0 * n));
    return 0;
}
