// Microbenchmark (tools only): does a non-FP64 instruction issue in the shadow of a DFMA?
// Every thread runs 8 independent DFMA chains and, per 8 DFMA, NI independent instructions of
// another pipe (KIND 0: IMAD, 1: FFMA, 2: LDS, 3: LOP3/XOR).  Prints the FP64 rate and the
// total warp-instruction rate per SM sub-partition cycle (1.965 GHz assumed).
#include <cstdio>
template <int KIND, int NI>
__global__ void k(double *out, int iters, double a, double b, int m, float fb) {
    __shared__ int sm[256 * 4];
    double x[8];
    int y[16];
    float f[16];
    for (int j = 0; j < 8; j++) x[j] = a + j * 1e-3 + threadIdx.x * 1e-9;
    for (int j = 0; j < 16; j++) { y[j] = threadIdx.x + j; f[j] = (float)j + fb; }
    for (int j = 0; j < 4; j++) sm[threadIdx.x * 4 + j] = (threadIdx.x * 4 + j * 7) & 1023;
    __syncthreads();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
#pragma unroll
            for (int j = 0; j < 8; j++) x[j] = fma(x[j], b, a);
#pragma unroll
            for (int j = 0; j < NI; j++) {
                if (KIND == 0) y[j] = y[j] * m + i;
                if (KIND == 1) f[j] = fmaf(f[j], fb, 1.0f);
                if (KIND == 2) y[j] = sm[y[j] & 1023];
                if (KIND == 3) y[j] = (y[j] ^ m) & (i | 0x55555);
            }
        }
    }
    double s = 0;
    for (int j = 0; j < 8; j++) s += x[j];
    for (int j = 0; j < 16; j++) s += y[j] + f[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int KIND, int NI>
void run(double *o, int grid, const char *name) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    k<KIND, NI><<<grid, 256>>>(o, 10, 1.0, 0.9999999, 3, 0.999f);
    cudaEventRecord(e0);
    k<KIND, NI><<<grid, 256>>>(o, iters, 1.0, 0.9999999, 3, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fp64 = (double)grid * 256 * iters * 64 / (ms * 1e-3);
    const double other = fp64 * NI / 8.0;
    printf("%-5s NI=%2d per 8 DFMA: FP64 %.2f T/s, other %.2f T/s, %.3f ms\n", name, NI,
           fp64 / 1e12, other / 1e12, ms);
}
int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *o;
    cudaMalloc(&o, (size_t)nsm * 8 * 256 * 8);
    const int g = nsm * 8;
    run<0, 0>(o, g, "none");
    run<0, 4>(o, g, "IMAD"); run<0, 8>(o, g, "IMAD"); run<0, 12>(o, g, "IMAD"); run<0, 16>(o, g, "IMAD");
    run<1, 4>(o, g, "FFMA"); run<1, 8>(o, g, "FFMA"); run<1, 12>(o, g, "FFMA"); run<1, 16>(o, g, "FFMA");
    run<2, 4>(o, g, "LDS"); run<2, 8>(o, g, "LDS"); run<2, 12>(o, g, "LDS");
    run<3, 4>(o, g, "LOP"); run<3, 8>(o, g, "LOP"); run<3, 16>(o, g, "LOP");
    return 0;
}
