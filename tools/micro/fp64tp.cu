// Microbenchmark (tools only): FP64 pipe throughput per opcode on all SMs (8 independent
// chains per thread, 256 threads, 8 CTAs per SM): DFMA, DADD, DMUL, and a DADD/DFMA mix.
#include <cstdio>
template <int OP>
__global__ void k(double *out, int iters, double a, double b) {
    double x[8];
    for (int j = 0; j < 8; j++) x[j] = a + j * 1e-3 + threadIdx.x * 1e-9;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (OP == 0) x[j] = fma(x[j], b, a);
                if (OP == 1) x[j] = __dadd_rn(x[j], b);
                if (OP == 2) x[j] = __dmul_rn(x[j], b);
                if (OP == 3) x[j] = (j & 1) ? __dadd_rn(x[j], b) : fma(x[j], b, a);
            }
        }
    }
    double s = 0;
    for (int j = 0; j < 8; j++) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
double run(double *o, int grid) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    k<OP><<<grid, 256>>>(o, 10, 1.0, 0.9999999);
    cudaEventRecord(e0);
    k<OP><<<grid, 256>>>(o, iters, 1.0, 0.9999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return (double)grid * 256 * iters * 64 / (ms * 1e-3);
}
int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *o;
    cudaMalloc(&o, (size_t)nsm * 8 * 256 * 8);
    const int g = nsm * 8;
    printf("DFMA %.2f T/s\n", run<0>(o, g) / 1e12);
    printf("DADD %.2f T/s\n", run<1>(o, g) / 1e12);
    printf("DMUL %.2f T/s\n", run<2>(o, g) / 1e12);
    printf("mix DADD/DFMA %.2f T/s\n", run<3>(o, g) / 1e12);
    return 0;
}
