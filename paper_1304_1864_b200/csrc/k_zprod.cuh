// k_zprod.cuh -- eigenvector components in product form (K6 without a back-substitution sweep).
//
// The twisted solve of Alg. 1 l.11
//   z_r = 1,  z_i = -l+_i z_{i+1} (i < r),  z_{k} = -u-_{k-1} z_{k-1} (k > r)
// consumes l+ bottom-up and u- top-down, i.e. against the directions in which the
// stationary (top-down) and progressive (bottom-up) transforms produce them.  In the
// projective form of those transforms (R8b: s_i = pF_i / qF_i with qF_{i+1} = D_i =
// d+_i qF_i, and p_k = PB_k / QB_k with QB_{k-1} = E_k = D-_k QB_k) the quotients
// telescope:
//   l+_i = ld_i / d+_i = ld_i qF_i / qF_{i+1},
//   u-_{k-1} = l_{k-1} d_{k-1} / D-_k = ld_{k-1} QB_k / QB_{k-1},
// so with PP_k = prod_{j<k} (-ld_j) (a property of the representation alone)
//   z_i = y_i / y_r,  y_i = qF_i / PP_i       (i <= r)
//   z_k = x_k / x_r,  x_k = QB_k PP_k         (k >= r).
// Every component is available in the direction the transforms run: the final
// fixed-twist factorization of k_rqi writes y_i and x_k (scaled by a per-column
// reference power of two) straight into Z, and k_zscale applies the per-column
// factors 1 / y_r, 1 / x_r and the exact 1 / ||z|| afterwards.  PP and 1/PP are
// computed once per representation (k_node_pp) as mantissa-exponent pairs.
#pragma once
#include <type_traits>

#include "kernels.cuh"

namespace mr3 {

// per row of a node: {PPm, IPPm, E (int bits), round(16 log2|PP_k|) (int bits)}: PP_k = PPm 2^E,
// 1/PP_k = IPPm 2^-E.
// The mantissas are products of the representation's ld in pair arithmetic, rounded
// once: z components come out to binary64 accuracy (the output precision).
constexpr int PP_STRIDE = 4;

__device__ __forceinline__ int expo_of(double x) {  // unbiased exponent of a normal double
    return (int)(((unsigned)__double2hiint(x) >> 20) & 0x7ffu) - 1023;
}
template <class R>
__device__ __forceinline__ void normalize_me(R &m, int &e) {  // m -> [1, 2) (or 0), e += shift
    if (hi(m) == 0.0 || !(fabs(hi(m)) < INFINITY)) return;
    const int k = expo_of(hi(m));
    m = scale_pow2(m, __hiloint2double((1023 - k) << 20, 0));
    e += k;
}

// One CTA per node: PP_k = prod_{j<k} (-ld_j) by a chunked multiplicative scan.
// root: pool rows at the node's row0; child nodes: pool rows at (node - first) * stride.
template <class R>
__global__ void __launch_bounds__(256) k_node_pp(NodeInfo *nodes, int first, double *pool,
                                                 int64_t stride, int root) {
    const int node = first + blockIdx.x;
    const NodeInfo nd = nodes[node];
    const int64_t n = nd.n;
    double *pp = pool + (root ? nd.row0 : (int64_t)blockIdx.x * stride) * PP_STRIDE;
    const int64_t C = (n + blockDim.x - 1) / blockDim.x;
    const int64_t r0 = (int64_t)threadIdx.x * C, r1 = min(r0 + C, n);
    // local product of the factors of rows [r0, r1) (factor j = -ld_j, j <= n - 2)
    R m = mk<R>(1.0);
    int e = 0;
    for (int64_t j = r0; j < r1; j++) {
        if (j <= n - 2) {
            m = mul(m, neg(load_row4<R>(nd.rep, j).ld));
            normalize_me(m, e);
        }
    }
    // exclusive multiplicative scan over the threads (tree in smem)
    __shared__ double sh_h[256], sh_l[256];
    __shared__ int sh_e[256];
    sh_h[threadIdx.x] = hi(m);
    sh_l[threadIdx.x] = lo_part(m);
    sh_e[threadIdx.x] = e;
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
        R vm = mk<R>(1.0);
        int ve = 0;
        const bool take = (int)threadIdx.x >= off;
        if (take) {
            vm = mk2<R>(sh_h[threadIdx.x - off], sh_l[threadIdx.x - off]);
            ve = sh_e[threadIdx.x - off];
        }
        __syncthreads();
        if (take) {
            R cur = mk2<R>(sh_h[threadIdx.x], sh_l[threadIdx.x]);
            int ce = sh_e[threadIdx.x] + ve;
            cur = mul(cur, vm);
            normalize_me(cur, ce);
            sh_h[threadIdx.x] = hi(cur);
            sh_l[threadIdx.x] = lo_part(cur);
            sh_e[threadIdx.x] = ce;
        }
        __syncthreads();
    }
    R pm = mk<R>(1.0);  // product of all factors before this thread's chunk
    int pe = 0;
    if (threadIdx.x > 0) {
        pm = mk2<R>(sh_h[threadIdx.x - 1], sh_l[threadIdx.x - 1]);
        pe = sh_e[threadIdx.x - 1];
    }
    for (int64_t j = r0; j < r1; j++) {
        const R ipm = div(mk<R>(1.0), pm);  // 1/PPm in (1/2, 1]
        double *o = pp + j * PP_STRIDE;
        o[0] = hi(pm);
        o[1] = hi(ipm);
        o[2] = __hiloint2double(0, pe);  // E as int bits (no F2I on the readers' path)
        // round(16 log2|PP_j|) as int bits (k_rqi_locate's 1/16-log2 bookkeeping)
        o[3] = __hiloint2double(0, (int)lrint(16.0 * (log2(fabs(hi(pm))) + (double)pe)));
        if (j <= n - 2) {
            pm = mul(pm, neg(load_row4<R>(nd.rep, j).ld));
            normalize_me(pm, pe);
        }
    }
    if (threadIdx.x == 0) nodes[node].pp = pp;
}

// per output column: where its rows are and the factors of k_zscale
struct ZCol {
    int64_t row0;  // first row of the node's block in T
    int32_t n;     // rows of the block
    int32_t r;     // twist index (rows <= r use cF, rows > r use cB)
    double cF, cB; // z_i = Z_i * cF (i <= r), z_k = Z_k * cB (k > r)
    double ss;     // ||z||^2 of the written column (compensated sums, scaled by cF, cB)
};

// Normalise each column: Z <- Z c / ||z|| (one read, one write of the block; ||z||^2 was
// accumulated by k_rqi while writing).  Grid-stride over (column, chunk of ZS_CHUNK rows);
// 16-byte vector accesses (4 per thread in flight) when the column segment is aligned.
constexpr int ZS_TPB = 256;
template <class OutT>
__global__ void __launch_bounds__(ZS_TPB) k_zscale(OutT *Z, int64_t ldz, int64_t ncols,
                                                 const ZCol *__restrict__ zc, int64_t maxn) {
    constexpr int V = 16 / sizeof(OutT);                  // elements per 16-byte vector
    constexpr int64_t CHUNK = (int64_t)ZS_TPB * 4 * V;    // rows per work unit
    using Vec = typename std::conditional<sizeof(OutT) == 8, double2, float4>::type;
    const int64_t per_col = (maxn + CHUNK - 1) / CHUNK;
    const int64_t total = ncols * per_col;
    for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
        const int64_t c = w / per_col, ch = w - c * per_col;
        const ZCol z = zc[c];
        const int64_t i0 = ch * CHUNK;
        if (z.n <= 0 || i0 >= z.n) continue;
        const double inv = 1.0 / sqrt(z.ss);
        const double fF = z.cF * inv, fB = z.cB * inv;
        OutT *col = Z + c * ldz + z.row0;
        const bool aligned = (reinterpret_cast<uintptr_t>(col) & 15) == 0;
        if (aligned && i0 + CHUNK <= z.n) {
            Vec *cv = reinterpret_cast<Vec *>(col + i0);
            Vec v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) v[u] = cv[threadIdx.x + u * ZS_TPB];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int64_t b = i0 + (int64_t)(threadIdx.x + u * ZS_TPB) * V;
                OutT *e = reinterpret_cast<OutT *>(&v[u]);
#pragma unroll
                for (int q = 0; q < V; q++) e[q] = (OutT)((double)e[q] * (b + q <= z.r ? fF : fB));
                cv[threadIdx.x + u * ZS_TPB] = v[u];
            }
        } else {  // ragged tail or misaligned segment: element-wise
            for (int64_t i = i0 + threadIdx.x; i < min(i0 + CHUNK, (int64_t)z.n); i += ZS_TPB)
                col[i] = (OutT)((double)col[i] * (i <= z.r ? fF : fB));
        }
    }
}

}  // namespace mr3
