// k_dense.cuh -- NEXT-4: the dense symmetric pipeline around the tridiagonal solver
// (Fig. 3: reduction to tridiagonal form, the mixed-precision
// tridiagonal eigensolver, back-transformation).
//
// Reduction A = Q T Q^T by Householder reflectors H_j = I - tau_j v_j v_j^T (the lower form of
// LAPACK's dsytd2: v_j(j+1) = 1, v_j(j+2:) stored in A(j+2:, j), e_j = A(j+1, j) = beta_j).
// Step j needs column j of A after the rank-2 updates of steps < j; the update of step j is
//   w_j = tau_j A22 v_j,  w_j += -(tau_j / 2) (w_j^T v_j) v_j,  A22 -= v_j w_j^T + w_j v_j^T
// (A22 = A(j+1:, j+1:)).  B200 form: the trailing block is streamed ONCE per step by
// k_sytd_fused, which applies step j-1's rank-2 update to it and, on the updated values,
// forms y_j = A22 v_j (the symmetric matrix-vector product, read down the columns: one warp
// per column, a fixed-order warp reduction, so the bits do not depend on scheduling).  The
// O(n) work between two such sweeps -- finishing w_{j-1} from y_{j-1}, updating column j,
// generating v_j -- is one CTA (k_sytd_col).  Memory: one read + one write of the trailing
// block per step (16 (n - j)^2 bytes), L2-resident once it is below ~126 MB.
// Back-transformation Z <- Q Z = H_0 (H_1 (... Z)) in blocks of DN_NB reflectors,
// H_j0 ... H_j1-1 = I - V T V^T (T from G = V^T V, k_larft), as three library GEMMs each.
#pragma once
#include "kernels.cuh"

namespace mr3 {

constexpr int DN_NB = 64;      // reflectors per back-transformation block
constexpr int DN_COLTPB = 256; // k_sytd_fused: 8 warps, one column each

// fixed-order CTA sum (every thread gets the total)
__device__ __forceinline__ double dn_block_sum(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < nw; i++) t += sh[i];
    return t;
}

// Step j's O(n) part (one CTA): finish w_{j-1} = tau y - (tau/2)(tau y^T v) v from y_{j-1},
// apply step j-1's update to column j, record d_j, and generate the reflector of x = A(j+1:, j)
// (dlarfg: beta = -sign(alpha) ||x||, tau = (beta - alpha) / beta, v = x / (alpha - beta) with
// v(j+1) = 1).  j = n - 1 only finishes the last update and records d_{n-1}.  Each thread
// keeps its rows r = j + tid + 1024 k (k < DN_KE) in registers: one read pass, one write
// pass and two CTA sums per step (the step is on the reduction's critical path).
constexpr int DN_KE = 8;  // rows per thread: n - j <= 8192
__global__ void __launch_bounds__(1024) k_sytd_col(double *A, int64_t lda, int n, int j,
                                                   const double *__restrict__ vprev,
                                                   const double *__restrict__ y, double *w,
                                                   double *vcur, double *tau, double *d,
                                                   double *e) {
    __shared__ double sh[32];
    __shared__ double s_b[3];  // w_{j-1}(j), v_{j-1}(j), alpha = x(j+1)
    double *colj = A + (int64_t)j * lda;
    const int tid = threadIdx.x;
    const double tp = j >= 1 ? tau[j - 1] : 0.0;
    double ck[DN_KE], vk[DN_KE], wk[DN_KE];
#pragma unroll
    for (int k = 0; k < DN_KE; k++) {
        const int r = j + tid + 1024 * k;
        ck[k] = r < n ? colj[r] : 0.0;
        vk[k] = (tp != 0.0 && r < n) ? vprev[r] : 0.0;
        wk[k] = (tp != 0.0 && r < n) ? tp * y[r] : 0.0;
    }
    if (tp != 0.0) {
        double part = 0.0;
#pragma unroll
        for (int k = 0; k < DN_KE; k++) part = fma(wk[k], vk[k], part);
        const double al = -0.5 * tp * dn_block_sum(part, sh);
#pragma unroll
        for (int k = 0; k < DN_KE; k++) {
            const int r = j + tid + 1024 * k;
            wk[k] = fma(al, vk[k], wk[k]);
            if (r < n) w[r] = wk[k];
        }
        if (tid == 0) {
            s_b[0] = wk[0];
            s_b[1] = vk[0];
        }
        __syncthreads();
        const double wj = s_b[0], vj = s_b[1];
#pragma unroll
        for (int k = 0; k < DN_KE; k++) ck[k] = ck[k] - vk[k] * wj - wk[k] * vj;
    }
    if (tid == 0) {
        d[j] = ck[0];
        colj[j] = ck[0];
    }
    if (j > n - 2) return;
    // reflector of x = A(j+1:n, j): alpha = x(j+1) (thread 1's first row), ||x(j+2:)||^2
    if (tid == 1) s_b[2] = ck[0];
    double part = 0.0;
#pragma unroll
    for (int k = 0; k < DN_KE; k++) {
        const int r = j + tid + 1024 * k;
        if (r >= j + 2 && r < n) part = fma(ck[k], ck[k], part);
    }
    const double xn2 = dn_block_sum(part, sh);  // (its barriers publish s_b[2])
    const double alpha = s_b[2];
    const bool id = xn2 == 0.0;  // nothing to annihilate: H = I
    const double beta = id ? alpha : -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
    const double sc = id ? 0.0 : 1.0 / (alpha - beta);
#pragma unroll
    for (int k = 0; k < DN_KE; k++) {
        const int r = j + tid + 1024 * k;
        if (r == j + 1) {
            vcur[r] = 1.0;
            colj[r] = beta;
        } else if (r >= j + 2 && r < n) {
            const double v = ck[k] * sc;
            vcur[r] = v;
            if (!id) colj[r] = v;  // (LAPACK storage of the reflector below the subdiagonal)
        }
    }
    if (tid == 0) {
        tau[j] = id ? 0.0 : (beta - alpha) / beta;
        e[j] = beta;
    }
}

// Step j's O((n - j)^2) part: DN_SEG warps per column c in (j, n), each over one contiguous
// segment of rows r > j: apply step j-1's update (A(r, c) -= v_{j-1}(r) w_{j-1}(c) +
// w_{j-1}(r) v_{j-1}(c)) and, on the updated values, accumulate A(r, c) v_j(r); the segment
// sums are added in a fixed order, y_j(c) = (A22 v_j)(c) by symmetry.  Rows r = j of these
// columns are never read again (row j of the result is e_j, recorded by k_sytd_col).  Several
// warps per column keep enough loads in flight when the trailing block is small.
constexpr int DN_SEG = 4;
constexpr int DN_CPB = DN_COLTPB / 32 / DN_SEG;  // columns per CTA (2)
__global__ void __launch_bounds__(DN_COLTPB) k_sytd_fused(double *A, int64_t lda, int n, int j,
                                                          const double *__restrict__ vprev,
                                                          const double *__restrict__ wprev,
                                                          const double *__restrict__ v,
                                                          const double *__restrict__ tau,
                                                          double *y) {
    __shared__ double part[DN_COLTPB / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = warp % DN_SEG;
    const int c = j + 1 + blockIdx.x * DN_CPB + warp / DN_SEG;
    const bool upd = j >= 1 && tau[j - 1] != 0.0;
    const int r0 = j + 1, m = n - r0;
    // segment rows [s0, s1): multiples of 32 rows so every warp load is one aligned run
    const int per = ((m + DN_SEG - 1) / DN_SEG + 31) & ~31;
    const int s0 = r0 + seg * per, s1 = min(n, s0 + per);
    double acc = 0.0;
    if (c < n) {
        double *col = A + (int64_t)c * lda;
        if (upd) {
            const double wc = wprev[c], vc = vprev[c];
#pragma unroll 4
            for (int r = s0 + lane; r < s1; r += 32) {
                const double a = col[r] - vprev[r] * wc - wprev[r] * vc;
                col[r] = a;
                acc = fma(a, v[r], acc);
            }
        } else {
#pragma unroll 4
            for (int r = s0 + lane; r < s1; r += 32) acc = fma(col[r], v[r], acc);
        }
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    if (seg == 0 && lane == 0 && c < n) {
        double t = 0.0;
        for (int q = 0; q < DN_SEG; q++) t += part[warp + q];
        y[c] = t;
    }
}

// V of reflectors j0 .. j0 + kb - 1 as an explicit (n - j0 - 1) x kb column-major matrix
// (rows j0 + 1 .. n - 1): zeros above the unit diagonal, the stored entries below
__global__ void k_build_v(const double *__restrict__ A, int64_t lda, int n, int j0, int kb,
                          double *V, int64_t ldv) {
    const int m = n - j0 - 1;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)m * kb) return;
    const int k = (int)(t / m), i = (int)(t % m);
    const int r = j0 + 1 + i, jr = j0 + k;  // row of A, reflector index
    double v;
    if (r < jr + 1)
        v = 0.0;
    else if (r == jr + 1)
        v = 1.0;
    else
        v = A[r + (int64_t)jr * lda];
    V[i + (int64_t)k * ldv] = v;
}

// dlarft (forward, columnwise): T upper triangular with H_j0 ... H_j0+kb-1 = I - V T V^T;
// T(k, k) = tau_k, T(0:k, k) = -tau_k T(0:k, 0:k) (V(:, 0:k)^T v_k), V^T V = G given.
// One CTA of kb threads; T column-major kb x kb.
__global__ void k_larft(const double *__restrict__ G, int kb, const double *__restrict__ tau, int j0,
                        double *T) {
    const int i = threadIdx.x;
    for (int q = i; q < kb * kb; q += blockDim.x) T[q] = 0.0;
    __syncthreads();
    for (int k = 0; k < kb; k++) {
        const double tk = tau[j0 + k];
        double t = 0.0;
        if (i < k)
            for (int l = i; l < k; l++) t += T[i + l * kb] * G[l + k * kb];
        __syncthreads();
        if (i < k) T[i + k * kb] = -tk * t;
        if (i == k) T[k + k * kb] = tk;
        __syncthreads();
    }
}

// max |A_ij| over the n x n matrix (bits of a non-negative double order as integers); NaN/inf
// entries set the maximum to inf (the tridiagonal solver reports them)
__global__ void k_dense_absmax(const double *__restrict__ A, int64_t lda, int n,
                               unsigned long long *out) {
    unsigned long long m = 0;
    const int64_t tot = (int64_t)n * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const double v = fabs(A[(t / n) * lda + (t % n)]);
        const unsigned long long u =
            (v == v) ? (unsigned long long)__double_as_longlong(v) : 0x7ff0000000000000ULL;
        m = u > m ? u : m;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
        m = x > m ? x : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
// A <- sc A (sc a power of 2: exact unless an entry becomes subnormal) / w <- sc w
__global__ void k_dense_scale(double *A, int64_t lda, int n, double sc) {
    const int64_t tot = (int64_t)n * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x)
        A[(t / n) * lda + (t % n)] *= sc;
}
__global__ void k_vec_scale(double *w, int64_t m, double sc) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) w[t] *= sc;
}

}  // namespace mr3
