// kernels.cuh -- device side of the hot path (K1..K7 of DESIGN.md).
//
// Every kernel is a template over the internal precision R (dd for fp64 I/O,
// double for fp32 I/O).  Representations are N-representations of lower
// bidiagonal factorizations LDL^T,
// stored row-major per row j as {d_j, lld_j, l_j, ld_j} (ld = d*l, lld = d*l^2
// are derived data, L405-L409).  All threads of a warp normally share one
// representation, so the per-row loads are warp-uniform broadcasts served by L1.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dd.cuh"

namespace mr3 {

struct NodeInfo {
    const double *rep;  // rows of 4 R values {d, lld, l, ld}
    int64_t n;          // rows (irreducible block size)
    int64_t row0;       // first row of the block in T
    double sig_hi, sig_lo;  // accumulated shift sigma (scaled units), Alg.1 l.19/29
    int32_t depth;
    int32_t block;
};

struct Items {  // eigenvalue slots, SoA over the requested index set (+ guards)
    int32_t *node;
    int32_t *k;      // block-local eigenvalue index, 1-based
    int64_t *col;    // output column (global), -1 = guard / not wanted
    void *lo, *hi;   // R brackets [lo, hi] in node coordinates
    double *lgap, *rgap;  // absolute gaps to the neighbours (node coordinates)
};

struct DevStats {
    unsigned long long bisect_rows;
    unsigned long long rqi_rows;
    int rqi_fallbacks;
    int rqi_iters_max;
    int robustness_failures;
    int largest_cluster;
    int n_clusters;
    int pad;
};

template <class R>
struct Row2 {
    R d, lld;
};
template <class R>
struct Row4 {
    R d, lld, l, ld;
};

__device__ __forceinline__ void ld2(const double *p, double &a, double &b) {
    double2 v = __ldg(reinterpret_cast<const double2 *>(p));
    a = v.x;
    b = v.y;
}

template <class R>
__device__ __forceinline__ Row2<R> load_row2(const double *rep, int64_t k);
template <>
__device__ __forceinline__ Row2<dd> load_row2<dd>(const double *rep, int64_t k) {
    Row2<dd> r;
    ld2(rep + 8 * k, r.d.hi, r.d.lo);
    ld2(rep + 8 * k + 2, r.lld.hi, r.lld.lo);
    return r;
}
template <>
__device__ __forceinline__ Row2<double> load_row2<double>(const double *rep, int64_t k) {
    Row2<double> r;
    ld2(rep + 4 * k, r.d, r.lld);
    return r;
}
template <class R>
__device__ __forceinline__ Row4<R> load_row4(const double *rep, int64_t k);
template <>
__device__ __forceinline__ Row4<dd> load_row4<dd>(const double *rep, int64_t k) {
    Row4<dd> r;
    ld2(rep + 8 * k, r.d.hi, r.d.lo);
    ld2(rep + 8 * k + 2, r.lld.hi, r.lld.lo);
    ld2(rep + 8 * k + 4, r.l.hi, r.l.lo);
    ld2(rep + 8 * k + 6, r.ld.hi, r.ld.lo);
    return r;
}
template <>
__device__ __forceinline__ Row4<double> load_row4<double>(const double *rep, int64_t k) {
    Row4<double> r;
    ld2(rep + 4 * k, r.d, r.lld);
    ld2(rep + 4 * k + 2, r.l, r.ld);
    return r;
}
template <class R>
__device__ __forceinline__ void store_row4(double *rep, int64_t k, R d, R lld, R l, R ld);
template <>
__device__ __forceinline__ void store_row4<dd>(double *rep, int64_t k, dd d, dd lld, dd l, dd ld) {
    double *p = rep + 8 * k;
    reinterpret_cast<double2 *>(p)[0] = make_double2(d.hi, d.lo);
    reinterpret_cast<double2 *>(p)[1] = make_double2(lld.hi, lld.lo);
    reinterpret_cast<double2 *>(p)[2] = make_double2(l.hi, l.lo);
    reinterpret_cast<double2 *>(p)[3] = make_double2(ld.hi, ld.lo);
}
template <>
__device__ __forceinline__ void store_row4<double>(double *rep, int64_t k, double d, double lld,
                                                   double l, double ld) {
    double *p = rep + 4 * k;
    reinterpret_cast<double2 *>(p)[0] = make_double2(d, lld);
    reinterpret_cast<double2 *>(p)[1] = make_double2(l, ld);
}

// pivot guard: |x| < pivmin -> -pivmin, so no +-inf ever reaches
// an error-free transform and the count treats the pivot as negative.
template <class R>
__device__ __forceinline__ R guard(R x, double pivmin) {
    return (fabs(hi(x)) < pivmin) ? mk<R>(-pivmin) : x;
}

// ---------------------------------------------------------------------------
// negcount(M, x) = #{eigenvalues of M = LDL^T below x} = #{j : d+_j < 0} of the
// stationary qd transform L+D+L+^T = LDL^T - xI (dstqds):
//   s_1 = -x ; d+_j = d_j + s_j ; s_{j+1} = lld_j * (s_j / d+_j) - x
// ("special forms of ... qd"; Sturm count S:182-188).
// ---------------------------------------------------------------------------
template <class R>
__device__ __forceinline__ int negcount(const double *__restrict__ rep, int64_t n, R x,
                                        double pivmin) {
    R s = neg(x);
    int cnt = 0;
    int64_t j = 0;
    Row2<R> cur = load_row2<R>(rep, 0);
#pragma unroll 1
    for (; j < n - 1; j++) {
        Row2<R> nxt = load_row2<R>(rep, j + 1);  // prefetch one row ahead
        R dp = guard(add(cur.d, s), pivmin);
        cnt += is_neg(dp) ? 1 : 0;
        s = sub(mul(cur.lld, div(s, dp)), x);
        cur = nxt;
    }
    R dp = guard(add(cur.d, s), pivmin);
    cnt += is_neg(dp) ? 1 : 0;
    return cnt;
}

// two shifts through the same rows (ILP 2)
template <class R>
__device__ __forceinline__ void negcount2(const double *__restrict__ rep, int64_t n, R x0, R x1,
                                          double pivmin, int &c0, int &c1) {
    R s0 = neg(x0), s1 = neg(x1);
    c0 = 0;
    c1 = 0;
    Row2<R> cur = load_row2<R>(rep, 0);
#pragma unroll 1
    for (int64_t j = 0; j < n - 1; j++) {
        Row2<R> nxt = load_row2<R>(rep, j + 1);
        R dp0 = guard(add(cur.d, s0), pivmin);
        R dp1 = guard(add(cur.d, s1), pivmin);
        c0 += is_neg(dp0) ? 1 : 0;
        c1 += is_neg(dp1) ? 1 : 0;
        s0 = sub(mul(cur.lld, div(s0, dp0)), x0);
        s1 = sub(mul(cur.lld, div(s1, dp1)), x1);
        cur = nxt;
    }
    R dp0 = guard(add(cur.d, s0), pivmin);
    R dp1 = guard(add(cur.d, s1), pivmin);
    c0 += is_neg(dp0) ? 1 : 0;
    c1 += is_neg(dp1) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// counter-based generator for the root perturbation (PAPER.md L901-L909,
// footnote: "any (fixed) sequence of pseudo-random numbers can be used"):
// u in [-1, 1] keyed by (seed, global row, field); independent of launch shape.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double uniform_pm1(uint64_t seed, uint64_t row, uint64_t field) {
    uint64_t z = mix64(seed ^ mix64(row * 2 + field));
    return (double)(z >> 11) * 0x1.0p-52 - 1.0;  // [-1, 1)
}

// ---------------------------------------------------------------------------
// K1a: ||T||_1, Gershgorin bounds, finiteness, split count (one CTA).
// ---------------------------------------------------------------------------
struct ScanInfo {
    double norm1, gl, gu;
    int nonfinite;
    int pad;
    long long nsplit;
};

template <class T>
__global__ void k_scan_input(const T *__restrict__ d, const T *__restrict__ e, int64_t n,
                             ScanInfo *out) {
    __shared__ double s_norm[32], s_gl[32], s_gu[32];
    __shared__ int s_bad[32];
    double nrm = 0.0, gl = INFINITY, gu = -INFINITY;
    int bad = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double di = (double)d[i];
        double el = i > 0 ? fabs((double)e[i - 1]) : 0.0;
        double er = i < n - 1 ? fabs((double)e[i]) : 0.0;
        if (!isfinite(di) || !isfinite(el) || !isfinite(er)) bad = 1;
        double r = el + er;
        nrm = fmax(nrm, fabs(di) + r);
        gl = fmin(gl, di - r);
        gu = fmax(gu, di + r);
    }
    for (int o = 16; o > 0; o >>= 1) {
        nrm = fmax(nrm, __shfl_xor_sync(0xffffffff, nrm, o));
        gl = fmin(gl, __shfl_xor_sync(0xffffffff, gl, o));
        gu = fmax(gu, __shfl_xor_sync(0xffffffff, gu, o));
        bad |= __shfl_xor_sync(0xffffffff, bad, o);
    }
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        s_norm[w] = nrm;
        s_gl[w] = gl;
        s_gu[w] = gu;
        s_bad[w] = bad;
    }
    __syncthreads();
    if (w == 0) {
        int nw = blockDim.x >> 5;
        nrm = l < nw ? s_norm[l] : 0.0;
        gl = l < nw ? s_gl[l] : INFINITY;
        gu = l < nw ? s_gu[l] : -INFINITY;
        bad = l < nw ? s_bad[l] : 0;
        for (int o = 16; o > 0; o >>= 1) {
            nrm = fmax(nrm, __shfl_xor_sync(0xffffffff, nrm, o));
            gl = fmin(gl, __shfl_xor_sync(0xffffffff, gl, o));
            gu = fmax(gu, __shfl_xor_sync(0xffffffff, gu, o));
            bad |= __shfl_xor_sync(0xffffffff, bad, o);
        }
        if (l == 0) {
            out->norm1 = nrm;
            out->gl = gl;
            out->gu = gu;
            out->nonfinite = bad;
        }
    }
    __syncthreads();
    // split count with the threshold written by the host into out->nsplit's slot? no:
    // splitting is evaluated by k_split_flags once ||T||_1 is known.
}

// |e_i| <= thr  (|e_i| <= eps_x ||T||) -> split after row i
template <class T>
__global__ void k_split_count(const T *__restrict__ e, int64_t n, double thr,
                              unsigned long long *cnt) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n - 1;
         i += (int64_t)gridDim.x * blockDim.x)
        if (fabs((double)e[i]) <= thr) c++;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffff, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

template <class T>
__global__ void k_split_list(const T *__restrict__ e, int64_t n, double thr, int64_t *pos,
                             unsigned long long *cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n - 1;
         i += (int64_t)gridDim.x * blockDim.x)
        if (fabs((double)e[i]) <= thr) pos[atomicAdd(cnt, 1ULL)] = i;
}

// ---------------------------------------------------------------------------
// K1b: root representation, one thread per irreducible block (Alg. 1 l.1-2).
// mu just outside the Gershgorin interval of the block (left: all d > 0,
// right: all d < 0: a definite LDL^T, L1022-L1025), then
//   d_1 = a_1 - mu ; l_i = e_i / d_i ; d_{i+1} = (a_{i+1} - mu) - l_i e_i
// in R, the random relative perturbation x <- x (1 + xi u) of all 2n-1 data
// (L901-L909), derived ld, lld, and certified root brackets.
// ---------------------------------------------------------------------------
struct BlockDesc {
    int64_t row0, n;
};

template <class R, class T>
__global__ void k_root(const T *__restrict__ d, const T *__restrict__ e, const BlockDesc *blocks,
                       int nblocks, double scale, int right_side, double xi, uint64_t seed,
                       double pivmin, double *rep_pool, int64_t rep_stride_rows,
                       NodeInfo *nodes, double *brk /* per block: lo(R) hi(R) as 4 doubles */,
                       int *fail) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    const int64_t r0 = blocks[b].row0, n = blocks[b].n;
    double *rep = rep_pool + r0 * 4 * Prec<R>::words;  // blocks own disjoint rows
    (void)rep_stride_rows;
    // block Gershgorin (scaled)
    double gl = INFINITY, gu = -INFINITY, nrm = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double di = (double)d[r0 + i] * scale;
        double r = (i > 0 ? fabs((double)e[r0 + i - 1]) * scale : 0.0) +
                   (i < n - 1 ? fabs((double)e[r0 + i]) * scale : 0.0);
        gl = fmin(gl, di - r);
        gu = fmax(gu, di + r);
        nrm = fmax(nrm, fabs(di) + r);
    }
    double pad = 4.0 * 1.1102230246251565e-16 * fmax(fmax(fabs(gl), fabs(gu)), nrm) + pivmin;
    bool right = right_side != 0;
    double mu = 0.0;
    bool ok = false;
    for (int attempt = 0; attempt < 40 && !ok; attempt++) {
        mu = right ? gu + pad : gl - pad;
        ok = true;
        // factor T_b - mu I
        R dcur = sub(mk<R>((double)d[r0] * scale), mk<R>(mu));
        for (int64_t i = 0; i < n; i++) {
            bool good = right ? (hi(dcur) < 0.0) : (hi(dcur) > 0.0);
            if (!good || !isfinite(hi(dcur))) {
                ok = false;
                break;
            }
            R li = mk<R>(0.0);
            R dnext = mk<R>(0.0);
            if (i < n - 1) {
                double ei = (double)e[r0 + i] * scale;
                li = div(mk<R>(ei), dcur);
                R a = sub(mk<R>((double)d[r0 + i + 1] * scale), mk<R>(mu));
                dnext = sub(a, mul(li, ei));
            }
            // perturb the data d_i, l_i (global row index keys the generator)
            uint64_t grow = (uint64_t)(r0 + i);
            R dp = mul(dcur, mk<R>(1.0));
            {
                double u = uniform_pm1(seed, grow, 0);
                dp = add(dcur, mul(dcur, xi * u));
            }
            R lp = li;
            if (i < n - 1) {
                double u = uniform_pm1(seed, grow, 1);
                lp = add(li, mul(li, xi * u));
            }
            R ldv = mul(dp, lp);
            R lldv = mul(ldv, lp);
            store_row4<R>(rep, i, dp, lldv, lp, ldv);
            dcur = dnext;
        }
        pad *= 16.0;
    }
    if (!ok) atomicExch(fail, 1);
    NodeInfo ni;
    ni.rep = rep;
    ni.n = n;
    ni.row0 = r0;
    ni.sig_hi = mu;
    ni.sig_lo = 0.0;
    ni.depth = 0;
    ni.block = b;
    nodes[b] = ni;
    // certified bracket for all eigenvalues of the block in root coordinates
    double span = gu - gl;
    double lo = right ? (gl - mu) - pad - 1e-3 * span : -pad;
    double hiv = right ? pad : (gu - mu) + pad + 1e-3 * span;
    if (!right) lo = -fmax(pad, pivmin * 4.0);
    for (int it = 0; it < 60; it++) {
        int c = negcount<R>(rep, n, mk<R>(lo), pivmin);
        if (c == 0) break;
        lo -= fmax(span, 1.0) * (double)(1 << (it < 20 ? it : 20));
    }
    for (int it = 0; it < 60; it++) {
        int c = negcount<R>(rep, n, mk<R>(hiv), pivmin);
        if (c == n) break;
        hiv += fmax(span, 1.0) * (double)(1 << (it < 20 ? it : 20));
    }
    brk[4 * b + 0] = lo;
    brk[4 * b + 1] = 0.0;
    brk[4 * b + 2] = hiv;
    brk[4 * b + 3] = 0.0;
}

// counts of the root at two shifts (value range -> index range)
template <class R>
__global__ void k_count_at(const NodeInfo *nodes, int node, double x0, double x1, double pivmin,
                           int *out) {
    const NodeInfo nd = nodes[node];
    int c0, c1;
    if (threadIdx.x == 0) {
        c0 = negcount<R>(nd.rep, nd.n, sub(mk<R>(x0), mk2<R>(nd.sig_hi, nd.sig_lo)), pivmin);
        out[0] = c0;
    } else if (threadIdx.x == 1) {
        c1 = negcount<R>(nd.rep, nd.n, sub(mk<R>(x1), mk2<R>(nd.sig_hi, nd.sig_lo)), pivmin);
        out[1] = c1;
    }
}

}  // namespace mr3
