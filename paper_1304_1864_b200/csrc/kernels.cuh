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
    const double *repx; // M_x: {d, lld} rounded to binary64, 2 per row
    int64_t n;          // rows (irreducible block size)
    int64_t row0;       // first row of the block in T
    double sig_hi, sig_lo;  // accumulated shift sigma (scaled units), Alg.1 l.19/29
    int32_t depth;
    int32_t block;
    int32_t parent;     // node this one was shifted from (-1: a root), for backtracking (R22)
    int32_t pad_;
    const double *pp;   // per row {PP, 1/PP, exponent} of prod_{j<k} (-ld_j) (k_zprod.cuh)
};

struct Items {  // eigenvalue slots, SoA over the requested index set (+ guards)
    int32_t *node;
    int32_t *k;      // block-local eigenvalue index, 1-based
    int64_t *col;    // output column (global), -1 = guard / not wanted
    void *lo, *hi;   // R brackets [lo, hi] in node coordinates
    double *lgap, *rgap;  // absolute gaps to the neighbours (node coordinates)
    double *x0;           // RQI starting point (binary64, node coordinates) or NaN: midpoint
    double *dx;           // |last Newton step| of the root binary_x phase behind x0 (INF: none)
    int32_t *twist;       // RQI twist index r (0-based row of the node), from k_rqi_locate
};

// CTA task: a run of consecutive list entries (items of ONE node) for the kernels
// that stage that node's rows through shared memory (k_bisect_s, k_rqi*)
struct RqiTask {
    int32_t first;  // offset into the item list
    int32_t cnt;    // items in this CTA
    int32_t node;
    int32_t pad;
};

struct DevStats {
    unsigned long long bisect_rows;    // binary_y Sturm rows
    unsigned long long bisect_rows_x;  // binary_x Sturm rows (fp64 phase)
    unsigned long long newton_rows_x;  // binary_x rows of Newton passes (subset of bisect_rows_x)
    // ---- fields above are plan-phase counters; execute resets from rqi_rows on
    unsigned long long rqi_rows;
    int rqi_fallbacks;
    int rqi_iters_max;
    int robustness_failures;
    int largest_cluster;
    int n_clusters;
    int pad;
    unsigned long long refine_rows_x;  // binary_x rows of the RQI start refinement (K2')
    int backtracks;       // clusters whose child was taken from the grandparent (R22)
    int backtrack_tries;  // clusters re-processed from the grandparent
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
constexpr int PFY = 2;  // binary_y rows prefetched ahead (32 B each)

template <class R>
__device__ __forceinline__ int negcount(const double *__restrict__ rep, int64_t n, R x,
                                        double pivmin) {
    R s = neg(x);
    int cnt = 0;
    Row2<R> ring[PFY];
#pragma unroll
    for (int u = 0; u < PFY; u++) ring[u] = load_row2<R>(rep, u < n ? u : n - 1);
    int64_t j = 0;
#pragma unroll 1
    for (; j + PFY <= n - 1; j += PFY) {
#pragma unroll
        for (int u = 0; u < PFY; u++) {
            Row2<R> cur = ring[u];
            int64_t nx = j + u + PFY;
            ring[u] = load_row2<R>(rep, nx < n ? nx : n - 1);
            R dp = guard(add(cur.d, s), pivmin);
            cnt += is_neg(dp) ? 1 : 0;
            s = sub(mul(cur.lld, div(s, dp)), x);
        }
    }
    // tail rows j .. n-2 (fewer than PFY), then the last pivot
#pragma unroll
    for (int u = 0; u < PFY; u++) {
        if (j + u < n - 1) {
            Row2<R> cur = ring[u];
            R dp = guard(add(cur.d, s), pivmin);
            cnt += is_neg(dp) ? 1 : 0;
            s = sub(mul(cur.lld, div(s, dp)), x);
        }
    }
    Row2<R> last = load_row2<R>(rep, n - 1);
    R dp = guard(add(last.d, s), pivmin);
    cnt += is_neg(dp) ? 1 : 0;
    return cnt;
}

// negcount in binary_x arithmetic on the narrowed copy M_x (§3.2,
// "Arithmetic used to approximate eigenvalues", L1064-L1111), in projective
// (division-free) form.  With s_j = p_j / q_j the dstqds step
//   d+_j = d_j + s_j ,  s_{j+1} = lld_j s_j / d+_j - x
// becomes  D_j = d_j q_j + p_j  (= d+_j q_j),  q_{j+1} = D_j,  p_{j+1} = lld_j p_j - x D_j,
// and d+_j < 0  <=>  sign(D_j) != sign(q_j).  Per row: two FMAs and one MUL, no
// reciprocal, and a dependent chain of two FMAs.  (p, q) is rescaled by a power of
// two every XB rows (exact); a non-finite state (overflow; unreachable for XB = 8
// unless |lld| > 1e38) redoes the block in the guarded ratio form.  A zero pivot
// needs no guard: D_j = 0 makes q_{j+1} = 0 and s_{j+1} = +-inf, which the next
// row absorbs exactly as IEEE arithmetic on the ratio form would.  The binary_x
// counts only steer the search: every bracket is certified by binary_y (dstqds)
// counts afterwards (k_bisect XPHASE), so this form needs no stability argument
// of its own beyond producing counts of a nearby matrix.
// The rows are read with a prefetch distance of XB rows; repx arrays carry XPAD
// padding rows beyond the last row so the prefetch never needs a bound check.
__device__ __forceinline__ int sign_bit(double v) {
    return (int)((unsigned)__double2hiint(v) >> 31);
}
__device__ __forceinline__ void nc_row_guarded(double d, double lld, double x, double pivmin,
                                               double &s, int &cnt) {
    double dp = d + s;
    dp = fabs(dp) < pivmin ? -pivmin : dp;
    cnt += dp < 0.0 ? 1 : 0;
    s = fma_rn(lld * s, rcp(dp), -x);
}
constexpr int XB = 8;    // rows per block (prefetch distance, rescale period)
constexpr int XPAD = 8;  // padding rows after every binary_x representation
__device__ __forceinline__ void xrow(const double2 r, const double x, double &p, double &q,
                                     unsigned &c) {
    const double D = fma_rn(r.x, q, p);
    c += (unsigned)(__double2hiint(D) ^ __double2hiint(q)) >> 31;
    p = fma_rn(-x, D, mul_rn(r.y, p));
    q = D;
}
__device__ __forceinline__ int negcount_x(const double *__restrict__ repx, int64_t n, double x,
                                          double pivmin) {
    const double2 *rx = reinterpret_cast<const double2 *>(repx);
    double p = -x, q = 1.0;
    unsigned c = 0;
    int64_t j = 0;
    if (n - 1 >= XB) {
        double2 r0 = __ldg(rx + 0), r1 = __ldg(rx + 1), r2 = __ldg(rx + 2), r3 = __ldg(rx + 3),
                r4 = __ldg(rx + 4), r5 = __ldg(rx + 5), r6 = __ldg(rx + 6), r7 = __ldg(rx + 7);
#pragma unroll 1
        for (; j + XB <= n - 1; j += XB) {
            const double p0 = p, q0 = q;
            const unsigned c0 = c;
            const double2 *nx = rx + j + XB;
            xrow(r0, x, p, q, c); r0 = __ldg(nx + 0);
            xrow(r1, x, p, q, c); r1 = __ldg(nx + 1);
            xrow(r2, x, p, q, c); r2 = __ldg(nx + 2);
            xrow(r3, x, p, q, c); r3 = __ldg(nx + 3);
            xrow(r4, x, p, q, c); r4 = __ldg(nx + 4);
            xrow(r5, x, p, q, c); r5 = __ldg(nx + 5);
            xrow(r6, x, p, q, c); r6 = __ldg(nx + 6);
            xrow(r7, x, p, q, c); r7 = __ldg(nx + 7);
            const unsigned ep = (unsigned)__double2hiint(p) & 0x7ff00000u;
            const unsigned eq = (unsigned)__double2hiint(q) & 0x7ff00000u;
            const unsigned em = ep > eq ? ep : eq;
            if (em == 0x7ff00000u) {  // overflow: redo the block in the guarded ratio form
                double s = p0 / q0;
                if (!(fabs(s) <= 1e300)) s = copysign(1e300, s);
                int cc = 0;
                for (int u = 0; u < XB; u++) {
                    const double2 r = __ldg(rx + j + u);
                    nc_row_guarded(r.x, r.y, x, pivmin, s, cc);
                }
                c = c0 + (unsigned)cc;
                p = s;
                q = 1.0;
            } else {  // exact power-of-two rescale to max exponent 2^0
                const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                p = mul_rn(p, sc);
                q = mul_rn(q, sc);
            }
        }
    }
#pragma unroll 1
    for (; j < n - 1; j++) xrow(__ldg(rx + j), x, p, q, c);  // fewer than XB rows
    const double D = fma_rn(__ldg(rx + (n - 1)).x, q, p);
    c += (unsigned)(__double2hiint(D) ^ __double2hiint(q)) >> 31;
    return (int)c;
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
// K1b: root representations (Alg. 1 l.1-2), chunk-parallel.
//
// mu just outside the Gershgorin interval of each block (left: T - mu I positive
// definite, all d > 0; right: negative definite; L1022-L1025), then the LDL^T of
// T - mu I: d_1 = c_1, d_{r} = c_r - e_{r-1}^2 / d_{r-1}, l_r = e_r / d_r, with
// c_r = a_r - mu.  The pivot recurrence is a continued fraction: with the state
// (p, q) (d_{r-1} = p/q) row r maps it by A_r = [[c_r, -e_{r-1}^2], [1, 0]].
// Chunks of RT_CH rows form their transfer matrices in R (k_root_chunkmat), one
// thread per block scans them (k_root_scan), and every chunk then runs the
// plain recurrence from its incoming pivot (k_root_factor).  The incoming pivot
// of a chunk differs from the sequential one only by the rounding of the 2x2
// products (relative ~ eps_y * O(n)), i.e. a relative perturbation of T far
// below the xi = eps_x perturbation that follows (reading R3).
// Then every datum d_i, l_i is perturbed x <- x (1 + xi u) (L901-L909), and the
// derived ld = d l, lld = d l^2 are formed.  A 1x1 block is left unperturbed
// (its eigenvalue is exactly d).
// ---------------------------------------------------------------------------
struct BlockDesc {
    int64_t row0, n;
};
struct ChunkDesc {
    int64_t row0;   // first row (global)
    int32_t len;    // rows in the chunk
    int32_t block;  // owning block
};
constexpr int RT_CH = 32;

template <class R>
struct Mat2 {
    R a, b, c, d;
};

template <class R>
__device__ __forceinline__ R scale2(R x, int e) {
    return mk2<R>(ldexp(hi(x), e), ldexp(lo_part(x), e));
}

template <class R, class T>
__global__ void k_root_gersh(const T *__restrict__ d, const T *__restrict__ e,
                             const BlockDesc *blocks, double scale, int right, double padmul,
                             double pivmin, double *mu_out, double *brk) {
    const int b = blockIdx.x;
    const int64_t r0 = blocks[b].row0, n = blocks[b].n;
    __shared__ double sg[32], su[32], sn[32];
    double gl = INFINITY, gu = -INFINITY, nrm = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double di = (double)d[r0 + i] * scale;
        double r = (i > 0 ? fabs((double)e[r0 + i - 1]) * scale : 0.0) +
                   (i < n - 1 ? fabs((double)e[r0 + i]) * scale : 0.0);
        gl = fmin(gl, di - r);
        gu = fmax(gu, di + r);
        nrm = fmax(nrm, fabs(di) + r);
    }
    for (int o = 16; o > 0; o >>= 1) {
        gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
        gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
        nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sg[w] = gl;
        su[w] = gu;
        sn[w] = nrm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); i++) {
            gl = fmin(gl, sg[i]);
            gu = fmax(gu, su[i]);
            nrm = fmax(nrm, sn[i]);
        }
        double pad = (4.0 * 1.1102230246251565e-16 * fmax(fmax(fabs(gl), fabs(gu)), nrm) + pivmin) *
                     padmul;
        double mu = right ? gu + pad : gl - pad;
        mu_out[b] = mu;
        // certified enclosure of the root's eigenvalues: the data are perturbed by
        // at most (1 + xi)^(2n) ~ 1 + 2 n xi relative, far inside the 1e-3 margin
        double lo, hi_;
        if (right) {
            lo = (gl - mu) * (1.0 + 1e-3) - pad;
            hi_ = 0.0;
        } else {
            lo = 0.0;
            hi_ = (gu - mu) * (1.0 + 1e-3) + pad;
        }
        brk[4 * b + 0] = lo;
        brk[4 * b + 1] = 0.0;
        brk[4 * b + 2] = hi_;
        brk[4 * b + 3] = 0.0;
    }
}

template <class R>
__device__ __forceinline__ R shifted_diag(double dv, double mu) {  // c = d - mu, exact in dd
    return sub(mk<R>(dv), mk<R>(mu));
}

template <class R, class T>
__global__ void k_root_chunkmat(const T *__restrict__ d, const T *__restrict__ e,
                                const ChunkDesc *chunks, int nch, const BlockDesc *blocks,
                                double scale, const double *mu, Mat2<R> *mats) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nch) return;
    const ChunkDesc ch = chunks[k];
    const int64_t b0 = blocks[ch.block].row0;
    const double m = mu[ch.block];
    Mat2<R> M;
    M.a = mk<R>(1.0);
    M.b = mk<R>(0.0);
    M.c = mk<R>(0.0);
    M.d = mk<R>(1.0);
    for (int j = 0; j < ch.len; j++) {
        const int64_t r = ch.row0 + j;
        R c = shifted_diag<R>((double)d[r] * scale, m);
        R na, nb;
        if (r > b0) {
            double ev = (double)e[r - 1] * scale;
            R e2 = mul(mk<R>(ev), ev);
            na = sub(mul(c, M.a), mul(e2, M.c));
            nb = sub(mul(c, M.b), mul(e2, M.d));
        } else {
            na = mul(c, M.a);
            nb = mul(c, M.b);
        }
        M.c = M.a;
        M.d = M.b;
        M.a = na;
        M.b = nb;
        if ((j & 7) == 7 || j == ch.len - 1) {  // projective: rescale by a power of 2
            double mx = fmax(fmax(fabs(hi(M.a)), fabs(hi(M.b))), fmax(fabs(hi(M.c)), fabs(hi(M.d))));
            int ex = 0;
            if (mx > 0) frexp(mx, &ex);
            M.a = scale2(M.a, -ex);
            M.b = scale2(M.b, -ex);
            M.c = scale2(M.c, -ex);
            M.d = scale2(M.d, -ex);
        }
    }
    mats[k] = M;
}

// incoming state of every chunk ((p, q) = (1, 0) at the top of the block): one CTA per
// block; each thread composes the transfer matrices of a run of chunks, a Hillis-Steele
// scan composes the runs (matrix products are associative; later chunks multiply from
// the left), and each thread then walks its run from the composed incoming state.
// Every product is rescaled by a power of two (the state is projective).
template <class R>
__device__ __forceinline__ Mat2<R> mat_mul(const Mat2<R> &X, const Mat2<R> &Y) {  // X * Y
    Mat2<R> Z;
    Z.a = add(mul(X.a, Y.a), mul(X.b, Y.c));
    Z.b = add(mul(X.a, Y.b), mul(X.b, Y.d));
    Z.c = add(mul(X.c, Y.a), mul(X.d, Y.c));
    Z.d = add(mul(X.c, Y.b), mul(X.d, Y.d));
    double mx = fmax(fmax(fabs(hi(Z.a)), fabs(hi(Z.b))), fmax(fabs(hi(Z.c)), fabs(hi(Z.d))));
    int ex = 0;
    if (mx > 0) frexp(mx, &ex);
    Z.a = scale2(Z.a, -ex);
    Z.b = scale2(Z.b, -ex);
    Z.c = scale2(Z.c, -ex);
    Z.d = scale2(Z.d, -ex);
    return Z;
}
constexpr int RS_TPB = 128;
template <class R>
__global__ void __launch_bounds__(RS_TPB) k_root_scan(const int *blk_chunk0, int nblocks,
                                                      const Mat2<R> *mats, R *states) {
    const int b = blockIdx.x;
    const int c0 = blk_chunk0[b], c1 = blk_chunk0[b + 1];
    const int nc = c1 - c0;
    const int per = (nc + RS_TPB - 1) / RS_TPB;
    const int r0 = c0 + threadIdx.x * per, r1 = min(r0 + per, c1);
    Mat2<R> L;  // composed transfer matrix of this thread's run (identity if empty)
    L.a = mk<R>(1.0);
    L.b = mk<R>(0.0);
    L.c = mk<R>(0.0);
    L.d = mk<R>(1.0);
    for (int k = r0; k < r1; k++) L = mat_mul<R>(mats[k], L);
    __shared__ Mat2<R> sm[RS_TPB];
    sm[threadIdx.x] = L;
    __syncthreads();
    for (int off = 1; off < RS_TPB; off <<= 1) {  // inclusive scan: S_t = L_t ... L_0
        Mat2<R> v = sm[threadIdx.x];
        const bool take = (int)threadIdx.x >= off;
        Mat2<R> u;
        if (take) u = sm[threadIdx.x - off];
        __syncthreads();
        if (take) sm[threadIdx.x] = mat_mul<R>(v, u);
        __syncthreads();
    }
    // incoming state of the run: S_{t-1} (1, 0)
    R p = mk<R>(1.0), q = mk<R>(0.0);
    if (threadIdx.x > 0) {
        const Mat2<R> E = sm[threadIdx.x - 1];
        p = E.a;
        q = E.c;
    }
    for (int k = r0; k < r1; k++) {
        states[2 * k] = p;
        states[2 * k + 1] = q;
        const Mat2<R> M = mats[k];
        R np = add(mul(M.a, p), mul(M.b, q));
        R nq = add(mul(M.c, p), mul(M.d, q));
        double mx = fmax(fabs(hi(np)), fabs(hi(nq)));
        int ex = 0;
        if (mx > 0) frexp(mx, &ex);
        p = scale2(np, -ex);
        q = scale2(nq, -ex);
    }
    (void)nblocks;
}

template <class R, class T>
__global__ void k_root_factor(const T *__restrict__ d, const T *__restrict__ e,
                              const ChunkDesc *chunks, int nch, const BlockDesc *blocks,
                              double scale, const double *mu, const R *states, int right,
                              double xi, uint64_t seed, double *rep_pool, double *repx_pool,
                              int *fail) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nch) return;
    const ChunkDesc ch = chunks[k];
    const int64_t b0 = blocks[ch.block].row0, bn = blocks[ch.block].n;
    const double m = mu[ch.block];
    R dprev = mk<R>(0.0);
    if (ch.row0 > b0) dprev = div(states[2 * k], states[2 * k + 1]);
    bool bad = false;
    for (int j = 0; j < ch.len; j++) {
        const int64_t r = ch.row0 + j;
        R c = shifted_diag<R>((double)d[r] * scale, m);
        R dr = c;
        if (r > b0) {
            double ev = (double)e[r - 1] * scale;
            R lprev = div(mk<R>(ev), dprev);
            dr = sub(c, mul(lprev, ev));
        }
        bool good = right ? (hi(dr) < 0.0) : (hi(dr) > 0.0);
        if (!good || !isfinite(hi(dr))) bad = true;
        R lr = mk<R>(0.0);
        if (r < b0 + bn - 1) lr = div(mk<R>((double)e[r] * scale), dr);
        R dp = dr, lp = lr;
        if (bn > 1) {
            dp = add(dr, mul(dr, xi * uniform_pm1(seed, (uint64_t)r, 0)));
            if (r < b0 + bn - 1) lp = add(lr, mul(lr, xi * uniform_pm1(seed, (uint64_t)r, 1)));
        }
        R ldv = mul(dp, lp);
        R lldv = mul(ldv, lp);
        store_row4<R>(rep_pool + r * 4 * Prec<R>::words, 0, dp, lldv, lp, ldv);
        reinterpret_cast<double2 *>(repx_pool)[r] = make_double2(hi(dp), hi(lldv));
        dprev = dr;
    }
    if (bad) atomicExch(fail, 1);
}

template <class R>
__global__ void k_root_nodes(const BlockDesc *blocks, int nblocks, const double *mu,
                             double *rep_pool, double *repx_pool, NodeInfo *nodes) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    NodeInfo ni;
    ni.rep = rep_pool + blocks[b].row0 * 4 * Prec<R>::words;
    ni.repx = repx_pool + blocks[b].row0 * 2;
    ni.n = blocks[b].n;
    ni.row0 = blocks[b].row0;
    ni.sig_hi = mu[b];
    ni.sig_lo = 0.0;
    ni.depth = 0;
    ni.block = b;
    ni.parent = -1;
    ni.pad_ = 0;
    ni.pp = nullptr;
    nodes[b] = ni;
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
