// k_rqi.cuh -- K5 + K6: singleton eigenpairs by Rayleigh quotient iteration on
// twisted factorizations, then normalisation, rounding to binary_x and the
// coalesced store of the Z column (Alg. 1 l.11-12, PAPER.md L652-L727,
// L1140-L1173; memory contract L1199-L1226).
//
// One thread per eigenpair; every CTA holds eigenpairs of ONE representation
// (the host groups the singletons by node), so the rows of that representation
// are staged through shared memory: tiles of RQ_TR rows (plus a halo below) are
// loaded cooperatively with cp.async into a double buffer while the previous
// tile is consumed, and all four sweeps read their rows from smem.
//
// Iteration j at shift lam:
//   F (stationary, top-down):   s_1 = -lam ; d+_i = d_i + s_i ; l+_i = ld_i / d+_i ;
//                               s_{i+1} = l+_i l_i s_i - lam ; count #{d+_i < 0}
//   B (progressive, bottom-up): p_n = d_n - lam ; D-_{i+1} = lld_i + p_{i+1} ;
//                               t = d_i / D-_{i+1} ; u-_i = l_i t ; p_i = p_{i+1} t - lam
//   gamma_k = s_k + p_k + lam ; r = argmin |gamma_k| (ties: smallest k)
//   ||z||^2 for twist k = 1 + W_k + V_k with the prefix norms
//       W_{k+1} = (l+_k)^2 (1 + W_k),  V_{k-1} = (u-_{k-1})^2 (1 + V_k)
//   (exact identities for z_r = 1, z_i = -l+_i z_{i+1} (i < r), z_{i+1} = -u-_i z_i),
//   kept in binary64: they only feed the RQ correction and the stopping test.
//   lam <- lam + gamma_r / ||z||^2          (RQ correction, L714-L717)
//   stop: |gamma_r|/||z|| <= k_rs gap eps_x sqrt(n)   (Eq. (3.6))
//         or |gamma_r|/||z||^2 <= 8 eps_y |lam|        (stagnation, L720-L723)
// The iterate is kept inside the certified bracket (the inertia of each factorization
// updates it); an iterate leaving it is replaced by the bracket midpoint (RQI "guarded
// by bisection", L315); after max_rqi iterations: bisection to relative
// eps_x sqrt(n) gaptol and one more twisted solve (L1154-L1163).
//
// Fixed twist (R9b): the binary_y factorizations run with the twist r located by
// k_rqi_locate, top-down to r and bottom-up to r interleaved (two chains per thread),
// in projective form (R8b).  The eigenvector (K6) is written by the last
// factorization itself in product form (k_zprod.cuh): z_i = y_i / y_r above the
// twist and x_k / x_r below it, so no back-substitution sweep and no checkpoint
// storage is needed on the regular path; k_zscale applies the per-column factors
// and the exact 1/||z|| (squares accumulated with compensated sums while writing).
// Only the rare fallback path keeps the sweep form (checkpoints of (s, W) and p every
// RQ_C rows, blocks recomputed when the sweep needs them in the other direction).
#pragma once
#include <type_traits>

#include "k_bisect.cuh"
#include "k_zprod.cuh"

namespace mr3 {

constexpr int RQ_C = 8;      // checkpoint block (rows)
constexpr int RQ_TR = 32;    // rows per staged tile = output tile rows (4 blocks)
constexpr int RQ_HALO = 8;   // rows staged below a tile (the sweeps need row t0 - 1)
constexpr int RQ_TPB = 128;  // threads per CTA


// state of an eigenpair handed from k_rqi_fb (iterations 1-2) to k_rqi (later iterations)
template <class R>
struct RqiResume {
    R lam, a, b, lam_out;  // current shift, guard bracket, converged eigenvalue (if done)
    int32_t iters;         // passes done
    int32_t erefF, erefB;  // scale references of the product-form z (k_zprod.cuh)
    int32_t flags;         // 1: converged, 2: z of the converged shift written
};

template <class R>
struct RqiArgs {
    const NodeInfo *nodes;
    Items it;
    const int32_t *list;   // singleton item ids
    const RqiTask *tasks;  // one per CTA
    R *ck_s, *ck_p;        // [nblk][S]
    double *ck_W;          // [nblk][S]
    ZCol *zc;              // per local column: rows, twist and factors for k_zscale
    int64_t S;             // checkpoint stride (CTAs in this launch * RQ_TPB)
    double pivmin, krs, eps_x, gaptol;
    double twist_w;     // twist weight slope: |gamma_k| (1 + twist_w |2k - n| / n) is minimised
    double root_widen;  // > 0: root-node brackets are binary_x brackets; the guard is widened
                        // by root_widen * n * |lambda| (relative robustness of the root, R8d)
    int maxit;
    int jobz_v;
    int split;  // split passes (R9d): 0 none, 1 iterations >= 3, 2 every iteration (1 item/CTA)
    int fuse_scale;  // 1: every CTA normalises its own columns at its end (no k_zscale launch)
    void *w;          // eigenvalue output (global positions)
    void *Z;          // eigenvector output (columns col - zcol0)
    int64_t ldz, zcol0;
    double unscale;   // multiply eigenvalues by this (exact power of 2)
    DevStats *st;
    int32_t *dbg_iters;  // optional (MR3_DEBUG): iterations per item
    double *dbg_trace;   // optional (MR3_DEBUG): 8 per item: x0 used, gap, r, res/tol per iteration
    unsigned long long *dbg_clk;  // optional (MR3_DEBUG): 4 per CTA: start, end (ns), rmin, rmax
    char *left;                   // k_rqi_fb: per list position, 1 = continue in k_rqi
    RqiResume<R> *resume;         // k_rqi_fb: per item id, state of the eigenpairs left
    const RqiResume<R> *resume_in;  // k_rqi: nullptr = fresh start, else continue from it
    int iter0;                    // k_rqi with resume_in: passes already done (uniform)
};

__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// caps a prefix norm W >= 0 (or NaN) near 1e250: an unsigned min on the high word orders
// non-negative doubles (and sends every NaN to the cap) in one integer instruction
__device__ __forceinline__ double clampbig(double x) {
    const unsigned h = (unsigned)__double2hiint(x);
    return __hiloint2double((int)min(h, 0x73d658e3u), __double2loint(x));
}

// sign(x) != sign(y) as 0/1 (the inertia of a projective step)
template <class R>
__device__ __forceinline__ int sgn_ne_R(R x, R y) {
    return (int)((unsigned)(__double2hiint(hi(x)) ^ __double2hiint(hi(y))) >> 31);
}
// v * 2^k (k <= 1023; results below the normal range flush to zero)
__device__ __forceinline__ double pow2mul_d(double v, int k) {
    return k < -1022 ? 0.0 : v * __hiloint2double((k + 1023) << 20, 0);
}
// ||z||^2 of a storing pass from the sum of the written squares in z_r = 1 units (reading
// R9e); a non-finite or sub-unit sum (z_r is one of the terms) cannot be a norm: 1 + nothing
__device__ __forceinline__ double nz2_of_ss(double ss) {
    return (ss >= 1.0 && ss <= 1e300) ? ss : 1.0;
}
// compensated (Kahan) sum of squares: sum += x^2
__device__ __forceinline__ void kahan_sq(double x, double &sum, double &comp) {
    const double y = fma(x, x, -comp);
    const double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
}

// ss += x^2 in pair arithmetic (two-prod + two-sum)
__device__ __forceinline__ void accum_sq(double x, double &sh, double &sl) {
    double p = x * x;
    double pe = fma(x, x, -p);
    double e;
    double sn = two_sum(sh, p, e);
    sl += e + pe;
    sh = sn;
}

// ---------------------------------------------------------------- staging
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// rows of ROWD doubles (4 R values per row of a binary_y representation, {d, lld}
// per row of the binary_x copy)
template <int ROWD_>
struct StageG {
    static constexpr int ROWD = ROWD_;             // doubles per row
    static constexpr int ROWS = RQ_TR + RQ_HALO;   // staged rows per tile
    static constexpr int TILE = ROWS * ROWD;       // doubles per tile buffer
};
template <class R>
struct Stage : StageG<4 * Prec<R>::words> {};

// rows [t0 - HALO, t0 + TR) of rep (clamped to [0, n)) -> buf, asynchronously; with
// pp != nullptr also the same rows of the node's PP array (4 doubles per row) -> buf + TILE
constexpr int PP_TILE = (RQ_TR + RQ_HALO) * 4;  // doubles of a staged PP tile
template <int ROWD>
__device__ __forceinline__ void stage_tile_g(double *buf, const double *rep, int64_t n, int64_t t0,
                                             const double *pp = nullptr) {
    constexpr int CH = StageG<ROWD>::ROWS * ROWD / 2;  // 16-byte chunks
    for (int c = threadIdx.x; c < CH; c += RQ_TPB) {
        int r = c / (ROWD / 2), off = (c % (ROWD / 2)) * 2;
        int64_t g = t0 - RQ_HALO + r;
        g = g < 0 ? 0 : (g >= n ? n - 1 : g);
        cp_async16(buf + r * ROWD + off, rep + g * ROWD + off);
    }
    if (pp != nullptr) {
        constexpr int CP = (RQ_TR + RQ_HALO) * 2;
        double *pb = buf + StageG<ROWD>::TILE;
        for (int c = threadIdx.x; c < CP; c += RQ_TPB) {
            int r = c >> 1, off = (c & 1) * 2;
            int64_t g = t0 - RQ_HALO + r;
            g = g < 0 ? 0 : (g >= n ? n - 1 : g);
            cp_async16(pb + r * 4 + off, pp + g * 4 + off);
        }
    }
    cp_async_commit();
}

// Run body(buf, t0) over all row tiles of the representation, ascending or
// descending, with the next tile's rows in flight while the current one is used.
// Every thread of the CTA must call this (barriers inside).
template <int ROWD, class Body>
__device__ __forceinline__ void staged_pass_g(double *smem, const double *rep, int64_t n, bool desc,
                                              Body body) {
    constexpr int TILE = StageG<ROWD>::TILE;
    const int ntile = (int)((n + RQ_TR - 1) / RQ_TR);
    auto t0_of = [&](int i) -> int64_t { return (int64_t)(desc ? ntile - 1 - i : i) * RQ_TR; };
    stage_tile_g<ROWD>(smem, rep, n, t0_of(0));
    for (int i = 0; i < ntile; i++) {
        if (i + 1 < ntile) {
            stage_tile_g<ROWD>(smem + ((i + 1) & 1) * TILE, rep, n, t0_of(i + 1));
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        body(smem + (i & 1) * TILE, t0_of(i));
        __syncthreads();
    }
}
template <class R, class Body>
__device__ __forceinline__ void staged_pass(double *smem, const double *rep, int64_t n, bool desc,
                                            Body body) {
    staged_pass_g<Stage<R>::ROWD>(smem, rep, n, desc, body);
}

template <class R>
__device__ __forceinline__ Row4<R> srow(const double *buf, int64_t t0, int64_t k);
template <>
__device__ __forceinline__ Row4<dd> srow<dd>(const double *buf, int64_t t0, int64_t k) {
    const double2 *p = reinterpret_cast<const double2 *>(buf + (k - t0 + RQ_HALO) * 8);
    double2 a = p[0], b = p[1], c = p[2], d = p[3];
    Row4<dd> r;
    r.d = mkdd(a.x, a.y);
    r.lld = mkdd(b.x, b.y);
    r.l = mkdd(c.x, c.y);
    r.ld = mkdd(d.x, d.y);
    return r;
}
template <>
__device__ __forceinline__ Row4<double> srow<double>(const double *buf, int64_t t0, int64_t k) {
    const double2 *p = reinterpret_cast<const double2 *>(buf + (k - t0 + RQ_HALO) * 4);
    double2 a = p[0], b = p[1];
    Row4<double> r;
    r.d = a.x;
    r.lld = a.y;
    r.l = b.x;
    r.ld = b.y;
    return r;
}

// Two tile streams at once: ascending tiles a0, a0+1, ... (nA of them) and descending
// tiles d0, d0-1, ... (nD of them); step i hands body the i-th tile of each stream
// (nullptr once a stream is exhausted).  Used by the fixed-twist sweeps (top-down
// rows < r and bottom-up rows > r) and by the z sweeps (rows <= r downward and rows
// > r upward): the two halves are independent recurrences, and interleaving them
// gives every thread two dependent chains at once.  smem: 4 tile buffers.  Collective.
template <int ROWD, class Body>
__device__ __forceinline__ void dual_staged_pass(double *smem, const double *rep, int64_t n, int a0,
                                                 int nA, int d0, int nD, Body body,
                                                 const double *pp = nullptr) {
    constexpr int TILE = StageG<ROWD>::TILE + PP_TILE;  // buffer stride (PP rows after the rows)
    const int steps = nA > nD ? nA : nD;
    auto bufA = [&](int b) -> double * { return smem + (b ? TILE : 0); };
    auto bufD = [&](int b) -> double * { return smem + (b ? 3 * TILE : 2 * TILE); };
    if (steps <= 0) return;
    if (nA > 0) stage_tile_g<ROWD>(bufA(0), rep, n, (int64_t)a0 * RQ_TR, pp);
    if (nD > 0) stage_tile_g<ROWD>(bufD(0), rep, n, (int64_t)d0 * RQ_TR, pp);
    for (int i = 0; i < steps; i++) {
        if (i + 1 < steps) {
            if (i + 1 < nA)
                stage_tile_g<ROWD>(bufA((i + 1) & 1), rep, n, (int64_t)(a0 + i + 1) * RQ_TR, pp);
            if (i + 1 < nD)
                stage_tile_g<ROWD>(bufD((i + 1) & 1), rep, n, (int64_t)(d0 - i - 1) * RQ_TR, pp);
            // stage_tile_g commits one group per call: wait until the current step's
            // groups are complete (at most the just-issued ones pending)
            if (i + 1 < nA && i + 1 < nD)
                cp_async_wait<2>();
            else
                cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        body(i < nA ? bufA(i & 1) : nullptr, (int64_t)(a0 + i) * RQ_TR,
             i < nD ? bufD(i & 1) : nullptr, (int64_t)(d0 - i) * RQ_TR);
        __syncthreads();
    }
}

// dynamic shared memory of k_rqi: 4 staged tiles (rows + PP rows), the two z tiles of a
// storing pass, per-thread column data
template <class R, class OutT>
constexpr size_t rqi_smem_bytes() {
    return 4 * (size_t)(Stage<R>::TILE + PP_TILE) * sizeof(double) +
           2 * 16 * (size_t)(RQ_TPB + 1) * sizeof(OutT) + 2 * RQ_TPB * sizeof(int64_t) +
           RQ_TPB * sizeof(int) + 4 * sizeof(int);
}

// ---------------------------------------------------------------- kernel
template <class R, class OutT>
__global__ void __launch_bounds__(RQ_TPB, 3) k_rqi(RqiArgs<R> A) {
    extern __shared__ __align__(16) double rq_dyn[];  // rqi_smem_bytes<R, OutT>()
    double *sstage = rq_dyn;                           // 4 tiles: dual_staged_pass
    OutT(*ztF)[RQ_TPB + 1] = reinterpret_cast<OutT(*)[RQ_TPB + 1]>(
        rq_dyn + 4 * (Stage<R>::TILE + PP_TILE));      // z tiles of a storing pass
    OutT(*ztB)[RQ_TPB + 1] = ztF + 16;
    int64_t *s_r = reinterpret_cast<int64_t *>(ztB + 16);
    int64_t *s_zoff = s_r + RQ_TPB;
    int *s_wz = reinterpret_cast<int *>(s_zoff + RQ_TPB);
    int &s_rmin = s_wz[RQ_TPB];
    int &s_rmax = s_wz[RQ_TPB + 1];

    const int tid = threadIdx.x;
    const RqiTask task = A.tasks[blockIdx.x];
    const NodeInfo nd = A.nodes[task.node];
    const int64_t n = nd.n;
    const int64_t slot = (int64_t)blockIdx.x * RQ_TPB + tid;
    const bool active = tid < task.cnt;
    int id = -1, k = 0;
    R lam = mk<R>(0.0), a = lam, b = lam, gr = lam, lam_out = lam;
    R A_a0 = lam, A_b0 = lam;  // incoming bracket (diagnostics)
    double nz2 = 1.0, gap = INFINITY;
    int64_t r = 0;
    unsigned long long rows = 0;
    int iters = 0;
    bool done = !active;
    if (active) {
        id = A.list[task.first + tid];
        k = A.it.k[id];
        a = reinterpret_cast<const R *>(A.it.lo)[id];
        b = reinterpret_cast<const R *>(A.it.hi)[id];
        lam = half(add(a, b));
        A_a0 = a;
        A_b0 = b;
        if (A.root_widen > 0.0 && nd.depth == 0) {
            const double wd = A.root_widen * (double)n * fmax(fabs(hi(a)), fabs(hi(b)));
            a = sub(a, mk<R>(wd));
            b = add(b, mk<R>(wd));
        }
        const double x0 = A.it.x0[id];  // refined start (K2'), inside the (widened) guard
        if (!isnan(x0) && lt(a, mk<R>(x0)) && lt(mk<R>(x0), b)) lam = mk<R>(x0);
        gap = fmin(A.it.lgap[id], A.it.rgap[id]);
        if (!(gap > 0.0)) gap = fmax(hi(sub(b, a)), 1e-300);
        r = A.it.twist[id];
        if (r < 0 || r >= n) r = n - 1;
        if (n == 1) {  // 1x1 block: the eigenpair is (d_1, e_1) exactly
            lam_out = load_row4<R>(nd.rep, 0).d;
            done = true;
        }
    }
    const double tol = A.krs * gap * A.eps_x * sqrt((double)n);
    // twist range of the CTA (the fixed-twist sweeps stage rows up to these)
    if (tid == 0) {
        s_rmin = (int)n;
        s_rmax = 0;
    }
    __syncthreads();
    if (active) {
        atomicMin(&s_rmin, (int)r);
        atomicMax(&s_rmax, (int)r);
    }
    __syncthreads();
    const int cta_rmin = s_rmin <= s_rmax ? s_rmin : 0;
    const int cta_rmax = s_rmin <= s_rmax ? s_rmax : (int)n - 1;
    if (A.dbg_clk && tid == 0) {
        A.dbg_clk[4 * blockIdx.x] = gtimer_ns();
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        A.dbg_clk[4 * blockIdx.x + 2] = (unsigned long long)smid |
                                        ((unsigned long long)(cta_rmin & 0xffffff) << 8) |
                                        ((unsigned long long)(cta_rmax & 0xffffff) << 32);
    }

    // output column of this eigenpair (rows of its block) and the factors for k_zscale
    const int64_t col0 = active ? A.it.col[id] : -1;
    OutT *zcol = (A.jobz_v && active && col0 >= 0)
                     ? reinterpret_cast<OutT *>(A.Z) + nd.row0 + (col0 - A.zcol0) * A.ldz
                     : nullptr;
    ZCol zinfo;
    zinfo.row0 = nd.row0;
    zinfo.n = (int32_t)n;
    zinfo.r = (int32_t)r;
    zinfo.cF = 1.0;
    zinfo.cB = 1.0;
    zinfo.ss = 1.0;
    bool zwritten = false, zfinal = false;
    int erefF = 0, erefB = 0;
    if (zcol != nullptr && n == 1) {  // 1x1 block: z = e_1
        zcol[0] = (OutT)1.0;
        zfinal = true;
    }
    int pdone = 0;  // passes done before this launch beyond A.iter0 (per eigenpair)
    if (active && A.resume_in != nullptr) {  // continue after k_rqi_fb's / k_rqi_chunk's passes
        const RqiResume<R> rs = A.resume_in[id];
        pdone = A.iter0 == 0 ? rs.iters : 0;
        lam = rs.lam;
        a = rs.a;
        b = rs.b;
        lam_out = rs.lam_out;
        erefF = rs.erefF;
        erefB = rs.erefB;
        done = (rs.flags & 1) != 0;
        zfinal = (rs.flags & 2) != 0;
    }

    // one twisted factorization at lam for the threads with `need`
    auto twisted = [&](bool need) -> int {
        // F: top-down, checkpoints (s, W) at every block start
        R s = neg(lam);
        double W = 0.0;
        int negc = 0;
        staged_pass<R>(sstage, nd.rep, n, false, [&](const double *buf, int64_t t0) {
            if (!need) return;
#pragma unroll
            for (int q = 0; q < RQ_TR / RQ_C; q++) {
                const int64_t b0 = t0 + q * RQ_C;
                if (b0 < n) {
                    A.ck_s[(b0 / RQ_C) * A.S + slot] = s;
                    A.ck_W[(b0 / RQ_C) * A.S + slot] = W;
                }
#pragma unroll
                for (int j = 0; j < RQ_C; j++) {
                    const int64_t kk = b0 + j;
                    if (kk < n) {
                        Row4<R> rw = srow<R>(buf, t0, kk);
                        R dp = guard(add(rw.d, s), A.pivmin);
                        negc += is_neg(dp) ? 1 : 0;
                        if (kk < n - 1) {
                            R lp = div(rw.ld, dp);
                            double l2 = hi(lp) * hi(lp);
                            W = clampbig(fma(l2, W, l2));
                            s = sub(mul(lp, mul(rw.l, s)), lam);
                        }
                    }
                }
            }
        });
        // B: bottom-up, argmin |gamma_k|, p checkpoints
        R p = mk<R>(0.0);
        double V = 0.0, best = INFINITY;
        int64_t rr = n - 1;
        R g_r = mk<R>(0.0);
        double z2 = 1.0;
        if (need) p = sub(load_row4<R>(nd.rep, n - 1).d, lam);
        staged_pass<R>(sstage, nd.rep, n, true, [&](const double *buf, int64_t t0) {
            if (!need) return;
#pragma unroll 1
            for (int q = RQ_TR / RQ_C - 1; q >= 0; q--) {
                const int64_t b0 = t0 + q * RQ_C;
                if (b0 >= n) continue;
                const int64_t blk = b0 / RQ_C;
                R sb[RQ_C];
                double wb[RQ_C];
                R s2 = A.ck_s[blk * A.S + slot];
                double W2 = A.ck_W[blk * A.S + slot];
#pragma unroll
                for (int j = 0; j < RQ_C; j++) {
                    const int64_t kk = b0 + j;
                    sb[j] = s2;
                    wb[j] = W2;
                    if (kk < n - 1) {
                        Row4<R> rw = srow<R>(buf, t0, kk);
                        R dp = guard(add(rw.d, s2), A.pivmin);
                        R lp = div(rw.ld, dp);
                        double l2 = hi(lp) * hi(lp);
                        W2 = clampbig(fma(l2, W2, l2));
                        s2 = sub(mul(lp, mul(rw.l, s2)), lam);
                    }
                }
#pragma unroll
                for (int j = RQ_C - 1; j >= 0; j--) {
                    const int64_t kk = b0 + j;
                    if (kk < n) {
                        if (j == 0) A.ck_p[blk * A.S + slot] = p;  // p at the block start
                        R g = add(add(sb[j], p), lam);
                        double ga = fabs(hi(g));
                        if (ga <= best) {
                            best = ga;
                            rr = kk;
                            g_r = g;
                            z2 = 1.0 + wb[j] + V;
                        }
                        if (kk > 0) {
                            Row4<R> rw = srow<R>(buf, t0, kk - 1);
                            R Dm = guard(add(rw.lld, p), A.pivmin);
                            R t = div(rw.d, Dm);
                            double u2 = hi(rw.l) * hi(t);
                            u2 *= u2;
                            V = clampbig(fma(u2, V, u2));
                            p = sub(mul(p, t), lam);
                        }
                    }
                }
            }
        });
        if (need) {
            r = rr;
            gr = g_r;
            nz2 = z2;
            rows += 3 * n;
        }
        return negc;
    };

    // One twisted factorization at lam with the twist index r fixed (from
    // k_rqi_locate): F rows 0..r-1 top-down and B rows n-1..r+1 bottom-up only --
    // n rows instead of the 3n of a full factorization with argmin.  Checkpoints:
    // s at every block start b0 <= r, p at every block start >= r (what the z
    // sweeps below need).  Returns the inertia of the twisted factorization
    // N_r Delta_r N_r^T = M - lam I, Delta_r = diag(d+_0..d+_{r-1}, gamma_r,
    // D-_{r+1}..D-_{n-1}), i.e. negcount(lam) (Sylvester).
    // Fixed-twist factorization in projective (division-free) form, as the Sturm counts
    // (R8b): top-down s = pF/qF with D = d qF + pF (= d+ qF), pF <- lld pF - lam D,
    // qF <- D; bottom-up p = pB/qB with E = lld_{k-1} qB + pB (= D-_k qB),
    // pB <- d_{k-1} pB - lam E, qB <- E.  Every row is two pair FMAs and a pair product
    // (no division on the dependent chain); l+ and u- enter only the binary64 norm
    // identities, formed off-chain.  Ratios s_b0, p_b0 are formed once per checkpoint.
    using G0 = std::integral_constant<bool, false>;
    using G1 = std::integral_constant<bool, true>;
    auto twisted_fixed = [&](bool need, bool store) -> int {
        if (need) zwritten = false;
        double sF = 0.0, cF_ = 0.0, sB = 0.0, cB_ = 0.0;  // Kahan sums of written squares
        const R mlam = neg(lam);
        R pF = mlam, qF = mk<R>(1.0);
        int EqF = 0, EqB = 0;  // exponents taken out of (pF, qF) / (pB, qB) by the rescaling
        double W = 0.0;
        int negc = 0;
        R pB = mk<R>(0.0), qB = mk<R>(1.0);
        double V = 0.0;
        if (need) pB = sub(load_row4<R>(nd.rep, n - 1).d, lam);
        // F: rows 0..r-1 ascending (tiles 0 .. cta_rmax/RQ_TR); B: rows n-1..r descending
        const int ntile = (int)((n + RQ_TR - 1) / RQ_TR);
        const int nA = cta_rmax / RQ_TR + 1;
        const int nD = ntile - cta_rmin / RQ_TR;
        auto sgn_ne = [](R x, R y) -> int {
            return (int)((unsigned)(__double2hiint(hi(x)) ^ __double2hiint(hi(y))) >> 31);
        };
        auto rescale_pq = [](R &x, R &y, int &E) {
            const unsigned ex = (unsigned)__double2hiint(hi(x)) & 0x7ff00000u;
            const unsigned ey = (unsigned)__double2hiint(hi(y)) & 0x7ff00000u;
            const unsigned em = ex > ey ? ex : ey;
            if (em == 0x7ff00000u || em == 0u) return;
            const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
            x = scale_pow2(x, sc);
            y = scale_pow2(y, sc);
            E += (int)(em >> 20) - 1023;
        };
        // z components in product form (k_zprod.cuh): row kk <= r: y = qF / PP_kk,
        // row kk >= r: x = QB PP_kk, written scaled by 2^-ref (ref from the previous pass)
        const bool wz = store && need && zcol != nullptr;
        const bool sq = store && need;  // squares summed (the norm of a storing pass, R9e)
        auto ppr = [&](int64_t kk, double &pm, double &ipm, int &e) {
            const double2 *q = reinterpret_cast<const double2 *>(nd.pp + kk * PP_STRIDE);
            const double2 a0 = __ldg(q), a1 = __ldg(q + 1);
            pm = a0.x;
            ipm = a0.y;
            e = __double2loint(a1.x);  // exponent stored as int bits (k_node_pp)
        };
        // the PP row of kk from the staged tile (rows follow the representation rows)
        auto sppr = [&](const double *buf, int64_t t0, int64_t kk, double &pm, double &ipm,
                        int &e) {
            const double2 *q = reinterpret_cast<const double2 *>(
                buf + Stage<R>::TILE + (kk - t0 + RQ_HALO) * 4);
            const double2 a0 = q[0], a1 = q[1];
            pm = a0.x;
            ipm = a0.y;
            e = __double2loint(a1.x);  // exponent stored as int bits (k_node_pp)
        };
        // value * 2^k (k <= 1023; results below the normal range flush to zero)
        auto pow2mul = [](double v, int k) -> double {
            return k < -1022 ? 0.0 : v * __hiloint2double((k + 1023) << 20, 0);
        };
        // compensated (Kahan) sums of the squares of the written F and B parts
        auto kahan = [](double x, double &sum, double &comp) {
            const double y = fma(x, x, -comp);
            const double t = sum + y;
            comp = (t - sum) - y;
            sum = t;
        };
        // one F row (rows < r) and one B row (rows > r); predicated commits keep the two
        // recurrences in one basic block so their dependent chains interleave
        // GUARD: rows may lie on the other side of some thread's twist (else every row of
        // the call commits: the block is below / above the whole CTA's twist range)
        auto frow = [&](auto guard, const double *bA, int64_t tA, int64_t kk) {
            constexpr bool GUARD = decltype(guard)::value;
            Row4<R> rw = srow<R>(bA, tA, kk);
            const R D = fma_dd(rw.d, qF, pF);
            const double lpx = hi(rw.ld) * hi(qF) * rcp_w(hi(D));  // l+ = ld / d+
            const double l2 = lpx * lpx;
            const double W2 = clampbig(fma(l2, W, l2));
            const R p2 = dot2_dd(mlam, D, rw.lld, pF);
            if (!GUARD || (int)kk < (int)r) {
                if (sq) {
                    double pm, ipm;
                    int e;
                    sppr(bA, tA, kk, pm, ipm, e);
                    const OutT zo = (OutT)pow2mul(hi(qF) * ipm, EqF - e - erefF);
                    ztF[(kk - tA) & 15][tid] = zo;
                    kahan((double)zo, sF, cF_);
                }
                negc += sgn_ne(D, qF);
                W = W2;
                pF = p2;
                qF = D;
            }
        };
        auto brow = [&](auto guard, const double *bD, int64_t tD, int64_t kk) {
            constexpr bool GUARD = decltype(guard)::value;
            Row4<R> rw = srow<R>(bD, tD, kk - 1);
            const R E = fma_dd(rw.lld, qB, pB);
            const double ux = hi(rw.ld) * hi(qB) * rcp_w(hi(E));  // u- = l d / D-
            const double u2 = ux * ux;
            const double V2 = clampbig(fma(u2, V, u2));
            const R P2 = dot2_dd(mlam, E, rw.d, pB);
            if (!GUARD || ((int)kk > (int)r && (int)kk < (int)n)) {
                if (sq) {
                    double pm, ipm;
                    int e;
                    sppr(bD, tD, kk, pm, ipm, e);
                    const OutT zo = (OutT)pow2mul(hi(qB) * pm, EqB + e - erefB);
                    ztB[(kk - tD) & 15][tid] = zo;
                    kahan((double)zo, sB, cB_);
                }
                negc += sgn_ne(E, qB);
                V = V2;
                pB = P2;  // p_{kk-1} = pB / qB
                qB = E;
            }
        };
        // storing pass: the written components go through two 16-row smem tiles (one per
        // stream) and leave as coalesced 128-byte column segments
        // (collective: with resumed eigenpairs the store flag can differ between threads)
        const bool cta_store = __syncthreads_or(store && A.jobz_v) != 0;
        if (cta_store) {
            // per column: the rows each stream writes (F: g < rF, B: g > rB; nothing if the
            // column is not written) and the column's base pointer
            reinterpret_cast<int2 *>(s_r)[tid] = wz ? make_int2((int)r, (int)r) : make_int2(-1, INT_MAX);
            reinterpret_cast<OutT **>(s_zoff)[tid] =
                wz ? reinterpret_cast<OutT *>(A.Z) + (col0 - A.zcol0) * A.ldz + nd.row0 : nullptr;
        }
        auto flush = [&](const double *bA, int64_t tA, int hA, const double *bD, int64_t tD,
                         int hD) {
            __syncthreads();
            const int warp = tid >> 5, lane = tid & 31, row = lane & 15;
            const int2 *rfb = reinterpret_cast<const int2 *>(s_r);
            OutT *const *zp = reinterpret_cast<OutT *const *>(s_zoff);
            const int gA = bA != nullptr ? (int)tA + 16 * hA + row : INT_MAX;
            const int gD = (bD != nullptr && (int)tD + 16 * hD + row < (int)n)
                               ? (int)tD + 16 * hD + row
                               : INT_MIN;
#pragma unroll 4
            for (int c = 2 * warp + (lane >> 4); c < RQ_TPB; c += 2 * (RQ_TPB / 32)) {
                const int2 rb = rfb[c];
                if (gA < rb.x) zp[c][gA] = ztF[row][c];
                if (gD > rb.y) zp[c][gD] = ztB[row][c];
            }
            __syncthreads();
        };
        dual_staged_pass<Stage<R>::ROWD>(
            sstage, nd.rep, n, 0, nA, ntile - 1, nD,
            [&](const double *bA, int64_t tA, const double *bD, int64_t tD) {
#pragma unroll 1
                for (int h = 0; h < 2; h++) {
                    if (need) {
#pragma unroll 1
                        for (int q = 2 * h; q < 2 * h + 2; q++) {
                            const int64_t b0F = tA + q * RQ_C;
                            const int64_t b0B = tD + (RQ_TR / RQ_C - 1 - q) * RQ_C;
                            // (CTA-uniform) blocks entirely below / above the twist range
                            const bool fastF = bA != nullptr && b0F + RQ_C <= cta_rmin;
                            const bool fastB = bD != nullptr && b0B > cta_rmax && b0B + RQ_C <= n;
                            const bool fF = bA != nullptr && b0F < r;
                            const bool fB = bD != nullptr && b0B + RQ_C > r && b0B < n;
                            if (fastF && fastB) {
#pragma unroll
                                for (int j = 0; j < RQ_C; j++) {
                                    frow(G0{}, bA, tA, b0F + j);
                                    brow(G0{}, bD, tD, b0B + RQ_C - 1 - j);
                                }
                            } else if (fF && fB) {
#pragma unroll
                                for (int j = 0; j < RQ_C; j++) {
                                    frow(G1{}, bA, tA, b0F + j);
                                    brow(G1{}, bD, tD, b0B + RQ_C - 1 - j);
                                }
                            } else if (fF) {
#pragma unroll
                                for (int j = 0; j < RQ_C; j++) frow(G1{}, bA, tA, b0F + j);
                            } else if (fB) {
#pragma unroll
                                for (int j = 0; j < RQ_C; j++) brow(G1{}, bD, tD, b0B + RQ_C - 1 - j);
                            }
                            if (fF) rescale_pq(pF, qF, EqF);
                            if (fB) rescale_pq(pB, qB, EqB);
                        }
                    }
                    if (cta_store) flush(bA, tA, h, bD, tD, 1 - h);
                }
            },
            cta_store ? nd.pp : nullptr);
        if (need) {
            gr = add(add(div(pF, qF), div(pB, qB)), lam);
            negc += is_neg(gr) ? 1 : 0;
            rows += n;
            // y_r = qF / PP_r and x_r = QB PP_r: references for the next pass and the
            // per-column factors (z_i = Z_i 2^refF / y_r, z_k = Z_k 2^refB / x_r)
            double pm = 1.0, ipm = 1.0;
            int e = 0;
            if (nd.pp != nullptr) ppr(r, pm, ipm, e);
            const double yr = hi(qF) * ipm, xr = hi(qB) * pm;
            const int eyr = EqF - e, exr = EqB + e;
            if (sq) {  // k_rqi_fb's storing-pass join, the same operations
                const OutT zo = (OutT)pow2mul(yr, eyr - erefF);
                kahan((double)zo, sF, cF_);
                const double fF = ldexp(1.0, erefF - eyr) / yr;
                const double fB = ldexp(1.0, erefB - exr) / xr;
                const double ss = fF * fF * sF + fB * fB * sB;
                nz2 = nz2_of_ss(ss);
                if (wz) {
                    zcol[r] = zo;
                    zinfo.cF = fF;
                    zinfo.cB = fB;
                    zinfo.ss = ss;
                    zwritten = true;
                }
            } else {
                nz2 = 1.0 + W + V;
            }
            erefF = eyr + expo_of(yr);
            erefB = exr + expo_of(xr);
        }
        return negc;
    };

    // ---- split pass (third and later RQI iterations): one eigenpair, the whole CTA ----
    // By then at most a few eigenpairs of the CTA are still iterating, and a CTA-wide
    // serial pass would cost a full n-row chain for them.  The projective transforms are
    // linear in (p, q): F row k maps (p, q) -> (lld_k p - lam (d_k q + p), d_k q + p) and
    // B row k -> (d_{k-1} p - lam (lld_{k-1} q + p), lld_{k-1} q + p).  The F rows [0, r)
    // and B rows (r, n) are cut into chunks (one per thread, proportional to length);
    // each thread forms its chunk's 2x2 transfer matrix (two basis solutions, pair
    // arithmetic), one thread per direction chains them into the chunk start states,
    // and every thread re-runs the true recurrence from its start (z in product form,
    // compensated norms, inertia).  The re-run end state of a chunk must equal the next
    // chunk's start to 2^-84 relative; otherwise the pass is redone serially.  Chain:
    // about 3 n / 128 rows instead of n / 2.
    struct SplitIO {
        R lam, gr;
        int64_t r, zoff;
        int erefF, erefB, wz, negc, bad, eyr, exr;
        double yr, xr, sF, cF, sB, cB, jF, jB;
    };
    __shared__ SplitIO sio;
    __shared__ int s_need[RQ_TPB];
    __shared__ int s_dbg_rel;  // (MR3_DEBUG) worst continuity of the last split pass, log2 * 16
    __shared__ double s_red[2 * (RQ_TPB / 32)][2];
    __shared__ int s_redi[RQ_TPB / 32][2];
    __shared__ double s_redj[RQ_TPB / 32][2];
    auto rescale_pq2 = [](R &x, R &y, int &E) {
        const unsigned ex = (unsigned)__double2hiint(hi(x)) & 0x7ff00000u;
        const unsigned ey = (unsigned)__double2hiint(hi(y)) & 0x7ff00000u;
        const unsigned em = ex > ey ? ex : ey;
        if (em == 0x7ff00000u || em == 0u) return;
        const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
        x = scale_pow2(x, sc);
        y = scale_pow2(y, sc);
        E += (int)(em >> 20) - 1023;
    };
    auto rescale_4 = [](R &a1, R &a2, R &a3, R &a4, int &E) {
        unsigned em = (unsigned)__double2hiint(hi(a1)) & 0x7ff00000u;
        unsigned t = (unsigned)__double2hiint(hi(a2)) & 0x7ff00000u;
        em = t > em ? t : em;
        t = (unsigned)__double2hiint(hi(a3)) & 0x7ff00000u;
        em = t > em ? t : em;
        t = (unsigned)__double2hiint(hi(a4)) & 0x7ff00000u;
        em = t > em ? t : em;
        if (em == 0x7ff00000u || em == 0u) return;
        const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
        a1 = scale_pow2(a1, sc);
        a2 = scale_pow2(a2, sc);
        a3 = scale_pow2(a3, sc);
        a4 = scale_pow2(a4, sc);
        E += (int)(em >> 20) - 1023;
    };
    auto split_pass = [&]() {  // collective; inputs and outputs in sio
        const R lam_s = sio.lam, mlam = neg(sio.lam);
        const int64_t rs = sio.r;
        OutT *zc = sio.wz ? reinterpret_cast<OutT *>(A.Z) + sio.zoff : nullptr;
        const int64_t LF = rs, LB = n - 1 - rs;
        int tF = (int)((RQ_TPB * LF + (LF + LB) / 2) / (LF + LB));
        if (LF > 0 && tF < 1) tF = 1;
        if (LB > 0 && tF > RQ_TPB - 1) tF = RQ_TPB - 1;
        const int tB = RQ_TPB - tF;
        const bool isF = tid < tF;
        const int c = isF ? tid : tid - tF, nc = isF ? tF : tB;
        // F: rows k0 .. k1-1 ascending; B: rows k0 .. k1+1 descending
        const int64_t k0 = isF ? LF * c / nc : n - 1 - LB * c / nc;
        const int64_t k1 = isF ? LF * (c + 1) / nc : n - 1 - LB * (c + 1) / nc;
        const int64_t len = isF ? k1 - k0 : k0 - k1;
        R *Mx = reinterpret_cast<R *>(sstage);  // 4 per thread: u = M (1, 0), v = M (0, 1)
        R *Sx = Mx + 4 * RQ_TPB;                // 2 per thread: start state (p, q)
        int *ME = reinterpret_cast<int *>(Sx + 2 * RQ_TPB);
        int *SE = ME + RQ_TPB;
        // phase 1: transfer matrix of the chunk
        {
            R up = mk<R>(1.0), uq = mk<R>(0.0), vp = mk<R>(0.0), vq = mk<R>(1.0);
            int EM = 0;
#pragma unroll 1
            for (int64_t j0 = 0; j0 < len; j0 += 8) {
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    if (j0 + j < len) {
                        const int64_t kk = isF ? k0 + j0 + j : k0 - j0 - j;
                        const Row4<R> rw = load_row4<R>(nd.rep, isF ? kk : kk - 1);
                        const R m1 = isF ? rw.d : rw.lld, m2 = isF ? rw.lld : rw.d;
                        const R U = fma_dd(m1, uq, up), V = fma_dd(m1, vq, vp);
                        up = dot2_dd(mlam, U, m2, up);
                        vp = dot2_dd(mlam, V, m2, vp);
                        uq = U;
                        vq = V;
                    }
                }
                rescale_4(up, uq, vp, vq, EM);
            }
            Mx[4 * tid] = up;
            Mx[4 * tid + 1] = uq;
            Mx[4 * tid + 2] = vp;
            Mx[4 * tid + 3] = vq;
            ME[tid] = EM;
        }
        __syncthreads();
        // phase 2: chunk start states, chained by one thread per direction
        if ((tid == 0 && tF > 0) || (tid == tF && tB > 0)) {
            R p = isF ? mlam : sub(load_row4<R>(nd.rep, n - 1).d, lam_s), q = mk<R>(1.0);
            int E = 0;
#pragma unroll 1
            for (int j = 0; j < nc; j++) {
                const int t = tid + j;
                Sx[2 * t] = p;
                Sx[2 * t + 1] = q;
                SE[t] = E;
                const R np = add(mul(p, Mx[4 * t]), mul(q, Mx[4 * t + 2]));
                const R nq = add(mul(p, Mx[4 * t + 1]), mul(q, Mx[4 * t + 3]));
                p = np;
                q = nq;
                E += ME[t];
                rescale_pq2(p, q, E);
            }
        }
        __syncthreads();
        // phase 3: the true recurrence from the start state
        R p = Sx[2 * tid], q = Sx[2 * tid + 1];
        int E = SE[tid];
        double s = 0.0, cmp = 0.0;
        int ng = 0;
        double zlast = 0.0, rnorm = 0.0;  // |z| and row norm at the chunk's last row
        const int eref = isF ? sio.erefF : sio.erefB;
#pragma unroll 1
        for (int64_t j0 = 0; j0 < len; j0 += 8) {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (j0 + j < len) {
                    const int64_t kk = isF ? k0 + j0 + j : k0 - j0 - j;
                    const Row4<R> rw = load_row4<R>(nd.rep, isF ? kk : kk - 1);
                    double pm = 1.0, ipm = 1.0;
                    int e = 0;
                    if (nd.pp != nullptr) {
                        const double2 *qq = reinterpret_cast<const double2 *>(nd.pp + kk * PP_STRIDE);
                        const double2 a0 = __ldg(qq), a1 = __ldg(qq + 1);
                        pm = a0.x;
                        ipm = a0.y;
                        e = __double2loint(a1.x);
                    }
                    // F: y_kk = qF / PP_kk; B: x_kk = QB PP_kk (written scaled by 2^-eref)
                    const double zv = isF ? pow2mul_d(hi(q) * ipm, E - e - eref)
                                          : pow2mul_d(hi(q) * pm, E + e - eref);
                    const OutT zo = (OutT)zv;
                    if (zc != nullptr) zc[kk] = zo;
                    kahan_sq((double)zo, s, cmp);
                    zlast = fabs(zv);
                    rnorm = fabs(hi(rw.d)) + fabs(hi(rw.lld)) + 2.0 * fabs(hi(rw.ld)) +
                            fabs(hi(lam_s));
                    const R m1 = isF ? rw.d : rw.lld, m2 = isF ? rw.lld : rw.d;
                    const R D = fma_dd(m1, q, p);
                    ng += sgn_ne_R<R>(D, q);
                    p = dot2_dd(mlam, D, m2, p);
                    q = D;
                }
            }
            rescale_pq2(p, q, E);
        }
        // continuity with the next chunk's start: a relative jump delta of the state at a
        // chunk boundary perturbs the recurrence there, i.e. adds about delta |z_k| ||row_k||
        // to the residual of the (scaled) vector; summed in squares per direction and
        // checked against the stopping tolerance by the owner
        int bad = 0;
        double jres = 0.0;
        if (c + 1 < nc) {
            const int t = tid + 1;
            const int dE = SE[t] - E;
            if (dE > 60 || dE < -60) {
                bad = 1;
            } else {
                const double sc = __hiloint2double((dE + 1023) << 20, 0);
                const R p2 = scale_pow2(Sx[2 * t], sc), q2 = scale_pow2(Sx[2 * t + 1], sc);
                const double mag = fmax(fabs(hi(p)), fabs(hi(q)));
                const double dif = fmax(fabs(hi(sub(p, p2))), fabs(hi(sub(q, q2))));
                const double rel = dif / mag;
                bad = !(rel <= 0x1p-60) ? 1 : 0;  // (beyond: the chunk chain is unusable)
                const double j1 = rel * fmax(zlast, 1e-300) * rnorm;
                jres = j1 * j1;
                if (A.dbg_trace) atomicMax(&s_dbg_rel, (int)(log2(dif / mag + 1e-300) * 16.0) + 32768);
            }
        } else {  // last chunk of its direction: the state at r
            if (isF) {
                sio.gr = div(p, q);  // s_r (F part of gamma_r)
                sio.yr = hi(q);
                sio.eyr = E;
            } else {
                sio.lam = div(p, q);  // p_r (B part); lam is no longer needed
                sio.xr = hi(q);
                sio.exr = E;
            }
        }
        // reductions: Kahan sums per direction, inertia, continuity
        const int warp = tid >> 5, lane = tid & 31;
        double sFv = isF ? s : 0.0, cFv = isF ? cmp : 0.0, sBv = isF ? 0.0 : s, cBv = isF ? 0.0 : cmp;
        double jF = isF ? jres : 0.0, jB = isF ? 0.0 : jres;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sFv += __shfl_down_sync(0xffffffffu, sFv, o);
            cFv += __shfl_down_sync(0xffffffffu, cFv, o);
            sBv += __shfl_down_sync(0xffffffffu, sBv, o);
            cBv += __shfl_down_sync(0xffffffffu, cBv, o);
            ng += __shfl_down_sync(0xffffffffu, ng, o);
            bad += __shfl_down_sync(0xffffffffu, bad, o);
            jF += __shfl_down_sync(0xffffffffu, jF, o);
            jB += __shfl_down_sync(0xffffffffu, jB, o);
        }
        if (lane == 0) {
            s_red[2 * warp][0] = sFv;
            s_red[2 * warp][1] = cFv;
            s_red[2 * warp + 1][0] = sBv;
            s_red[2 * warp + 1][1] = cBv;
            s_redi[warp][0] = ng;
            s_redi[warp][1] = bad;
            s_redj[warp][0] = jF;
            s_redj[warp][1] = jB;
        }
        __syncthreads();
        if (tid == 0) {
            double a1 = 0, a2 = 0, a3 = 0, a4 = 0;
            int i1 = 0, i2 = 0;
            for (int w = 0; w < RQ_TPB / 32; w++) {
                a1 += s_red[2 * w][0];
                a2 += s_red[2 * w][1];
                a3 += s_red[2 * w + 1][0];
                a4 += s_red[2 * w + 1][1];
                i1 += s_redi[w][0];
                i2 += s_redi[w][1];
                sio.jF = (w == 0 ? 0.0 : sio.jF) + s_redj[w][0];
                sio.jB = (w == 0 ? 0.0 : sio.jB) + s_redj[w][1];
            }
            sio.sF = a1;
            sio.cF = a2;
            sio.sB = a3;
            sio.cB = a4;
            sio.negc = i1;
            sio.bad = i2;
            if (tF == 0) {  // r = 0: no F rows, s_0 = -lam, qF = 1
                sio.gr = mlam;
                sio.yr = 1.0;
                sio.eyr = 0;
            }
            if (tB == 0) {  // r = n - 1: p_{n-1} = d_{n-1} - lam, QB = 1
                sio.lam = sub(load_row4<R>(nd.rep, n - 1).d, lam_s);
                sio.xr = 1.0;
                sio.exr = 0;
            }
        }
        __syncthreads();
    };
    // all eigenpairs of the CTA with `need`, one split pass each; returns the inertia
    auto split_all = [&](bool need, bool store) -> int {
        if (need) zwritten = false;
        s_need[tid] = need ? 1 : 0;
        __syncthreads();
        int myc = 0;
        bool redo = false;
#pragma unroll 1
        for (int j = 0; j < RQ_TPB; j++) {
            if (!s_need[j]) continue;  // (uniform)
            const bool wzj = store && zcol != nullptr;
            if (tid == j) {
                sio.lam = lam;
                sio.r = r;
                sio.erefF = erefF;
                sio.erefB = erefB;
                sio.wz = wzj ? 1 : 0;
                sio.zoff = wzj ? (col0 - A.zcol0) * A.ldz + nd.row0 : 0;
            }
            if (tid == 0) s_dbg_rel = 0;
            __syncthreads();
            split_pass();
            if (tid == j && A.dbg_trace) A.dbg_trace[8 * (int64_t)id + 7] = (s_dbg_rel - 32768) / 16.0;
            if (tid == j) {
                if (sio.bad) {
                    redo = true;
                } else {
                    const R sr = sio.gr, pr = sio.lam;
                    gr = add(add(sr, pr), lam);
                    myc = sio.negc + (is_neg(gr) ? 1 : 0);
                    rows += n;
                    double pm = 1.0, ipm = 1.0;
                    int e = 0;
                    if (nd.pp != nullptr) {
                        const double2 *qq = reinterpret_cast<const double2 *>(nd.pp + r * PP_STRIDE);
                        pm = qq[0].x;
                        ipm = qq[0].y;
                        e = __double2loint(qq[1].x);
                    }
                    const double yr = sio.yr * ipm, xr = sio.xr * pm;
                    const int eyr = sio.eyr - e, exr = sio.exr + e;
                    double sF = sio.sF, cF_ = sio.cF;
                    const OutT zo = (OutT)pow2mul_d(yr, eyr - erefF);
                    kahan_sq((double)zo, sF, cF_);
                    const double fF = ldexp(1.0, erefF - eyr) / yr;
                    const double fB = ldexp(1.0, erefB - exr) / xr;
                    nz2 = fF * fF * (sF - cF_) + fB * fB * (sio.sB - sio.cB);
                    // residual added by the chunk-boundary jumps (normalised vector)
                    const double jr = sqrt(fF * fF * sio.jF + fB * fB * sio.jB) / sqrt(nz2);
                    if (!(jr <= 0.125 * tol)) redo = true;
                    if (wzj && !redo) {
                        zcol[r] = zo;
                        zinfo.cF = fF;
                        zinfo.cB = fB;
                        zinfo.ss = nz2;
                        zwritten = true;
                    }
                    if (!redo) {
                        erefF = eyr + expo_of(yr);
                        erefB = exr + expo_of(xr);
                    } else {
                        rows -= n;
                    }
                }
            }
            __syncthreads();
        }
        // a chunk chain that lost accuracy: the serial pass for those eigenpairs
        if (__syncthreads_or(redo)) {
            const int c2 = twisted_fixed(redo, store);
            if (redo) myc = c2;
        }
        return myc;
    };

#pragma unroll 1
    for (iters = A.iter0 + 1; iters <= A.maxit; iters++) {
        // an eigenpair that converged in the first (non-storing) pass joins the next
        // pass of its CTA at the same shift to write z (instead of an extra pass later)
        const int itp = iters + pdone;  // this eigenpair's iteration number
        const bool store_only =
            A.jobz_v && itp >= 2 && done && !zfinal && zcol != nullptr && n > 1;
        const bool need = (!done || store_only) && itp <= A.maxit;
        if (!__syncthreads_or(need)) break;
        const int c = ((iters <= 2 && A.split < 2) || n < 4 * RQ_TPB || !A.split)
                          ? twisted_fixed(need, A.jobz_v && itp >= 2)
                                                     : split_all(need, A.jobz_v && itp >= 2);
        if (store_only) zfinal = zwritten;
        if (need && !store_only) {
            if (c >= k) {
                if (lt(lam, b)) b = lam;
            } else {
                if (lt(a, lam)) a = lam;
            }
            double g = hi(gr);
            double corr = g / nz2;
            R lam_new = add(lam, mk<R>(corr));
            if (A.dbg_trace) {
                double *tr = A.dbg_trace + 8 * (int64_t)id;
                if (iters == 1) {
                    const double x0 = A.it.x0[id];
                    tr[0] = isnan(x0) ? -0.5 * hi(sub(A_b0, A_a0)) : 1.0;  // -(half-width) if unrefined
                    tr[1] = gap;
                    tr[2] = (double)r;
                }
                if (iters <= 5) tr[2 + iters] = fabs(g) / sqrt(nz2) / tol;
            }
            if (fabs(g) / sqrt(nz2) <= tol || fabs(corr) <= 8.0 * Prec<R>::eps * fabs(hi(lam)) ||
                g == 0.0) {
                lam_out = lam_new;
                done = true;
                zfinal = zwritten;  // z of this (converged) factorization is in Z
            } else {
                if (!(lt(a, lam_new) && lt(lam_new, b))) lam_new = half(add(a, b));
                lam = lam_new;
            }
        }
    }
    // converged in the first (non-storing) pass: one more pass at the same shift writes z
    {
        const bool extra = A.jobz_v && done && !zfinal && zcol != nullptr && n > 1;
        if (__syncthreads_or(extra)) {
            twisted_fixed(extra, true);
            if (extra) zfinal = zwritten;
        }
    }
    // fallback: bisection to relative eps_x sqrt(n) gaptol, then one more solve
    const bool fb = !done;
    if (__syncthreads_or(fb)) {
        if (fb) {
            double rtol = A.eps_x * sqrt((double)n) * A.gaptol;
#pragma unroll 1
            for (int it2 = 0; it2 < 400; it2++) {
                R w = sub(b, a);
                if (hi(w) <= fmax(2.0 * rtol * fmax(fabs(hi(a)), fabs(hi(b))), 1e-300)) break;
                R mid = half(add(a, b));
                if (!(lt(a, mid) && lt(mid, b))) break;
                if (negcount<R>(nd.rep, n, mid, A.pivmin) >= k)
                    b = mid;
                else
                    a = mid;
                rows += n;
            }
            lam = half(add(a, b));
        }
        twisted(fb);
        if (fb) {
            R lam_new = add(lam, mk<R>(hi(gr) / nz2));
            lam_out = (lt(a, lam_new) && lt(lam_new, b)) ? lam_new : lam;
            atomicAdd(&A.st->rqi_fallbacks, 1);
            iters = A.maxit + 1;
        }
    }
    int64_t col = -1;
    if (active) {
        // eigenvalue output: w = (lambda[M] + sigma) * 2^-scale  (Alg. 1 l.12)
        R lt_ = add(lam_out, mk2<R>(nd.sig_hi, nd.sig_lo));
        col = A.it.col[id];
        if (col >= 0) {
            if (sizeof(OutT) == 4)
                reinterpret_cast<float *>(A.w)[col] = (float)(hi(lt_) * A.unscale);
            else
                reinterpret_cast<double *>(A.w)[col] = hi(lt_) * A.unscale;
        }
        reinterpret_cast<R *>(A.it.lo)[id] = lam_out;  // keep lambda[M] for diagnostics
        atomicMax(&A.st->rqi_iters_max, iters);
        if (A.dbg_iters) A.dbg_iters[id] = iters;
    }
    if (A.dbg_clk) {
        atomicMax(&A.dbg_clk[4 * blockIdx.x + 1], gtimer_ns());
        atomicMax(&A.dbg_clk[4 * blockIdx.x + 3],
                  (unsigned long long)iters | ((unsigned long long)(tid == 0 ? id : 0) << 8));
    }
    if (!A.jobz_v) {
        if (active && rows) atomicAdd(&A.st->rqi_rows, rows);
        return;
    }
    // K6 epilogue fused (A.fuse_scale): the CTA normalises its own columns as soon as it is
    // done -- the HBM traffic of the scaling overlaps the other CTAs' arithmetic (collective)
    auto fused_scale = [&]() {
        if (!A.fuse_scale) return;
        ZCol *szc = reinterpret_cast<ZCol *>(sstage);
        OutT **szp = reinterpret_cast<OutT **>(szc + RQ_TPB);
        __syncthreads();  // (sstage is free: the last staged pass ended with a barrier)
        szc[tid] = zinfo;
        szp[tid] = zcol;  // nullptr: no column
        __syncthreads();
        constexpr int V = 16 / sizeof(OutT);
        using Vec = typename std::conditional<sizeof(OutT) == 8, double2, float4>::type;
#pragma unroll 1
        for (int j = 0; j < RQ_TPB; j++) {
            OutT *col = szp[j];
            if (col == nullptr) continue;  // (uniform)
            const ZCol z = szc[j];
            const double inv = 1.0 / sqrt(z.ss);
            const double fF = z.cF * inv, fB = z.cB * inv;
            const int64_t nn = z.n;
            const bool aligned = (reinterpret_cast<uintptr_t>(col) & 15) == 0;
            const int64_t nv = aligned ? nn / V : 0;  // whole vectors
            Vec *cv = reinterpret_cast<Vec *>(col);
            constexpr int U = 8;
#pragma unroll 1
            for (int64_t b0 = 0; b0 < nv; b0 += (int64_t)U * RQ_TPB) {
                Vec v[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t i = b0 + u * RQ_TPB + tid;
                    if (i < nv) v[u] = cv[i];
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t i = b0 + u * RQ_TPB + tid;
                    if (i < nv) {
                        OutT *e = reinterpret_cast<OutT *>(&v[u]);
#pragma unroll
                        for (int q = 0; q < V; q++)
                            e[q] = (OutT)((double)e[q] * (i * V + q <= z.r ? fF : fB));
                        cv[i] = v[u];
                    }
                }
            }
            for (int64_t i = nv * V + tid; i < nn; i += RQ_TPB)  // tail / misaligned
                col[i] = (OutT)((double)col[i] * (i <= z.r ? fF : fB));
        }
    };

    // ---------------- fallback only: z by sweeps from the checkpoints of twisted() ------
    // (the regular path wrote z in product form during its last fixed-twist pass)
    const bool mine = zcol != nullptr && fb && !zfinal;
    if (!__syncthreads_or(mine)) {
        if (zcol != nullptr) A.zc[col0 - A.zcol0] = zinfo;
        if (active && rows) atomicAdd(&A.st->rqi_rows, rows);
        fused_scale();
        return;
    }
    const double inv = 1.0 / sqrt(nz2);
    double ss_hi = 0.0, ss_lo = 0.0;
    const double tiny = 1e-250;
    // two sweeps outward from the twist r, interleaved:
    //   D: rows k <= r, downward, z_r = 1, z_k = -l+_k z_{k+1}
    //      (z_k = -(ld_{k+1}/ld_k) z_{k+2} if z_{k+1} == 0)
    //   U: rows k > r, upward, z_k = -u-_{k-1} z_{k-1}
    //      (z_k = -(ld_{k-2}/ld_{k-1}) z_{k-2} if z_{k-1} == 0)
    // l+ / u- of each 8-row block are recomputed from the checkpoints of twisted().
    R z1D = mk<R>(0.0), z2D = mk<R>(0.0), ldn = mk<R>(0.0);        // z_{k+1}, z_{k+2}, ld_{k+1}
    R z1U = mk<R>(0.0), z2U = mk<R>(0.0);                          // z_{k-1}, z_{k-2}
    R ldm1 = mk<R>(0.0), ldm2 = mk<R>(0.0), ucarry = mk<R>(0.0);  // ld_{k-1}, ld_{k-2}, u-_{b0-1}
    auto put = [&](int64_t kk, R z) {
        if (fabs(hi(z)) < tiny) z = mk<R>(0.0);
        const OutT zo = (OutT)hi(mul(z, inv));
        accum_sq((double)zo, ss_hi, ss_lo);
        zcol[kk] = zo;
        return z;
    };
    auto drecompute = [&](const double *buf, int64_t t0, int64_t b0, R *lpb) {
        R s = A.ck_s[(b0 / RQ_C) * A.S + slot];
#pragma unroll
        for (int j = 0; j < RQ_C; j++) {
            const int64_t kk = b0 + j;
            lpb[j] = mk<R>(0.0);
            if (kk < n - 1 && kk < r) {
                Row4<R> rw = srow<R>(buf, t0, kk);
                R dp = guard(add(rw.d, s), A.pivmin);
                R lp = div(rw.ld, dp);
                lpb[j] = lp;
                s = sub(mul(lp, mul(rw.l, s)), lam);
            }
        }
    };
    auto dz = [&](const double *buf, int64_t t0, int64_t b0, const R *lpb) {
#pragma unroll
        for (int j = RQ_C - 1; j >= 0; j--) {
            const int64_t kk = b0 + j;
            if (kk > r || kk >= n) continue;
            Row4<R> rw = srow<R>(buf, t0, kk);
            R z;
            if (kk == r)
                z = mk<R>(1.0);
            else if (hi(z1D) == 0.0 && fabs(hi(z2D)) > tiny)
                z = neg(mul(div(ldn, rw.ld), z2D));
            else
                z = neg(mul(lpb[j], z1D));
            z = put(kk, z);
            z2D = z1D;
            z1D = z;
            ldn = rw.ld;
        }
    };
    // u-_k for k in [b0, e), e = min(b0 + C, n - 1), from the checkpoint p_{b0+C}
    auto urecompute = [&](const double *buf, int64_t t0, int64_t b0, R *ub) {
        const int64_t e = (b0 + RQ_C < n - 1) ? b0 + RQ_C : n - 1;
        R p;
        if (e == b0 + RQ_C)
            p = A.ck_p[((b0 + RQ_C) / RQ_C) * A.S + slot];
        else
            p = sub(srow<R>(buf, t0, n - 1).d, lam);
#pragma unroll
        for (int j = RQ_C - 1; j >= 0; j--) {
            const int64_t kk = b0 + j;
            ub[j] = mk<R>(0.0);
            if (kk < e) {
                Row4<R> rw = srow<R>(buf, t0, kk);
                R Dm = guard(add(rw.lld, p), A.pivmin);
                R t = div(rw.d, Dm);
                ub[j] = mul(rw.l, t);
                p = sub(mul(p, t), lam);
            }
        }
    };
    auto uz = [&](const double *buf, int64_t t0, int64_t b0, const R *ub) {
#pragma unroll
        for (int j = 0; j < RQ_C; j++) {
            const int64_t kk = b0 + j;
            const R uprev = (j == 0) ? ucarry : ub[j == 0 ? 0 : j - 1];
            if (kk < n) {
                const R ldk = srow<R>(buf, t0, kk).ld;
                if (kk == r) {
                    z1U = mk<R>(1.0);
                    z2U = mk<R>(0.0);
                } else if (kk > r) {
                    R z;
                    if (hi(z1U) == 0.0 && fabs(hi(z2U)) > tiny)
                        z = neg(mul(div(ldm2, ldm1), z2U));
                    else
                        z = neg(mul(uprev, z1U));
                    z = put(kk, z);
                    z2U = z1U;
                    z1U = z;
                }
                ldm2 = ldm1;
                ldm1 = ldk;
            }
        }
        ucarry = ub[RQ_C - 1];
    };
    {
        // the fallback's full factorization chose its own twists: range of the sweeping threads
        __syncthreads();
        if (tid == 0) {
            s_rmin = (int)n;
            s_rmax = 0;
        }
        __syncthreads();
        if (mine) {
            atomicMin(&s_rmin, (int)r);
            atomicMax(&s_rmax, (int)r);
        }
        __syncthreads();
        const int fr_min = s_rmin <= s_rmax ? s_rmin : 0;
        const int fr_max = s_rmin <= s_rmax ? s_rmax : (int)n - 1;
        const int ntile = (int)((n + RQ_TR - 1) / RQ_TR);
        const int tmin = fr_min / RQ_TR, tmax = fr_max / RQ_TR;
        // U: ascending from the tile of the smallest twist; D: descending from the largest
        dual_staged_pass<Stage<R>::ROWD>(
            sstage, nd.rep, n, tmin, ntile - tmin, tmax, tmax + 1,
            [&](const double *bU, int64_t tU, const double *bD, int64_t tD) {
                if (!mine) return;
#pragma unroll 1
                for (int q = 0; q < RQ_TR / RQ_C; q++) {
                    const int64_t b0D = tD + (RQ_TR / RQ_C - 1 - q) * RQ_C;
                    const int64_t b0U = tU + q * RQ_C;
                    const bool dD = bD != nullptr && b0D <= r && b0D < n;
                    const bool dU = bU != nullptr && b0U < n && b0U + RQ_C - 1 >= r;
                    if (bU != nullptr && b0U < n && b0U + RQ_C - 1 < r) {  // below the twist
                        ldm2 = srow<R>(bU, tU, b0U + RQ_C - 2).ld;
                        ldm1 = srow<R>(bU, tU, b0U + RQ_C - 1).ld;
                    }
                    if (dD) {
                        R lpb[RQ_C];
                        drecompute(bD, tD, b0D, lpb);
                        dz(bD, tD, b0D, lpb);
                    }
                    if (dU) {
                        R ub[RQ_C];
                        urecompute(bU, tU, b0U, ub);
                        uz(bU, tU, b0U, ub);
                    }
                }
            });
        if (mine) rows += n + 1;
    }
    if (zcol != nullptr) {
        if (mine) {  // written normalised by the estimate; k_zscale renormalises exactly
            zinfo.r = (int32_t)r;
            zinfo.cF = 1.0;
            zinfo.cB = 1.0;
            zinfo.ss = ss_hi + ss_lo;
        }
        A.zc[col0 - A.zcol0] = zinfo;
    }
    (void)ss_hi;
    (void)ss_lo;
    if (active && rows) atomicAdd(&A.st->rqi_rows, rows);
    fused_scale();
}

// ---------------------------------------------------------------------------
// K5a: twist index of each singleton ("determine
// r = argmin_k |gamma_k|"), located once in binary_x on the narrowed copy M_x
// (L1071): a full twisted factorization at lam_loc = lam_start + 1e-4 gap --
// close to lambda on the scale of the gap, far from it on the scale of the
// binary_x rounding -- so |gamma_k| ~ |lambda - lam_loc| / z_k^2 and the argmin
// picks a row where the eigenvector is large.  The binary_y iterations (k_rqi)
// then keep r fixed and need only n rows per factorization: the RQ correction
// gamma_r / ||z||^2 is exact to first order for any r with z_r != 0, and the
// stopping test (Eq. (3.6)) is evaluated on the actual binary_y gamma_r.
//   F: s_0 = -lam ; d+_i = d_i + s_i ; s_{i+1} = lld_i s_i / d+_i - lam
//   B: p_{n-1} = d_{n-1} - lam ; D-_{i+1} = lld_i + p_{i+1} ; p_i = d_i p_{i+1} / D-_{i+1} - lam
//   (both evaluated in projective form, see below)
//   gamma_k = s_k + p_k + lam ;  r = argmin |gamma_k| w_k (ties: smallest k),
//   w_k = 1 + 3 |2k - n| / n in [1, 4]: the chosen |gamma_r| is within 4x of the minimum
//   (Dhillon-Parlett: any twist with |gamma_r| = O(min) gives the same quality of z;
//   the stopping test is applied to the binary_y gamma_r actually used)
// Evaluated without the cancellation in s_k + p_k + lam: with theta_k = prod_{j<k} d+_j
// (leading minor of M - lam, = the projective qF before row k) and phi_k = prod_{j>k} D-_j
// (trailing minor, = QB at row k), gamma_k = det(M - lam) / (theta_k phi_k) (Cramer's rule
// on [(M - lam)^-1]_kk), so argmin_k |gamma_k| w_k = argmax_k log2|theta_k phi_k| - log2 w_k.
// One sweep: F (top-down, theta) and B (bottom-up, phi) interleaved over all rows,
// meeting at the middle.  A 32-row tile is reached first by one stream, which keeps its
// candidate row there -- the row where its half of the eigenvector, y_k = theta_k / PP_k
// (F) or x_k = phi_k PP_k (B) (k_zprod.cuh), is largest -- and its log2 magnitude; the
// other stream evaluates the score at that row when it arrives.  Candidates cost 8 bytes
// per tile and eigenpair (in ck_W); the log2 magnitudes are the exponent-mantissa bits
// of the binary64 values read as fixed point (error < 0.09, irrelevant for a factor-4
// tolerant choice).
// ---------------------------------------------------------------------------
template <class R>
__global__ void __launch_bounds__(RQ_TPB) k_rqi_locate(RqiArgs<R> A) {
    __shared__ __align__(16) double sx[4 * (StageG<2>::TILE + PP_TILE)];
    const int tid = threadIdx.x;
    const RqiTask task = A.tasks[blockIdx.x];
    const NodeInfo nd = A.nodes[task.node];
    const int64_t n = nd.n;
    const int64_t slot = (int64_t)blockIdx.x * RQ_TPB + tid;
    const bool active = tid < task.cnt && n > 1;
    int id = -1;
    double lam = 0.0;
    if (tid < task.cnt) {
        id = A.list[task.first + tid];
        const double a = hi(reinterpret_cast<const R *>(A.it.lo)[id]);
        const double b = hi(reinterpret_cast<const R *>(A.it.hi)[id]);
        double gap = fmin(A.it.lgap[id], A.it.rgap[id]);
        if (!(gap > 0.0) || !(gap < INFINITY)) gap = fmax(b - a, 1e-300);
        const double x0 = A.it.x0[id];
        const double wd = (A.root_widen > 0.0 && nd.depth == 0)
                              ? A.root_widen * (double)n * fmax(fabs(a), fabs(b))
                              : 0.0;  // as k_rqi's guard
        lam = (!isnan(x0) && x0 > a - wd && x0 < b + wd) ? x0 : 0.5 * (a + b);
        lam += 1e-4 * gap;
        if (n <= 1) A.it.twist[id] = 0;
    }
    if (n <= 1) return;  // (uniform over the CTA: one node per CTA)
    const int ntile = (int)((n + RQ_TR - 1) / RQ_TR);
    int *cand = reinterpret_cast<int *>(A.ck_W);  // per tile: the reference of its int16 records
    // log2|PP| of the tile's row tr (staged PP rows; slot 3 holds {-1023 - log2|PP|,
    // -1023 + log2|PP|} as two floats, k_node_pp)
    // (PP slot 3: round(16 log2|PP_k|) as int bits, k_node_pp)
    auto lpp16 = [](const double *buf, int tr) -> int {
        return reinterpret_cast<const int *>(buf + StageG<2>::TILE + (tr + RQ_HALO) * 4 + 3)[0];
    };
    // 16 log2|v| + 16 * 1023 (piecewise linear, integer: exponent and top 4 mantissa bits)
    auto l16 = [](double v) -> int { return (__double2hiint(v) & 0x7fffffff) >> 16; };
    auto rescale2 = [](double &x, double &y, int &E) {
        const unsigned ex = (unsigned)__double2hiint(x) & 0x7ff00000u;
        const unsigned ey = (unsigned)__double2hiint(y) & 0x7ff00000u;
        const unsigned em = ex > ey ? ex : ey;
        if (em == 0x7ff00000u || em == 0u) return;
        const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
        x *= sc;
        y *= sc;
        E += (int)(em >> 20) - 1023;
    };
    const float wfac = (float)(A.twist_w / (double)n);
    auto logw = [&](int64_t k) -> int {  // 16 log2 of the twist weight 1 + w |2k - n| / n
        return __float2int_rn(16.0f * __log2f(fmaf(wfac, fabsf(2.0f * (float)k - (float)n), 1.0f)));
    };
    // F: theta (projective pf/qf, exponent EF); B: phi (pb/qb, EB)
    double pf = -lam, qf = 1.0, pb = 0.0, qb = 1.0;
    int EF = 0, EB = 0;
    if (active) pb = __ldg(nd.repx + 2 * (n - 1)) - lam;
    int best = INT_MIN;  // in 1/16 log2 units
    int64_t rr = n / 2;  // (kept if every score is -inf: no usable twist information)
    // tile i is reached first by F iff 2 i < ntile - 1, by B iff 2 i > ntile - 1, by both
    // at the same step iff 2 i == ntile - 1 (F's rows of that tile are run first then).
    // The stream that reaches a row first stores its log2 half-vector magnitude
    // (log2|y_k| = log2|theta_k| - log2|PP_k| for F, log2|x_k| = log2|phi_k| + log2|PP_k|
    // for B) as int16 in 1/16 units relative to the tile's first value (per tile, float);
    // the other stream adds its own at the same row: log2|gamma_k|^-1 + const =
    // log2|y_k| + log2|x_k|, minus log2 w (the tile's).  Every row is scored (localised
    // eigenvectors peak within a few rows).  The mode is uniform over the CTA at every step.
    // [tile][slot][32 rows] int16: one 64-byte record per tile and eigenpair (4 x 16 B)
    uint4 *hist = reinterpret_cast<uint4 *>(A.ck_s);
    int EF16 = 0, EB16 = 0;  // 16 EF, 16 EB (log2 bookkeeping in 1/16 units)
    // MODE 0: keep the tile's values in h (registers; stored at the tile end as int8 in whole
    // log2 units below the tile maximum, 32 bytes per tile and eigenpair); MODE 1: score
    // against h (the other stream's values, unpacked to 1/16 units relative to its maximum)
    auto frow = [&](auto mode, auto guard, const double *bA, int tr, int kk, int base,
                    int (&h)[32]) {
        constexpr int MODE = decltype(mode)::value;
        constexpr bool GUARD = decltype(guard)::value;
        if (GUARD && kk >= n) return;
        const int l = l16(qf) + EF16 - lpp16(bA, tr);  // 16 log2|y_kk| (+ const)
        if (MODE == 0) {
            h[tr] = l;
        } else {
            const int sc = l + h[tr] + base;
            const bool up = sc > best;
            best = up ? sc : best;
            rr = up ? kk : rr;
        }
        if (!GUARD || kk < n - 1) {
            const double2 rw = *reinterpret_cast<const double2 *>(bA + (tr + RQ_HALO) * 2);
            const double D = fma_rn(rw.x, qf, pf);
            pf = fma_rn(-lam, D, mul_rn(rw.y, pf));
            qf = D;
        }
    };
    auto brow = [&](auto mode, auto guard, const double *bD, int tr, int kk, int base,
                    int (&h)[32]) {
        constexpr int MODE = decltype(mode)::value;
        constexpr bool GUARD = decltype(guard)::value;
        if (GUARD && kk >= n) return;
        const int l = l16(qb) + EB16 + lpp16(bD, tr);  // 16 log2|x_kk| (+ const)
        if (MODE == 0) {
            h[tr] = l;
        } else {
            const int sc = l + h[tr] + base;
            const bool up = sc > best;
            best = up ? sc : best;
            rr = up ? kk : rr;
        }
        if (kk > 0) {
            const double2 rw = *reinterpret_cast<const double2 *>(bD + (tr - 1 + RQ_HALO) * 2);
            const double E = fma_rn(rw.y, qb, pb);
            pb = fma_rn(-lam, E, mul_rn(rw.x, pb));
            qb = E;
        }
    };
    auto rescale2f = [&](double &x, double &y, int &E, int &E16) {
        rescale2(x, y, E);
        E16 = E << 4;
    };
    using M0 = std::integral_constant<int, 0>;
    using M1 = std::integral_constant<int, 1>;
    using G0 = std::integral_constant<bool, false>;
    using G1 = std::integral_constant<bool, true>;
    // -> 16 (value - tile maximum); clamped rows (code -127 in tiles flagged by hstore) come
    // back as -2^24: such a row is not a twist candidate -- clamping it to 127 units below
    // the tile maximum would overstate it, and where the other half-vector varies as fast the
    // opposite way (strongly localised eigenvectors, e.g. the spectrum ends of a
    // Householder-reduced T) that made a far row with |z_r| ~ 0 win the argmax
    auto hload = [&](int t, int (&h)[32], bool clamped) {
        const uint4 *src = hist + ((int64_t)t * A.S + slot) * 2;
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const uint4 v = src[u];
            const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int b = 0; b < 4; b++)
                    h[16 * u + 4 * q + b] = (int)(signed char)((w[q] >> (8 * b)) & 0xffu) * 16;
        }
        if (clamped) {  // (rows exactly 127 units below the maximum go too: no candidates)
#pragma unroll
            for (int r = 0; r < 32; r++) h[r] = h[r] == -127 * 16 ? -(1 << 24) : h[r];
        }
    };
    auto hstore = [&](int t, const int (&h)[32]) -> int {  // 2 x the tile maximum + clamp flag
        int m = INT_MIN, mn = INT_MAX;
#pragma unroll
        for (int r = 0; r < 32; r++) {
            m = max(m, h[r]);
            mn = min(mn, h[r]);
        }
        const bool clamped = mn == INT_MIN || ((mn - m + 8) >> 4) < -127;
        uint4 *dst = hist + ((int64_t)t * A.S + slot) * 2;
#pragma unroll
        for (int u = 0; u < 2; u++) {
            unsigned w[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                unsigned acc = 0;
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int hv = h[16 * u + 4 * q + b];
                    const int d = hv == INT_MIN ? -127 : max((hv - m + 8) >> 4, -127);  // nearest
                    acc |= ((unsigned)d & 0xffu) << (8 * b);
                }
                w[q] = acc;
            }
            dst[u] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return m * 2 + (clamped ? 1 : 0);
    };
    // both streams over one step's tiles, rows interleaved (fully unrolled: the packed
    // int16 rows live in registers)
    auto step = [&](auto mode, auto guard, const double *bA, int64_t tA, const double *bD,
                    int64_t tD, int basef, int baseb, int (&hf)[32], int (&hb)[32]) {
#pragma unroll
        for (int q = 0; q < RQ_TR / RQ_C; q++) {
            const int oF = q * RQ_C, oB = (RQ_TR / RQ_C - 1 - q) * RQ_C;
#pragma unroll
            for (int j = 0; j < RQ_C; j++) {
                frow(mode, guard, bA, oF + j, (int)tA + oF + j, basef, hf);
                brow(mode, guard, bD, oB + RQ_C - 1 - j, (int)tD + oB + RQ_C - 1 - j, baseb, hb);
            }
            rescale2f(pf, qf, EF, EF16);
            rescale2f(pb, qb, EB, EB16);
        }
    };
    dual_staged_pass<2>(
        sx, nd.repx, n, 0, ntile, ntile - 1, ntile,
        [&](const double *bA, int64_t tA, const double *bD, int64_t tD) {
            if (!active) return;
            const int iA = (int)(tA / RQ_TR), iD = (int)(tD / RQ_TR);
            const bool guard = tA + RQ_TR > n - 1 || tD + RQ_TR > n - 1 || tD == 0;
            int hf[32], hb[32];
#pragma unroll
            for (int u = 0; u < 32; u++) hf[u] = hb[u] = INT_MIN;
            if (2 * iA < ntile - 1) {  // first half: store
                if (guard)
                    step(M0{}, G1{}, bA, tA, bD, tD, 0, 0, hf, hb);
                else
                    step(M0{}, G0{}, bA, tA, bD, tD, 0, 0, hf, hb);
                cand[(int64_t)iA * A.S + slot] = hstore(iA, hf);
                cand[(int64_t)iD * A.S + slot] = hstore(iD, hb);
                return;
            }
            if (2 * iA == ntile - 1) {  // middle tile (odd ntile): F stores, then B scores
#pragma unroll
                for (int q = 0; q < RQ_TR / RQ_C; q++) {
#pragma unroll
                    for (int j = 0; j < RQ_C; j++)
                        frow(M0{}, G1{}, bA, q * RQ_C + j, (int)tA + q * RQ_C + j, 0, hf);
                    rescale2f(pf, qf, EF, EF16);
                }
                // (the same tile: F's values as they are, no quantisation)
                const int baseb = -logw(tD + RQ_TR / 2);
#pragma unroll
                for (int q = RQ_TR / RQ_C - 1; q >= 0; q--) {
#pragma unroll
                    for (int j = RQ_C - 1; j >= 0; j--)
                        brow(M1{}, G1{}, bD, q * RQ_C + j, (int)tD + q * RQ_C + j, baseb, hf);
                    rescale2f(pb, qb, EB, EB16);
                }
                return;
            }
            // second half: score every row against the other stream's stored value
            const int cA = cand[(int64_t)iA * A.S + slot], cD = cand[(int64_t)iD * A.S + slot];
            hload(iA, hf, (cA & 1) != 0);
            hload(iD, hb, (cD & 1) != 0);
            const int basef = (cA >> 1) - logw(tA + RQ_TR / 2);
            const int baseb = (cD >> 1) - logw(tD + RQ_TR / 2);
            if (guard)
                step(M1{}, G1{}, bA, tA, bD, tD, basef, baseb, hf, hb);
            else
                step(M1{}, G0{}, bA, tA, bD, tD, basef, baseb, hf, hb);
        },
        nd.pp);
    // F's candidates (tiles reached by F first) scored against B: B evaluated those in
    // its own later tiles; B's candidates scored by F likewise.  Rows scored: one per tile.
    if (active) A.it.twist[id] = (int32_t)rr;
}

// sort keys (node, twist index) of the singletons for k_rqi's CTA grouping
__global__ void k_twist_keys(const int32_t *__restrict__ list, int cnt,
                             const int32_t *__restrict__ item_node,
                             const int32_t *__restrict__ twist, unsigned long long *keys,
                             int32_t *vals) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const int id = list[t];
    keys[t] = ((unsigned long long)(unsigned)item_node[id] << 32) | (unsigned)twist[id];
    vals[t] = id;
}

// CTA tasks for k_rqi / k_bisect_s: runs of <= per consecutive items of the same node
// (one CTA of 1024 threads; two chunked scans).
__global__ void __launch_bounds__(1024) k_rqi_tasks(const int32_t *__restrict__ singles, int cnt,
                                                    const int32_t *__restrict__ item_node,
                                                    int32_t *seg_begin /* cnt+1 */,
                                                    RqiTask *tasks, int *ntasks, int per) {
    __shared__ int sh[33];
    __shared__ int carry[2];
    if (threadIdx.x < 2) carry[threadIdx.x] = 0;
    __syncthreads();
    // pass 1: node segments
    for (int base = 0; base < cnt; base += blockDim.x) {
        int p = base + threadIdx.x;
        int start = 0;
        if (p < cnt) start = (p == 0 || item_node[singles[p]] != item_node[singles[p - 1]]) ? 1 : 0;
        int tot;
        int ex = block_excl_scan(start, &tot, sh);
        if (p < cnt && start) seg_begin[carry[0] + ex] = p;
        __syncthreads();
        if (threadIdx.x == 0) carry[0] += tot;
        __syncthreads();
    }
    const int nseg = carry[0];
    if (threadIdx.x == 0) seg_begin[nseg] = cnt;
    __syncthreads();
    // pass 2: per segment, ceil(len / TPB) tasks
    for (int base = 0; base < nseg; base += blockDim.x) {
        int sgi = base + threadIdx.x;
        int nt = 0, b0 = 0, len = 0;
        if (sgi < nseg) {
            b0 = seg_begin[sgi];
            len = seg_begin[sgi + 1] - b0;
            nt = (len + per - 1) / per;
        }
        int tot;
        int ex = block_excl_scan(nt, &tot, sh);
        for (int q = 0; q < nt; q++) {
            RqiTask t;
            t.first = b0 + q * per;
            t.cnt = min(per, len - q * per);
            t.node = item_node[singles[b0]];
            t.pad = 0;
            tasks[carry[1] + ex + q] = t;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry[1] += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *ntasks = carry[1];
}

}  // namespace mr3
