// k_rqi.cuh -- K5 + K6: singleton eigenpairs by Rayleigh quotient iteration on
// twisted factorizations, then normalisation, rounding to binary_x and the
// coalesced store of the Z column (Alg. 1 l.11-12, PAPER.md L652-L727,
// L1140-L1173; memory contract L1199-L1226).
//
// One thread per eigenpair.  Iteration j at shift lam:
//   F (stationary, top-down):   s_1 = -lam ; d+_i = d_i + s_i ; l+_i = ld_i / d+_i ;
//                               s_{i+1} = l+_i l_i s_i - lam ; count #{d+_i < 0}
//   B (progressive, bottom-up): p_n = d_n - lam ; D-_{i+1} = lld_i + p_{i+1} ;
//                               t = d_i / D-_{i+1} ; u-_i = l_i t ; p_i = p_{i+1} t - lam
//   gamma_k = s_k + p_k + lam ; r = argmin |gamma_k| (ties: smallest k)
//   ||z||^2 for twist k = 1 + W_k + V_k with the prefix norms
//       W_{k+1} = (l+_k)^2 (1 + W_k),  V_{k-1} = (u-_{k-1})^2 (1 + V_k)
//   (exact identities for z_r = 1, z_i = -l+_i z_{i+1} (i < r), z_{i+1} = -u-_i z_i),
//   kept in binary64: they only feed the RQ correction and the stopping test.
//   The output is normalised with that estimate and the exact ||z|| is summed
//   (pair arithmetic) while the column is written; k_fixnorm rescales the few
//   columns whose estimate was off by more than 2^-54.
//   lam <- lam + gamma_r / ||z||^2          (RQ correction, L714-L717)
//   stop: |gamma_r|/||z|| <= k_rs gap eps_x sqrt(n)   (Eq. (3.6))
//         or |gamma_r|/||z||^2 <= 8 eps_y |lam|        (stagnation, L720-L723)
// The iterate is kept inside the certified bracket (F's count updates it); an
// iterate leaving it is replaced by the bracket midpoint (RQI "guarded by
// bisection", L315); after max_rqi iterations: bisection to relative
// eps_x sqrt(n) gaptol and one more twisted solve (L1154-L1163).
//
// Storage: the forward state (s, W) and backward state p are checkpointed every
// C rows (6 B/row/eigenpair in dd) instead of storing whole sweeps; each block
// of C rows is recomputed into registers when a sweep needs it in the other
// direction (SURVEY.md §7 hard part 2, option (c)).
#pragma once
#include "k_bisect.cuh"

namespace mr3 {

constexpr int RQ_C = 8;     // checkpoint block (rows)
constexpr int RQ_TR = 32;   // output tile rows (4 checkpoint blocks)
constexpr int RQ_TPB = 128; // threads per CTA

template <class R>
struct RqiArgs {
    const NodeInfo *nodes;
    Items it;
    const int32_t *list;
    int cnt;
    R *ck_s, *ck_p;         // [nblk][S]
    double *ck_W;           // [nblk][S]
    double *fac;            // per local column: 1/||written column|| (fp64 output), 0 = exact
    int64_t S;              // checkpoint stride (threads in this launch)
    double pivmin, krs, eps_x, gaptol;
    int maxit;
    int jobz_v;
    void *w;          // eigenvalue output (global positions)
    void *Z;          // eigenvector output (columns col - zcol0)
    int64_t ldz, zcol0;
    double unscale;   // multiply eigenvalues by this (exact power of 2)
    DevStats *st;
};

__device__ __forceinline__ double clampbig(double x) { return fmin(x, 1e250); }

// ss += x^2 in pair arithmetic (two-prod + two-sum)
__device__ __forceinline__ void accum_sq(double x, double &sh, double &sl) {
    double p = x * x;
    double pe = fma(x, x, -p);
    double e;
    double sn = two_sum(sh, p, e);
    sl += e + pe;
    sh = sn;
}

// F sweep with checkpoints; returns count(lam)
template <class R>
__device__ __forceinline__ int rq_forward(const double *__restrict__ rep, int64_t n, R lam,
                                          double pivmin, R *ck_s, double *ck_W, int64_t S,
                                          int64_t slot) {
    R s = neg(lam);
    double W = 0.0;
    int negc = 0;
#pragma unroll 1
    for (int64_t b0 = 0; b0 < n; b0 += RQ_C) {
        ck_s[(b0 / RQ_C) * S + slot] = s;
        ck_W[(b0 / RQ_C) * S + slot] = W;
#pragma unroll
        for (int j = 0; j < RQ_C; j++) {
            int64_t k = b0 + j;
            if (k < n) {
                Row4<R> r = load_row4<R>(rep, k);
                R dp = guard(add(r.d, s), pivmin);
                negc += is_neg(dp) ? 1 : 0;
                if (k < n - 1) {
                    R lp = div(r.ld, dp);
                    double l2 = hi(lp) * hi(lp);
                    W = clampbig(fma(l2, W, l2));
                    s = sub(mul(lp, mul(r.l, s)), lam);
                }
            }
        }
    }
    return negc;
}

// B sweep: recompute each forward block, argmin |gamma_k|, norms, p checkpoints
template <class R>
__device__ __forceinline__ void rq_backward(const double *__restrict__ rep, int64_t n, R lam,
                                            double pivmin, const R *ck_s, const double *ck_W,
                                            R *ck_p, int64_t S, int64_t slot, int64_t &r_out,
                                            R &g_out, double &nz2_out) {
    Row4<R> rl = load_row4<R>(rep, n - 1);
    R p = sub(rl.d, lam);
    double V = 0.0;
    double best = INFINITY;
    int64_t r = n - 1;
    R gr = mk<R>(0.0);
    double nz2 = 1.0;
    const int64_t nblk = (n + RQ_C - 1) / RQ_C;
#pragma unroll 1
    for (int64_t blk = nblk - 1; blk >= 0; blk--) {
        const int64_t b0 = blk * RQ_C;
        R sbuf[RQ_C];
        double wbuf[RQ_C];
        R s = ck_s[blk * S + slot];
        double W = ck_W[blk * S + slot];
#pragma unroll
        for (int j = 0; j < RQ_C; j++) {
            int64_t k = b0 + j;
            sbuf[j] = s;
            wbuf[j] = W;
            if (k < n - 1) {
                Row4<R> r4 = load_row4<R>(rep, k);
                R dp = guard(add(r4.d, s), pivmin);
                R lp = div(r4.ld, dp);
                double l2 = hi(lp) * hi(lp);
                W = clampbig(fma(l2, W, l2));
                s = sub(mul(lp, mul(r4.l, s)), lam);
            }
        }
#pragma unroll
        for (int j = RQ_C - 1; j >= 0; j--) {
            int64_t k = b0 + j;
            if (k < n) {
                if (j == 0) ck_p[blk * S + slot] = p;  // p at the block start
                R g = add(add(sbuf[j], p), lam);
                double ga = fabs(hi(g));
                if (ga <= best) {
                    best = ga;
                    r = k;
                    gr = g;
                    nz2 = 1.0 + wbuf[j] + V;
                }
                if (k > 0) {
                    Row4<R> r4 = load_row4<R>(rep, k - 1);
                    R Dm = guard(add(r4.lld, p), pivmin);
                    R t = div(r4.d, Dm);
                    double u2 = hi(r4.l) * hi(t);
                    u2 *= u2;
                    V = clampbig(fma(u2, V, u2));
                    p = sub(mul(p, t), lam);
                }
            }
        }
    }
    r_out = r;
    g_out = gr;
    nz2_out = nz2;
}

template <class R, class OutT>
__global__ void __launch_bounds__(RQ_TPB) k_rqi(RqiArgs<R> A) {
    __shared__ OutT tile[RQ_TR][RQ_TPB + 1];
    __shared__ int64_t s_r[RQ_TPB], s_n[RQ_TPB], s_row0[RQ_TPB], s_col[RQ_TPB];
    __shared__ int64_t s_nmax;

    const int tid = threadIdx.x;
    const int64_t slot = (int64_t)blockIdx.x * RQ_TPB + tid;
    const bool active = slot < A.cnt;
    int id = -1;
    NodeInfo nd;
    nd.n = 0;
    nd.rep = nullptr;
    nd.row0 = 0;
    int k = 0;
    R lam = mk<R>(0.0), a = lam, b = lam, gr = lam, lam_out = lam;
    double nz2 = 1.0;
    int64_t r = 0;
    double gap = INFINITY;
    unsigned long long rows = 0;
    int iters = 0;
    bool fallback = false;

    if (active) {
        id = A.list[slot];
        nd = A.nodes[A.it.node[id]];
        k = A.it.k[id];
        a = reinterpret_cast<const R *>(A.it.lo)[id];
        b = reinterpret_cast<const R *>(A.it.hi)[id];
        lam = half(add(a, b));
        gap = fmin(A.it.lgap[id], A.it.rgap[id]);
        if (!(gap > 0.0)) gap = fmax(hi(sub(b, a)), 1e-300);
        const double tol = A.krs * gap * A.eps_x * sqrt((double)nd.n);
        bool done = false;
        if (nd.n == 1) {  // 1x1 block: the eigenpair is (d_1, e_1) exactly
            lam_out = load_row4<R>(nd.rep, 0).d;
            r = 0;
            nz2 = 1.0;
            done = true;
            iters = 0;
        }
#pragma unroll 1
        for (iters = 1; !done && iters <= A.maxit; iters++) {
            int c = rq_forward<R>(nd.rep, nd.n, lam, A.pivmin, A.ck_s, A.ck_W, A.S, slot);
            rq_backward<R>(nd.rep, nd.n, lam, A.pivmin, A.ck_s, A.ck_W, A.ck_p, A.S, slot, r, gr,
                           nz2);
            rows += 3 * nd.n;
            if (c >= k) {
                if (lt(lam, b)) b = lam;
            } else {
                if (lt(a, lam)) a = lam;
            }
            double g = hi(gr), z2 = nz2;
            double corr = g / z2;
            R lam_new = add(lam, mk<R>(corr));
            if (fabs(g) / sqrt(z2) <= tol ||
                fabs(corr) <= 8.0 * Prec<R>::eps * fabs(hi(lam)) || g == 0.0) {
                lam_out = lam_new;
                done = true;
                break;
            }
            if (!(lt(a, lam_new) && lt(lam_new, b))) lam_new = half(add(a, b));
            lam = lam_new;
        }
        if (!done && nd.n > 1) {
            // fallback: bisection to relative eps_x sqrt(n) gaptol, one more solve
            fallback = true;
            double rtol = A.eps_x * sqrt((double)nd.n) * A.gaptol;
#pragma unroll 1
            for (int it2 = 0; it2 < 400; it2++) {
                R w = sub(b, a);
                if (hi(w) <= fmax(2.0 * rtol * fmax(fabs(hi(a)), fabs(hi(b))), 1e-300)) break;
                R mid = half(add(a, b));
                if (!(lt(a, mid) && lt(mid, b))) break;
                if (negcount<R>(nd.rep, nd.n, mid, A.pivmin) >= k)
                    b = mid;
                else
                    a = mid;
                rows += nd.n;
            }
            lam = half(add(a, b));
            rq_forward<R>(nd.rep, nd.n, lam, A.pivmin, A.ck_s, A.ck_W, A.S, slot);
            rq_backward<R>(nd.rep, nd.n, lam, A.pivmin, A.ck_s, A.ck_W, A.ck_p, A.S, slot, r, gr,
                           nz2);
            rows += 3 * nd.n;
            R lam_new = add(lam, mk<R>(hi(gr) / nz2));
            lam_out = (lt(a, lam_new) && lt(lam_new, b)) ? lam_new : lam;
            atomicAdd(&A.st->rqi_fallbacks, 1);
            iters = A.maxit + 1;
        }
        // eigenvalue output: w = (lambda[M] + sigma) * 2^-scale  (Alg. 1 l.12)
        R lt_ = add(lam_out, mk2<R>(nd.sig_hi, nd.sig_lo));
        int64_t col = A.it.col[id];
        if (col >= 0) {
            if (sizeof(OutT) == 4)
                reinterpret_cast<float *>(A.w)[col] = (float)(hi(lt_) * A.unscale);
            else
                reinterpret_cast<double *>(A.w)[col] = hi(lt_) * A.unscale;
        }
        reinterpret_cast<R *>(A.it.lo)[id] = lam_out;  // keep lambda[M] for diagnostics
        atomicMax(&A.st->rqi_iters_max, iters);
    }
    if (!A.jobz_v) {
        if (active && rows) atomicAdd(&A.st->rqi_rows, rows);
        return;
    }

    // ---------------- final stage: z from the twisted factorization at lam -----
    int64_t col = active ? A.it.col[id] : -1;
    s_r[tid] = r;
    s_n[tid] = active ? nd.n : 0;
    s_row0[tid] = nd.row0;
    s_col[tid] = col - A.zcol0;
    if (tid == 0) s_nmax = 0;
    __syncthreads();
    if (active && col >= 0) atomicMax((unsigned long long *)&s_nmax, (unsigned long long)nd.n);
    __syncthreads();
    const int64_t nmax = s_nmax;
    const bool mine = active && col >= 0;
    // 1/||z|| from the binary64 norm estimate; the exact norm of what is written
    // is summed in pair arithmetic (ss) and checked at the end
    const double inv = 1.0 / sqrt(nz2);
    double ss_hi = 0.0, ss_lo = 0.0;
    const double tiny = 1e-250;
    OutT *Zo = reinterpret_cast<OutT *>(A.Z);
    const int warp = tid >> 5, lane = tid & 31;

    // D sweep: rows k <= r, top-down tiles from the last one, z_r = 1,
    // z_k = -l+_k z_{k+1}  (z_k = -(ld_{k+1}/ld_k) z_{k+2} if z_{k+1} == 0)
    {
        R z1 = mk<R>(0.0), z2 = mk<R>(0.0);  // z_{k+1}, z_{k+2}
        const int64_t ntile = (nmax + RQ_TR - 1) / RQ_TR;
#pragma unroll 1
        for (int64_t tt = ntile - 1; tt >= 0; tt--) {
            const int64_t t0 = tt * RQ_TR;
            if (mine && t0 <= r) {
#pragma unroll 1
                for (int q = RQ_TR / RQ_C - 1; q >= 0; q--) {
                    const int64_t b0 = t0 + q * RQ_C;
                    if (b0 > r || b0 >= nd.n) continue;
                    R lpb[RQ_C];
                    R s = A.ck_s[(b0 / RQ_C) * A.S + slot];
#pragma unroll
                    for (int j = 0; j < RQ_C; j++) {
                        int64_t kk = b0 + j;
                        lpb[j] = mk<R>(0.0);
                        if (kk < nd.n - 1 && kk < r) {
                            Row4<R> r4 = load_row4<R>(nd.rep, kk);
                            R dp = guard(add(r4.d, s), A.pivmin);
                            R lp = div(r4.ld, dp);
                            lpb[j] = lp;
                            s = sub(mul(lp, mul(r4.l, s)), lam);
                        }
                    }
#pragma unroll
                    for (int j = RQ_C - 1; j >= 0; j--) {
                        int64_t kk = b0 + j;
                        if (kk > r || kk >= nd.n) continue;
                        R z;
                        if (kk == r) {
                            z = mk<R>(1.0);
                        } else if (hi(z1) == 0.0 && fabs(hi(z2)) > tiny) {
                            Row4<R> ra = load_row4<R>(nd.rep, kk);
                            Row4<R> rb = load_row4<R>(nd.rep, kk + 1);
                            z = neg(mul(div(rb.ld, ra.ld), z2));
                        } else {
                            z = neg(mul(lpb[j], z1));
                        }
                        if (fabs(hi(z)) < tiny) z = mk<R>(0.0);
                        OutT zo = (OutT)hi(mul(z, inv));
                        tile[kk - t0][tid] = zo;
                        accum_sq((double)zo, ss_hi, ss_lo);
                        z2 = z1;
                        z1 = z;
                    }
                }
            }
            __syncthreads();
            for (int c = warp; c < RQ_TPB; c += RQ_TPB / 32) {
                const int64_t row = t0 + lane;
                if (s_col[c] >= 0 && s_n[c] > 0 && row < s_n[c] && row <= s_r[c])
                    Zo[(s_row0[c] + row) + s_col[c] * A.ldz] = tile[lane][c];
            }
            __syncthreads();
        }
        if (mine) rows += r + 1;
    }
    // U sweep: rows k > r, bottom-up tiles, z_k = -u-_{k-1} z_{k-1}
    // (z_k = -(ld_{k-2}/ld_{k-1}) z_{k-2} if z_{k-1} == 0)
    {
        R z1 = mk<R>(0.0), z2 = mk<R>(0.0);  // z_{k-1}, z_{k-2}
        R ucarry = mk<R>(0.0);              // u-_{b0-1}
        const int64_t ntile = (nmax + RQ_TR - 1) / RQ_TR;
#pragma unroll 1
        for (int64_t tt = 0; tt < ntile; tt++) {
            const int64_t t0 = tt * RQ_TR;
            if (mine && t0 + RQ_TR - 1 >= r) {
#pragma unroll 1
                for (int q = 0; q < RQ_TR / RQ_C; q++) {
                    const int64_t b0 = t0 + q * RQ_C;
                    if (b0 + RQ_C - 1 < r || b0 >= nd.n) continue;
                    // recompute u-_k for k in [b0, e), e = min(b0 + C, n - 1)
                    R ub[RQ_C];
                    const int64_t e = (b0 + RQ_C < nd.n - 1) ? b0 + RQ_C : nd.n - 1;
                    R p;
                    if (e == b0 + RQ_C)
                        p = A.ck_p[((b0 + RQ_C) / RQ_C) * A.S + slot];
                    else
                        p = sub(load_row4<R>(nd.rep, nd.n - 1).d, lam);
#pragma unroll
                    for (int j = RQ_C - 1; j >= 0; j--) {
                        int64_t kk = b0 + j;
                        ub[j] = mk<R>(0.0);
                        if (kk < e) {
                            Row4<R> r4 = load_row4<R>(nd.rep, kk);
                            R Dm = guard(add(r4.lld, p), A.pivmin);
                            R t = div(r4.d, Dm);
                            ub[j] = mul(r4.l, t);
                            p = sub(mul(p, t), lam);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < RQ_C; j++) {
                        int64_t kk = b0 + j;
                        R uprev = (j == 0) ? ucarry : ub[j == 0 ? 0 : j - 1];
                        if (kk < nd.n) {
                            if (kk == r) {
                                z1 = mk<R>(1.0);
                                z2 = mk<R>(0.0);
                            } else if (kk > r) {
                                R z;
                                if (hi(z1) == 0.0 && fabs(hi(z2)) > tiny) {
                                    Row4<R> ra = load_row4<R>(nd.rep, kk - 2);
                                    Row4<R> rb = load_row4<R>(nd.rep, kk - 1);
                                    z = neg(mul(div(ra.ld, rb.ld), z2));
                                } else {
                                    z = neg(mul(uprev, z1));
                                }
                                if (fabs(hi(z)) < tiny) z = mk<R>(0.0);
                                OutT zo = (OutT)hi(mul(z, inv));
                                tile[kk - t0][tid] = zo;
                                accum_sq((double)zo, ss_hi, ss_lo);
                                z2 = z1;
                                z1 = z;
                            }
                        }
                    }
                    ucarry = ub[RQ_C - 1];
                }
            }
            __syncthreads();
            for (int c = warp; c < RQ_TPB; c += RQ_TPB / 32) {
                const int64_t row = t0 + lane;
                if (s_col[c] >= 0 && s_n[c] > 0 && row < s_n[c] && row > s_r[c])
                    Zo[(s_row0[c] + row) + s_col[c] * A.ldz] = tile[lane][c];
            }
            __syncthreads();
        }
        if (mine) rows += nd.n - r;
    }
    if (mine && A.fac) {
        // exact sum of squares of the written column vs 1 (fp64 output only)
        double dev = (ss_hi - 1.0) + ss_lo;
        A.fac[col - A.zcol0] = fabs(dev) > 0x1p-54 ? 1.0 / sqrt(ss_hi + ss_lo) : 0.0;
    }
    if (active && rows) atomicAdd(&A.st->rqi_rows, rows);
}

// rescale the columns whose binary64 norm estimate missed by more than 2^-54
// (one CTA per column; columns with fac == 0 are already unit vectors)
template <class OutT>
__global__ void k_fixnorm(OutT *Z, int64_t ldz, int64_t ncols, const double *fac,
                          const int64_t *row0n /* unused: whole column */, int64_t n) {
    const int64_t c = blockIdx.x;
    if (c >= ncols) return;
    const double f = fac[c];
    if (f == 0.0) return;
    OutT *col = Z + c * ldz;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) col[i] = (OutT)((double)col[i] * f);
}

}  // namespace mr3
