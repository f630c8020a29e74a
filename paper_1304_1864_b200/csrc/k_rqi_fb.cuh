// k_rqi_fb.cuh -- K5 main phase: the first two RQI iterations of every singleton with the
// two halves of each twisted factorization in two threads (Alg. 1 l.11-12, PAPER.md
// L652-L727, L1140-L1173; the same arithmetic as k_rqi's fixed-twist pass, reading R9b/R9c).
//
// A fixed-twist factorization at lam with twist r is two independent recurrences that
// meet at r (SURVEY.md App. A in projective form, reading R8b):
//   F (stationary, rows 0..r-1, top-down):    D = d qF + pF,  pF <- lld pF - lam D,  qF <- D
//   B (progressive, rows n-1..r+1, bottom-up): E = lld_{k-1} qB + pB, pB <- d_{k-1} pB - lam E,
//                                               qB <- E
// joined by gamma_r = pF/qF + pB/qB + lam, ||z||^2 = 1 + W + V and the inertia of
// N_r Delta_r N_r^T (Sylvester).  k_rqi runs F and B interleaved in one thread (two chains,
// ILP 2); here every eigenpair owns TWO threads -- an F thread in the CTA's first two warps and
// a B thread in the last two -- so the SM scheduler interleaves the chains across warps (it
// picks any ready warp; a statically interleaved instruction stream stalls on the first
// unready one), and each thread carries one chain's state.  At the end of a pass the two
// threads exchange their end states through shared memory and evaluate the RQ correction, the
// stopping test (Eq. (3.6)) and the bracket update identically.
//
// Scope: iterations 1 and 2 (the non-storing pass at the RQI start and the storing pass that
// writes z in product form, k_zprod.cuh) -- all that almost every singleton needs (config 5:
// all but one of 50 000).  An eigenpair that is not finished after them is handed to k_rqi
// with its state (RqiResume: shift, bracket, scale references, flags), which continues with
// split passes (R9d) and the bisection fallback.  The Z columns of the finished eigenpairs are
// normalised by the CTA itself when it is done (as k_rqi's fused epilogue) or by k_zscale.
#pragma once
#include "k_rqi.cuh"

namespace mr3 {

constexpr int FB_NP = 64;           // eigenpairs per CTA
constexpr int FB_TPB = 2 * FB_NP;   // threads: F threads of pairs 0..63, then their B threads

template <class R>
struct FBX {  // end state of one half of a twisted factorization (exchanged through smem)
    R p, q;
    double nrm, s, c;  // W or V; Kahan sum of the written squares and its compensation
    int negc, E;
};

// dynamic shared memory: 4 staged tiles (rows + PP rows; after a pass they hold the exchanged
// end states, at the end the epilogue's column table), the two z tiles of a storing pass and
// the per-column store data.  33 KB in dd: 6 CTAs (768 threads) per SM, one wave for
// 50 000 eigenpairs on 148 SMs.
template <class R, class OutT>
constexpr size_t fb_smem_bytes() {
    return 4 * (size_t)(Stage<R>::TILE + PP_TILE) * sizeof(double) +
           2 * 16 * (size_t)(FB_NP + 1) * sizeof(OutT) + 2 * FB_NP * sizeof(int64_t) +
           4 * sizeof(int);
}
static_assert(2 * FB_NP * sizeof(FBX<dd>) <= 4 * (Stage<dd>::TILE + PP_TILE) * sizeof(double),
              "the exchange area aliases the staging tiles");

// DOT2: the row update in "two dot products" form -- p' = (lld - lam) p - (lam d) q and
// q' = d q + p (F; B likewise with d and lld exchanged) -- both from the state (p, q), so
// the dependent chain per row is one pair dot product instead of two pair FMAs in sequence;
// lld - lam and lam d are off the chain.  The same recurrence in exact arithmetic; every step
// is exact for data and shift perturbed by O(eps_y) relative (reading R8b).  ~40% more FP64
// instructions per row, about half the dependent latency.
template <class R, class OutT, bool DOT2>
__global__ void __launch_bounds__(FB_TPB, 6) k_rqi_fb(RqiArgs<R> A) {
    extern __shared__ __align__(16) double fb_dyn[];
    double *sstage = fb_dyn;
    OutT(*ztF)[FB_NP + 1] =
        reinterpret_cast<OutT(*)[FB_NP + 1]>(fb_dyn + 4 * (Stage<R>::TILE + PP_TILE));
    OutT(*ztB)[FB_NP + 1] = ztF + 16;
    int2 *s_rb = reinterpret_cast<int2 *>(ztB + 16);          // per column: F rows < x, B rows > y
    OutT **s_zp = reinterpret_cast<OutT **>(s_rb + FB_NP);    // per column: base pointer
    FBX<R> *xch = reinterpret_cast<FBX<R> *>(sstage);         // [2][FB_NP], between passes
    int *s_lim = reinterpret_cast<int *>(s_zp + FB_NP);       // rmin, rmax

    const int tid = threadIdx.x;
    const int role = tid / FB_NP;  // 0: F (top-down), 1: B (bottom-up); warp-uniform
    const int pi = tid - role * FB_NP;
    const RqiTask task = A.tasks[blockIdx.x];
    const NodeInfo nd = A.nodes[task.node];
    const int64_t n = nd.n;
    const bool active = pi < task.cnt;
    int id = -1, k = 0;
    R lam = mk<R>(0.0), a = lam, b = lam, gr = lam, lam_out = lam;
    double nz2 = 1.0, gap = INFINITY;
    int64_t r = 0;
    unsigned long long rows = 0;
    int iters = 0;
    bool done = !active;
    if (active) {
        id = A.list[task.first + pi];
        k = A.it.k[id];
        a = reinterpret_cast<const R *>(A.it.lo)[id];
        b = reinterpret_cast<const R *>(A.it.hi)[id];
        lam = half(add(a, b));
        if (A.root_widen > 0.0 && nd.depth == 0) {  // rigorous guard of a root bracket (R8d)
            const double wd = A.root_widen * (double)n * fmax(fabs(hi(a)), fabs(hi(b)));
            a = sub(a, mk<R>(wd));
            b = add(b, mk<R>(wd));
        }
        const double x0 = A.it.x0[id];
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
    if (tid == 0) {
        s_lim[0] = (int)n;
        s_lim[1] = 0;
    }
    __syncthreads();
    if (active && role == 0) {
        atomicMin(&s_lim[0], (int)r);
        atomicMax(&s_lim[1], (int)r);
    }
    __syncthreads();
    const int cta_rmin = s_lim[0] <= s_lim[1] ? s_lim[0] : 0;
    const int cta_rmax = s_lim[0] <= s_lim[1] ? s_lim[1] : (int)n - 1;

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
    if (zcol != nullptr && n == 1) {
        if (role == 0) zcol[0] = (OutT)1.0;
        zfinal = true;
    }

    using G0 = std::integral_constant<bool, false>;
    using G1 = std::integral_constant<bool, true>;
    // one fixed-twist factorization at lam for the eigenpairs with `need` (collective)
    // (STORE is a compile-time flag: the non-storing pass carries no z-store code per row)
    auto pass = [&](bool need, auto store_c) -> int {
        constexpr bool STORE = decltype(store_c)::value;
        if (need) zwritten = false;
        const R mlam = neg(lam);
        R px = mlam, qx = mk<R>(1.0);  // F: (pF, qF); B: (pB, qB)
        int Ex = 0, negc = 0;
        double nrm = 0.0, ks = 0.0, kc = 0.0;
        if (need && role == 1) px = sub(load_row4<R>(nd.rep, n - 1).d, lam);
        const int ntile = (int)((n + RQ_TR - 1) / RQ_TR);
        const int nA = cta_rmax / RQ_TR + 1;
        const int nD = ntile - cta_rmin / RQ_TR;
        const bool wz = STORE && need && zcol != nullptr;
        const int eref = role == 0 ? erefF : erefB;
        auto rescale = [](R &x, R &y, int &E) {
            const unsigned ex = (unsigned)__double2hiint(hi(x)) & 0x7ff00000u;
            const unsigned ey = (unsigned)__double2hiint(hi(y)) & 0x7ff00000u;
            const unsigned em = ex > ey ? ex : ey;
            if (em == 0x7ff00000u || em == 0u) return;
            const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
            x = scale_pow2(x, sc);
            y = scale_pow2(y, sc);
            E += (int)(em >> 20) - 1023;
        };
        auto sppr = [&](const double *buf, int64_t t0, int64_t kk, double &pm, double &ipm,
                        int &e) {
            const double2 *q = reinterpret_cast<const double2 *>(
                buf + Stage<R>::TILE + (kk - t0 + RQ_HALO) * 4);
            const double2 a0 = q[0], a1 = q[1];
            pm = a0.x;
            ipm = a0.y;
            e = __double2loint(a1.x);
        };
        // F row kk (< r): y_kk = qF / PP_kk is component kk of the product-form z
        // (zt: this thread's slot of the z tile row kk; a storing pass computes and stages the
        // component unconditionally -- columns not written are masked by s_rb at the flush)
        auto frow = [&](auto guard, const double *bA, int64_t tA, int64_t kk, OutT *zt) {
            constexpr bool GUARD = decltype(guard)::value;
            const Row4<R> rw = srow<R>(bA, tA, kk);
            const R D = fma_dd(rw.d, qx, px);
            // (a storing pass takes ||z||^2 from the written squares, R9e: no norm identity)
            double N2 = 0.0;
            if (!STORE) {
                const double lpx = hi(rw.ld) * hi(qx) * rcp_w(hi(D));  // l+ = ld / d+
                const double l2 = lpx * lpx;
                N2 = clampbig(fma(l2, nrm, l2));
            }
            const R p2 = DOT2 ? dot2_dd(add(rw.lld, mlam), px, mul(mlam, rw.d), qx)
                              : dot2_dd(mlam, D, rw.lld, px);
            if (!GUARD || (int)kk < (int)r) {
                if (STORE) {
                    double pm, ipm;
                    int e;
                    sppr(bA, tA, kk, pm, ipm, e);
                    const OutT zo = (OutT)pow2mul_d(hi(qx) * ipm, Ex - e - eref);
                    *zt = zo;
                    kahan_sq((double)zo, ks, kc);
                }
                negc += sgn_ne_R<R>(D, qx);
                if (!STORE) nrm = N2;
                px = p2;
                qx = D;
            }
        };
        // B row kk (> r): x_kk = QB PP_kk
        auto brow = [&](auto guard, const double *bD, int64_t tD, int64_t kk, OutT *zt) {
            constexpr bool GUARD = decltype(guard)::value;
            const Row4<R> rw = srow<R>(bD, tD, kk - 1);
            const R E = fma_dd(rw.lld, qx, px);
            double N2 = 0.0;
            if (!STORE) {
                const double ux = hi(rw.ld) * hi(qx) * rcp_w(hi(E));  // u- = l d / D-
                const double u2 = ux * ux;
                N2 = clampbig(fma(u2, nrm, u2));
            }
            const R P2 = DOT2 ? dot2_dd(add(rw.d, mlam), px, mul(mlam, rw.lld), qx)
                              : dot2_dd(mlam, E, rw.d, px);
            if (!GUARD || ((int)kk > (int)r && (int)kk < (int)n)) {
                if (STORE) {
                    double pm, ipm;
                    int e;
                    sppr(bD, tD, kk, pm, ipm, e);
                    const OutT zo = (OutT)pow2mul_d(hi(qx) * pm, Ex + e - eref);
                    *zt = zo;
                    kahan_sq((double)zo, ks, kc);
                }
                negc += sgn_ne_R<R>(E, qx);
                if (!STORE) nrm = N2;
                px = P2;
                qx = E;
            }
        };
        const bool cta_store = STORE && A.jobz_v;  // uniform over the CTA
        if (cta_store && role == 0) {
            s_rb[pi] = wz ? make_int2((int)r, (int)r) : make_int2(-1, INT_MAX);
            s_zp[pi] = wz ? reinterpret_cast<OutT *>(A.Z) + (col0 - A.zcol0) * A.ldz + nd.row0
                          : nullptr;
        }
        // the written components of one 16-row half tile per stream leave as coalesced
        // 128-byte column segments (each half-warp writes 16 rows of one column)
        auto flush = [&](const double *bA, int64_t tA, int hA, const double *bD, int64_t tD,
                         int hD) {
            __syncthreads();
            const int warp = tid >> 5, lane = tid & 31, row = lane & 15;
            const int gA = bA != nullptr ? (int)tA + 16 * hA + row : INT_MAX;
            const int gD = (bD != nullptr && (int)tD + 16 * hD + row < (int)n)
                               ? (int)tD + 16 * hD + row
                               : INT_MIN;
#pragma unroll 4
            for (int c = 2 * warp + (lane >> 4); c < FB_NP; c += 2 * (FB_TPB / 32)) {
                const int2 rb = s_rb[c];
                if (gA < rb.x) s_zp[c][gA] = ztF[row][c];
                if (gD > rb.y) s_zp[c][gD] = ztB[row][c];
            }
            __syncthreads();
        };
        dual_staged_pass<Stage<R>::ROWD>(
            sstage, nd.rep, n, 0, nA, ntile - 1, nD,
            [&](const double *bA, int64_t tA, const double *bD, int64_t tD) {
#pragma unroll 1
                for (int h = 0; h < 2; h++) {
                    if (need) {
                        if (role == 0) {
                            if (bA != nullptr) {
#pragma unroll 1
                                for (int q = 2 * h; q < 2 * h + 2; q++) {
                                    const int64_t b0 = tA + q * RQ_C;
                                    OutT *zt = &ztF[(q & 1) * RQ_C][pi];
                                    if (b0 + RQ_C <= cta_rmin) {  // below every twist: no guard
#pragma unroll
                                        for (int j = 0; j < RQ_C; j++)
                                            frow(G0{}, bA, tA, b0 + j, zt + j * (FB_NP + 1));
                                        rescale(px, qx, Ex);
                                    } else if (b0 < r) {
#pragma unroll
                                        for (int j = 0; j < RQ_C; j++)
                                            frow(G1{}, bA, tA, b0 + j, zt + j * (FB_NP + 1));
                                        rescale(px, qx, Ex);
                                    }
                                }
                            }
                        } else if (bD != nullptr) {
#pragma unroll 1
                            for (int q = 2 * h; q < 2 * h + 2; q++) {
                                const int64_t b0 = tD + (RQ_TR / RQ_C - 1 - q) * RQ_C;
                                OutT *zt = &ztB[((RQ_TR / RQ_C - 1 - q) & 1) * RQ_C][pi];
                                if (b0 > cta_rmax && b0 + RQ_C <= n) {  // above every twist
#pragma unroll
                                    for (int j = 0; j < RQ_C; j++)
                                        brow(G0{}, bD, tD, b0 + RQ_C - 1 - j,
                                             zt + (RQ_C - 1 - j) * (FB_NP + 1));
                                    rescale(px, qx, Ex);
                                } else if (b0 + RQ_C > r && b0 < n) {
#pragma unroll
                                    for (int j = 0; j < RQ_C; j++)
                                        brow(G1{}, bD, tD, b0 + RQ_C - 1 - j,
                                             zt + (RQ_C - 1 - j) * (FB_NP + 1));
                                    rescale(px, qx, Ex);
                                }
                            }
                        }
                    }
                    if (cta_store) flush(bA, tA, h, bD, tD, 1 - h);
                }
            },
            cta_store ? nd.pp : nullptr);
        // exchange the end states; both threads of a pair evaluate the same join
        FBX<R> mine;
        mine.p = px;
        mine.q = qx;
        mine.nrm = nrm;
        mine.s = ks;
        mine.c = kc;
        mine.negc = negc;
        mine.E = Ex;
        xch[role * FB_NP + pi] = mine;
        __syncthreads();
        const FBX<R> F = role == 0 ? mine : xch[pi];
        const FBX<R> B = role == 1 ? mine : xch[FB_NP + pi];
        __syncthreads();  // (xch is rewritten by the next pass)
        int negt = 0;
        if (need) {
            gr = add(add(div(F.p, F.q), div(B.p, B.q)), lam);
            negt = F.negc + B.negc + (is_neg(gr) ? 1 : 0);
            rows += n;
            double pm = 1.0, ipm = 1.0;
            int e = 0;
            if (nd.pp != nullptr) {
                const double2 *q = reinterpret_cast<const double2 *>(nd.pp + r * PP_STRIDE);
                const double2 a0 = __ldg(q), a1 = __ldg(q + 1);
                pm = a0.x;
                ipm = a0.y;
                e = __double2loint(a1.x);
            }
            const double yr = hi(F.q) * ipm, xr = hi(B.q) * pm;
            const int eyr = F.E - e, exr = B.E + e;
            if (STORE) {  // ||z||^2 = the sum of the written squares in z_r = 1 units (R9e)
                const OutT zo = (OutT)pow2mul_d(yr, eyr - erefF);
                double sF = F.s, cF_ = F.c;
                kahan_sq((double)zo, sF, cF_);
                const double fF = ldexp(1.0, erefF - eyr) / yr;
                const double fB = ldexp(1.0, erefB - exr) / xr;
                const double ss = fF * fF * sF + fB * fB * B.s;
                nz2 = nz2_of_ss(ss);
                if (wz) {
                    if (role == 0) zcol[r] = zo;
                    zinfo.cF = fF;
                    zinfo.cB = fB;
                    zinfo.ss = ss;
                    zwritten = true;
                }
            } else {
                nz2 = 1.0 + F.nrm + B.nrm;
            }
            erefF = eyr + expo_of(yr);
            erefB = exr + expo_of(xr);
        }
        return negt;
    };

    const int maxit = A.maxit < 2 ? A.maxit : 2;
    int passes = 0;  // passes this eigenpair took part in
#pragma unroll 1
    for (iters = 1; iters <= maxit; iters++) {
        const bool store_only =
            A.jobz_v && iters >= 2 && done && !zfinal && zcol != nullptr && n > 1;
        const bool need = !done || store_only;
        if (!__syncthreads_or(need)) break;
        const int c = (A.jobz_v && iters >= 2) ? pass(need, std::integral_constant<bool, true>{})
                                                : pass(need, std::integral_constant<bool, false>{});
        if (need) passes = iters;
        if (store_only) zfinal = zwritten;
        if (need && !store_only) {
            if (c >= k) {
                if (lt(lam, b)) b = lam;
            } else {
                if (lt(a, lam)) a = lam;
            }
            const double g = hi(gr);
            const double corr = g / nz2;
            R lam_new = add(lam, mk<R>(corr));
            if (fabs(g) / sqrt(nz2) <= tol || fabs(corr) <= 8.0 * Prec<R>::eps * fabs(hi(lam)) ||
                g == 0.0) {
                lam_out = lam_new;
                done = true;
                zfinal = zwritten;
            } else {
                if (!(lt(a, lam_new) && lt(lam_new, b))) lam_new = half(add(a, b));
                lam = lam_new;
            }
        }
    }
    // finished: converged with z in Z (or no vectors wanted); otherwise k_rqi continues
    const bool finished = active && done && (zfinal || zcol == nullptr);
    if (active && role == 0) {
        A.left[task.first + pi] = finished ? 0 : 1;
        if (finished) {
            const R lt_ = add(lam_out, mk2<R>(nd.sig_hi, nd.sig_lo));
            if (col0 >= 0) {
                if (sizeof(OutT) == 4)
                    reinterpret_cast<float *>(A.w)[col0] = (float)(hi(lt_) * A.unscale);
                else
                    reinterpret_cast<double *>(A.w)[col0] = hi(lt_) * A.unscale;
            }
            reinterpret_cast<R *>(A.it.lo)[id] = lam_out;
            atomicMax(&A.st->rqi_iters_max, passes);
            if (A.dbg_iters) A.dbg_iters[id] = passes;
            if (zcol != nullptr) A.zc[col0 - A.zcol0] = zinfo;
        } else {
            RqiResume<R> rs;
            rs.lam = lam;
            rs.a = a;
            rs.b = b;
            rs.lam_out = lam_out;
            rs.iters = passes;
            rs.erefF = erefF;
            rs.erefB = erefB;
            rs.flags = (done ? 1 : 0) | (zfinal ? 2 : 0);
            A.resume[id] = rs;
        }
        if (rows) atomicAdd(&A.st->rqi_rows, rows);
    }
    // K6 epilogue: normalise the finished columns of this CTA (collective)
    if (!A.jobz_v || !A.fuse_scale) return;
    ZCol *szc = reinterpret_cast<ZCol *>(sstage);
    OutT **szp = reinterpret_cast<OutT **>(szc + FB_NP);
    __syncthreads();
    if (role == 0) {
        szc[pi] = zinfo;
        szp[pi] = finished ? zcol : nullptr;
    }
    __syncthreads();
    constexpr int V = 16 / sizeof(OutT);
    using Vec = typename std::conditional<sizeof(OutT) == 8, double2, float4>::type;
#pragma unroll 1
    for (int j = 0; j < FB_NP; j++) {
        OutT *col = szp[j];
        if (col == nullptr) continue;  // (uniform)
        const ZCol z = szc[j];
        const double inv = 1.0 / sqrt(z.ss);
        const double fF = z.cF * inv, fB = z.cB * inv;
        const int64_t nn = z.n;
        const bool aligned = (reinterpret_cast<uintptr_t>(col) & 15) == 0;
        const int64_t nv = aligned ? nn / V : 0;
        Vec *cv = reinterpret_cast<Vec *>(col);
        constexpr int U = 8;
#pragma unroll 1
        for (int64_t b0 = 0; b0 < nv; b0 += (int64_t)U * FB_TPB) {
            Vec v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t i = b0 + u * FB_TPB + tid;
                if (i < nv) v[u] = cv[i];
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t i = b0 + u * FB_TPB + tid;
                if (i < nv) {
                    OutT *e = reinterpret_cast<OutT *>(&v[u]);
#pragma unroll
                    for (int q = 0; q < V; q++)
                        e[q] = (OutT)((double)e[q] * (i * V + q <= z.r ? fF : fB));
                    cv[i] = v[u];
                }
            }
        }
        for (int64_t i = nv * V + tid; i < nn; i += FB_TPB)
            col[i] = (OutT)((double)col[i] * (i <= z.r ? fF : fB));
    }
}

}  // namespace mr3
