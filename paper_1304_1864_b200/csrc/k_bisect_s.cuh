// k_bisect_s.cuh -- K2: batched bisection / multisection with CTA-synchronous Sturm
// counts over shared-memory-staged representation rows.
//
// Same computation as the per-thread form described in k_bisect.cuh (PAPER.md
// Alg. 1 l.3 and l.16, L302-L304, L326-L328; Eq. (2.2); rtol =
// 1e-2 gaptol, L1294-L1295; binary_x phase L1064-L1111): a group of G lanes
// owns one eigenvalue index k and cuts its bracket [a, b] (count(a) < k <=
// count(b)) into G+1 parts per round.  What differs is only where the rows come
// from: every CTA holds items of ONE representation (host-built tasks), and all
// its threads evaluate their Sturm counts together, tile by tile, from rows
// staged through shared memory with cp.async (double-buffered).  A count is n
// rows for every item, so the threads of a CTA stay in step naturally; a thread
// whose item has converged idles through the remaining rounds of its CTA.  The
// rows come from smem at broadcast (every lane reads the same row), so the
// dependent recurrence is never exposed to L2 latency.
// The path of every index depends only on (representation, k, bracket, G): the
// CTA composition changes when a thread idles, never what it computes.
#pragma once
#include "k_bisect.cuh"

namespace mr3 {

constexpr int BS_TPB = 128;  // threads per CTA (maximum; launches pick 32..128)
constexpr int BS_TR = 256;   // rows per staged tile
constexpr int BS_TILE = BS_TR * 4;  // doubles per tile buffer (rows of up to 32 B)
constexpr int NEWTON_MAXPASS_DEFAULT = 8;  // Newton x-phase passes before the tail launch

__device__ __forceinline__ void bs_cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void bs_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void bs_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// rows [t0, t0 + BS_TR) of M_x ({d, lld} binary64, 16 B per row)
__device__ __forceinline__ void stage_x_tile(double *buf, const double *repx, int64_t n, int64_t t0) {
    const int rows = (int)min((int64_t)BS_TR, n - t0);
    for (int c = threadIdx.x; c < rows; c += blockDim.x) bs_cp_async16(buf + 2 * c, repx + 2 * (t0 + c));
    bs_commit();
}
// {d, lld} of rows [t0, t0 + BS_TR) of M_y (first 2 R of each 4-R row)
template <class R>
__device__ __forceinline__ void stage_y_tile(double *buf, const double *rep, int64_t n, int64_t t0) {
    constexpr int W = Prec<R>::words;
    const int rows = (int)min((int64_t)BS_TR, n - t0);
    for (int c = threadIdx.x; c < rows * W; c += blockDim.x) {
        const int r = c / W, off = (c % W) * 2;
        bs_cp_async16(buf + r * 2 * W + off, rep + (t0 + r) * 4 * W + off);
    }
    bs_commit();
}

// body(buf, t0, rows) over all tiles; collective (every thread of the CTA calls it)
template <class Stage, class Body>
__device__ __forceinline__ void tile_pass(double *smem, int64_t n, Stage stage, Body body) {
    const int ntile = (int)((n + BS_TR - 1) / BS_TR);
    stage(smem, (int64_t)0);
    for (int i = 0; i < ntile; i++) {
        if (i + 1 < ntile) {
            stage(smem + ((i + 1) & 1) * BS_TILE, (int64_t)(i + 1) * BS_TR);
            bs_wait<1>();
        } else {
            bs_wait<0>();
        }
        __syncthreads();
        const int64_t t0 = (int64_t)i * BS_TR;
        body(smem + (i & 1) * BS_TILE, t0, (int)min((int64_t)BS_TR, n - t0));
        __syncthreads();
    }
}

template <class R>
__device__ __forceinline__ Row2<R> yrow(const double *buf, int j);
template <>
__device__ __forceinline__ Row2<dd> yrow<dd>(const double *buf, int j) {
    const double2 *p = reinterpret_cast<const double2 *>(buf + 4 * j);
    const double2 u = p[0], v = p[1];
    Row2<dd> r;
    r.d = mkdd(u.x, u.y);
    r.lld = mkdd(v.x, v.y);
    return r;
}
template <>
__device__ __forceinline__ Row2<double> yrow<double>(const double *buf, int j) {
    const double2 u = *reinterpret_cast<const double2 *>(buf + 2 * j);
    Row2<double> r;
    r.d = u.x;
    r.lld = u.y;
    return r;
}

// ---------------------------------------------------------------------------
// CTA-collective Sturm counts (every thread calls; `need` selects who counts).
// binary_x: projective dstqds of negcount_x (kernels.cuh), rescaled every XB rows.
// binary_y: projective dstqds in R (below); the guarded ratio form of kernels.cuh
// only as the overflow fallback.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int count_x_cta(double *smem, const NodeInfo &nd, bool need, double x,
                                           double pivmin) {
    const int64_t n = nd.n;
    double p = -x, q = 1.0;
    unsigned c = 0;
    tile_pass(
        smem, n, [&](double *buf, int64_t t0) { stage_x_tile(buf, nd.repx, n, t0); },
        [&](const double *buf, int64_t t0, int rows) {
            if (!need) return;
            const double2 *t = reinterpret_cast<const double2 *>(buf);
            const bool last = t0 + rows == n;
            const int full = last ? rows - 1 : rows;
            int j = 0;
#pragma unroll 1
            for (; j + XB <= full; j += XB) {
                const double p0 = p, q0 = q;
                const unsigned c0 = c;
#pragma unroll
                for (int u = 0; u < XB; u++) xrow(t[j + u], x, p, q, c);
                const unsigned ep = (unsigned)__double2hiint(p) & 0x7ff00000u;
                const unsigned eq = (unsigned)__double2hiint(q) & 0x7ff00000u;
                const unsigned em = ep > eq ? ep : eq;
                if (em == 0x7ff00000u) {  // overflow: redo the block in the guarded ratio form
                    double s = p0 / q0;
                    if (!(fabs(s) <= 1e300)) s = copysign(1e300, s);
                    int cc = 0;
                    for (int u = 0; u < XB; u++) nc_row_guarded(t[j + u].x, t[j + u].y, x, pivmin, s, cc);
                    c = c0 + (unsigned)cc;
                    p = s;
                    q = 1.0;
                } else {
                    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                    p = mul_rn(p, sc);
                    q = mul_rn(q, sc);
                }
            }
#pragma unroll 1
            for (; j < full; j++) xrow(t[j], x, p, q, c);
            if (last) {
                const double D = fma_rn(t[rows - 1].x, q, p);
                c += (unsigned)(__double2hiint(D) ^ __double2hiint(q)) >> 31;
            } else {
                const unsigned ep = (unsigned)__double2hiint(p) & 0x7ff00000u;
                const unsigned eq = (unsigned)__double2hiint(q) & 0x7ff00000u;
                const unsigned em = ep > eq ? ep : eq;
                if (em != 0x7ff00000u) {
                    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                    p = mul_rn(p, sc);
                    q = mul_rn(q, sc);
                }
            }
        });
    return (int)c;
}

// binary_y Sturm count in the projective (division-free) form of negcount_x,
// carried out in R (pair arithmetic for fp64 I/O): with s_j = p_j / q_j,
//   D_j = d_j q_j + p_j,  q_{j+1} = D_j,  p_{j+1} = lld_j p_j - x D_j,
//   d+_j < 0  <=>  sign(D_j) != sign(q_j).
// Each step is a relative perturbation of O(eps_y) of d_j, lld_j, x and the
// state, like the dstqds it rewrites (no division, so no pivot guard is needed:
// D_j = 0 gives q_{j+1} = 0, i.e. s_{j+1} = inf, which the next row absorbs);
// per row two pair FMAs and one pair product, a dependent chain of two FMAs.
// (p, q) is rescaled by an exact power of two every XB rows; an overflow (only
// possible for |lld| > 1e38) redoes the block in the guarded ratio form.
// One binary_x pass giving the Sturm count at x and the Newton ratio f/f' of
// f(x) = det(M_x - x I) = D_{n-1} (x the projective scale factors): the x-derivative
// of the projective recurrence is carried along,
//   D'_j = d_j q'_j + p'_j,  q'_{j+1} = D'_j,  p'_{j+1} = lld_j p'_j - D_j - x D'_j,
// (p'_0 = -1, q'_0 = 0), rescaled with (p, q) by the same power of two (the ratio is
// scale-free).  Six FP64 instructions per row; the derivative chain runs beside the
// value chain.
// mode 0: count at x with f'/f and f''/f (three chains: the state and its first and second
// x-derivatives); mode 1: counts at x and at x2 (the second chain runs the count at x2,
// the third idles) -- the same per-row cost, chosen per thread
__device__ __forceinline__ void count_xn_cta(double *smem, const NodeInfo &nd, bool need, double x,
                                             double pivmin, int &cnt, double &ratio, double &f2,
                                             int mode = 0, double x2 = 0.0, int *cnt2 = nullptr) {
    const int64_t n = nd.n;
    // (p, q) and their first and second x-derivatives: f = det(M_x - x I) (scaled) is the
    // last D, f' and f'' the last D' and D''
    const double sB = mode ? 0.0 : 1.0, xB = mode ? x2 : x;
    double p = -x, q = 1.0, pd = mode ? -x2 : -1.0, qd = mode ? 1.0 : 0.0, pdd = 0.0, qdd = 0.0;
    unsigned c = 0, cB = 0;
    bool bad = false;
    tile_pass(
        smem, n, [&](double *buf, int64_t t0) { stage_x_tile(buf, nd.repx, n, t0); },
        [&](const double *buf, int64_t t0, int rows) {
            if (!need) return;
            const double2 *t = reinterpret_cast<const double2 *>(buf);
            const bool last = t0 + rows == n;
            const int full = last ? rows - 1 : rows;
            auto row = [&](const double2 r) {
                const double D = fma_rn(r.x, q, p);
                const double Dd = fma_rn(r.x, qd, pd);
                const double Ddd = fma_rn(r.x, qdd, pdd);
                c += (unsigned)(__double2hiint(D) ^ __double2hiint(q)) >> 31;
                cB += (unsigned)(__double2hiint(Dd) ^ __double2hiint(qd)) >> 31;
                const double pn = fma_rn(-x, D, mul_rn(r.y, p));
                pdd = fma_rn(-x, Ddd, fma_rn(r.y, pdd, (-2.0 * sB) * Dd));  // (mode 1: stays 0)
                pd = fma_rn(-xB, Dd, fma_rn(r.y, pd, -sB * D));
                p = pn;
                q = D;
                qd = Dd;
                qdd = Ddd;
            };
            int j = 0;
#pragma unroll 1
            for (; j < full; j += XB) {
                const int je = min(j + XB, full);
                if (je - j == XB) {
#pragma unroll
                    for (int u = 0; u < XB; u++) row(t[j + u]);
                } else {
                    for (int u = j; u < je; u++) row(t[u]);
                }
                // one power of two for all four (the largest exponent -> 2^0)
                unsigned em = (unsigned)__double2hiint(p) & 0x7ff00000u;
                em = max(em, (unsigned)__double2hiint(q) & 0x7ff00000u);
                em = max(em, (unsigned)__double2hiint(pd) & 0x7ff00000u);
                em = max(em, (unsigned)__double2hiint(qd) & 0x7ff00000u);
                em = max(em, (unsigned)__double2hiint(pdd) & 0x7ff00000u);
                em = max(em, (unsigned)__double2hiint(qdd) & 0x7ff00000u);
                if (em == 0x7ff00000u) {
                    bad = true;  // overflow: count and ratio unreliable -> caller bisects
                    p = -x;
                    q = 1.0;
                    pd = mode ? -x2 : -1.0;
                    qd = mode ? 1.0 : 0.0;
                    pdd = 0.0;
                    qdd = 0.0;
                } else {
                    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                    p *= sc;
                    q *= sc;
                    pd *= sc;
                    qd *= sc;
                    pdd *= sc;
                    qdd *= sc;
                }
            }
            if (last) {
                const double D = fma_rn(t[rows - 1].x, q, p);
                const double Dd = fma_rn(t[rows - 1].x, qd, pd);
                const double Ddd = fma_rn(t[rows - 1].x, qdd, pdd);
                c += (unsigned)(__double2hiint(D) ^ __double2hiint(q)) >> 31;
                cB += (unsigned)(__double2hiint(Dd) ^ __double2hiint(qd)) >> 31;
                ratio = D / Dd;
                f2 = Ddd / D;
            }
        });
    cnt = (int)c;
    if (cnt2) *cnt2 = (int)cB;
    if (__syncthreads_or(bad)) {  // rare: recount the affected threads (collective calls)
        const int c2 = count_x_cta(smem, nd, need && bad, x, pivmin);
        const int c3 = count_x_cta(smem, nd, need && bad && mode == 1, x2, pivmin);
        if (bad) {
            ratio = NAN;
            f2 = NAN;
            cnt = c2;
            if (cnt2) *cnt2 = c3;
        }
    }
}

// Sturm-count bisection accelerated by Newton steps on f(x) = det(M_x - x I) (G = 1):
// every pass returns count(x) (the bracket invariant count(a) < k <= count(b) is kept
// exactly as in bisection) and f/f'; the next point is the Newton iterate when it lies
// inside the bracket and the bracket has been shrinking, else the midpoint.  Once the
// Newton step is below tol/4 the next point is placed tol/4 beyond the estimate on the
// other side, so one more pass closes the bracket to width <= tol/2.  Convergence is
// quadratic near a simple eigenvalue; a bracket holding several eigenvalues is reduced
// by the counts (any Newton iterate outside the bracket falls back to bisection).
__device__ __forceinline__ void newton_cta(double *smem, const NodeInfo &nd, double &a, double &b,
                                           bool active, int k, double rtol, double absfloor,
                                           double tolmul, double pivmin,
                                           unsigned long long &rows, int64_t n, int &passes,
                                           int maxpass, bool &converged, double &est_last,
                                           double &step_last) {
    bool mdone = !active;
    passes = 0;
    converged = false;
    est_last = NAN;        // Newton estimate x - f/f' of the last pass (the RQI start, R10)
    step_last = INFINITY;  // |f/f'| of that pass
    double xn = NAN;
    double r1 = INFINITY, r2 = INFINITY;  // |Newton step| of the last two Newton passes
    int nnewton = 0;
    bool close = false;  // next pass: counts at xn -+ tol/4 (closes the bracket around xn)
#pragma unroll 1
    for (int round = 0; round < 4000; round++) {
        double x = a, x2 = a;
        bool need = false;
        double tol = 0.0;
        bool took_newton = false;
        int mode = 0;
        if (!mdone) {
            const double w = b - a;
            tol = tolmul * fmax(2.0 * rtol * fmax(fabs(a), fabs(b)), absfloor);
            if (w <= tol) {
                mdone = true;
                converged = true;
            } else if (passes >= maxpass) {
                mdone = true;  // left to the many-lane multisection (tail launch)
            } else if (close && !isnan(xn)) {
                mode = 1;
                x = xn - 0.25 * tol;
                x2 = xn + 0.25 * tol;
                need = (a < x && x < b) || (a < x2 && x2 < b);
                if (!need) mdone = true;
            } else {
                // Newton while its steps contract (|step| at least halves every round)
                // and stay inside the bracket; bisection otherwise
                const bool contracting = nnewton < 2 || r1 <= 0.5 * r2;
                took_newton = !isnan(xn) && xn > a && xn < b && contracting && nnewton < 12;
                x = took_newton ? xn : 0.5 * (a + b);
                need = a < x && x < b;
                if (!need) mdone = true;  // no representable progress
            }
        }
        if (!__syncthreads_or(!mdone)) break;
        int c = 0, c2 = 0;
        double ratio = NAN, f2 = NAN;
        count_xn_cta(smem, nd, need, x, pivmin, c, ratio, f2, mode, x2, &c2);
        if (need && mode == 1) {  // closing pass: two counts
            rows += n;
            passes++;
            if (c >= k)
                b = fmin(b, x);
            else
                a = fmax(a, x);
            if (c2 >= k)
                b = fmin(b, x2);
            else
                a = fmax(a, x2);
            close = false;
            xn = NAN;
        } else if (need) {
            rows += n;
            passes++;
            if (c >= k)
                b = x;
            else
                a = x;
            xn = NAN;
            close = false;
            est_last = NAN;
            step_last = INFINITY;
            if (fabs(ratio) < INFINITY) {
                // Laguerre's step when the nearest eigenvalue on the side the count points
                // to is lambda_k itself (count(x) = k: the largest root <= x; count(x) =
                // k - 1: the smallest root > x): for a polynomial with real roots it then
                // converges monotonically (cubically) to that root; Newton's otherwise
                double step = ratio;
                if ((c == k || c == k - 1) && fabs(f2) < INFINITY) {
                    const double G = 1.0 / ratio, N = (double)n;
                    const double H = G * G - f2;  // sum 1 / (x - lambda_j)^2
                    const double sq = sqrt(fmax((N - 1.0) * (N * H - G * G), 0.0));
                    const double den = c == k ? G + sq : G - sq;  // left: > 0, right: < 0
                    if (den != 0.0 && (c == k ? den > 0.0 : den < 0.0)) step = N / den;
                }
                const double est = x - step;
                est_last = est;
                step_last = fabs(step);
                if (took_newton || nnewton == 0) {
                    nnewton++;
                    r2 = r1;
                    r1 = fabs(step);
                }
                // close the bracket around the estimate in one two-count pass once the step
                // is below tol/4, or once the error after it -- cubic convergence, with the
                // constant from the last two steps: r1^4 / r2^3 -- is predicted below tol/8
                xn = est;
                const bool cubic = nnewton >= 2 && r2 < INFINITY && r1 < 0.5 * r2;
                const double perr = cubic ? r1 * (r1 / r2) * (r1 / r2) * (r1 / r2) : INFINITY;
                close = fabs(step) <= 0.25 * tol || perr <= 0.125 * tol;
                // error estimate of est for the RQI start (k_refine_flags): a direct bound
                // (negative) from the observed cubic contraction, with a factor 4 and an
                // ulp floor; else the step (the quadratic model there)
                if (cubic) step_last = -fmax(4.0 * perr, 2.0 * 1.1102230246251565e-16 * fabs(est));
            }
        }
    }
}

// two shifts per thread through the same rows (two independent FMA chains: the
// binary_x row chain is two dependent DFMAs, so one chain per thread leaves the
// FP64 pipe waiting on latency at the 2-3 warps per scheduler a 50000-item
// launch provides)
__device__ __forceinline__ bool xrescale(double &p, double &q) {
    const unsigned ep = (unsigned)__double2hiint(p) & 0x7ff00000u;
    const unsigned eq = (unsigned)__double2hiint(q) & 0x7ff00000u;
    const unsigned em = ep > eq ? ep : eq;
    if (em == 0x7ff00000u) return false;
    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
    p = mul_rn(p, sc);
    q = mul_rn(q, sc);
    return true;
}
// (overflow path, inlined: a non-inline callee taking references would force the
// hot recurrence state into local memory)
__device__ __forceinline__ void xblock_ratio(const double2 *t, int j0, int j1, double x,
                                             double pivmin, double &p, double &q, unsigned &c) {
    double s = p / q;
    if (!(fabs(s) <= 1e300)) s = copysign(1e300, s);
    int cc = 0;
    for (int u = j0; u < j1; u++) nc_row_guarded(t[u].x, t[u].y, x, pivmin, s, cc);
    c += (unsigned)cc;
    p = s;
    q = 1.0;
}
__device__ __forceinline__ void count_x2_cta(double *smem, const NodeInfo &nd, bool need, double xa,
                                             double xb, double pivmin, int &ca, int &cb) {
    const int64_t n = nd.n;
    double pa = -xa, qa = 1.0, pb = -xb, qb = 1.0;
    unsigned c0 = 0, c1 = 0;
    tile_pass(
        smem, n, [&](double *buf, int64_t t0) { stage_x_tile(buf, nd.repx, n, t0); },
        [&](const double *buf, int64_t t0, int rows) {
            if (!need) return;
            const double2 *t = reinterpret_cast<const double2 *>(buf);
            const bool last = t0 + rows == n;
            const int full = last ? rows - 1 : rows;
            int j = 0;
#pragma unroll 1
            for (; j < full; j += XB) {
                const int je = min(j + XB, full);
                const double pa0 = pa, qa0 = qa, pb0 = pb, qb0 = qb;
                const unsigned ca0 = c0, cb0 = c1;
                if (je - j == XB) {
#pragma unroll
                    for (int u = 0; u < XB; u++) {
                        const double2 r = t[j + u];
                        xrow(r, xa, pa, qa, c0);
                        xrow(r, xb, pb, qb, c1);
                    }
                } else {
                    for (int u = j; u < je; u++) {
                        xrow(t[u], xa, pa, qa, c0);
                        xrow(t[u], xb, pb, qb, c1);
                    }
                }
                if (!xrescale(pa, qa)) {
                    pa = pa0;
                    qa = qa0;
                    c0 = ca0;
                    xblock_ratio(t, j, je, xa, pivmin, pa, qa, c0);
                }
                if (!xrescale(pb, qb)) {
                    pb = pb0;
                    qb = qb0;
                    c1 = cb0;
                    xblock_ratio(t, j, je, xb, pivmin, pb, qb, c1);
                }
            }
            if (last) {
                const double Da = fma_rn(t[rows - 1].x, qa, pa);
                c0 += (unsigned)(__double2hiint(Da) ^ __double2hiint(qa)) >> 31;
                const double Db = fma_rn(t[rows - 1].x, qb, pb);
                c1 += (unsigned)(__double2hiint(Db) ^ __double2hiint(qb)) >> 31;
            }
        });
    ca = (int)c0;
    cb = (int)c1;
}

template <class R>
struct YState {
    R p, q;
    int c;
};
template <class R>
__device__ __forceinline__ void yrow_proj(const Row2<R> &rw, R mx, YState<R> &st) {
    const R D = fma_dd(rw.d, st.q, st.p);
    st.c += (int)((unsigned)(__double2hiint(hi(D)) ^ __double2hiint(hi(st.q))) >> 31);
    st.p = fma_dd(mx, D, mul(rw.lld, st.p));
    st.q = D;
}
template <class R>
__device__ __forceinline__ bool yrescale(YState<R> &st) {
    const unsigned ep = (unsigned)__double2hiint(hi(st.p)) & 0x7ff00000u;
    const unsigned eq = (unsigned)__double2hiint(hi(st.q)) & 0x7ff00000u;
    const unsigned em = ep > eq ? ep : eq;
    if (em == 0x7ff00000u || !(fabs(lo_part(st.p)) < INFINITY) || !(fabs(lo_part(st.q)) < INFINITY))
        return false;
    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
    st.p = scale_pow2(st.p, sc);
    st.q = scale_pow2(st.q, sc);
    return true;
}
// rows [j0, j1) of a tile in the guarded ratio form from a saved state (overflow path)
template <class R>
__device__ __forceinline__ void yblock_ratio(const double *buf, int j0, int j1, R x, double pivmin,
                                          YState<R> &st) {
    R s = div(st.p, st.q);
    if (!(fabs(hi(s)) <= 1e300)) s = mk<R>(copysign(1e300, hi(s)));
    for (int j = j0; j < j1; j++) {
        const Row2<R> rw = yrow<R>(buf, j);
        R dp = guard(add(rw.d, s), pivmin);
        st.c += is_neg(dp) ? 1 : 0;
        s = sub(mul(rw.lld, div(s, dp)), x);
    }
    st.p = s;
    st.q = mk<R>(1.0);
}

// one or two shifts per thread (two: xa and xb through the same rows, ILP 2)
template <class R, bool TWO>
__device__ __forceinline__ void count_y_cta(double *smem, const NodeInfo &nd, bool need, R xa,
                                            R xb, double pivmin, int &ca, int &cb) {
    const int64_t n = nd.n;
    const R ma = neg(xa), mb = neg(xb);
    YState<R> A{ma, mk<R>(1.0), 0}, B{mb, mk<R>(1.0), 0};
    tile_pass(
        smem, n, [&](double *buf, int64_t t0) { stage_y_tile<R>(buf, nd.rep, n, t0); },
        [&](const double *buf, int64_t t0, int rows) {
            if (!need) return;
            const bool last = t0 + rows == n;
            const int full = last ? rows - 1 : rows;
            int j = 0;
#pragma unroll 1
            for (; j < full; j += XB) {
                const int je = min(j + XB, full);
                const YState<R> A0 = A, B0 = B;
                if (je - j == XB) {
#pragma unroll
                    for (int u = 0; u < XB; u++) {
                        const Row2<R> rw = yrow<R>(buf, j + u);
                        yrow_proj<R>(rw, ma, A);
                        if (TWO) yrow_proj<R>(rw, mb, B);
                    }
                } else {
                    for (int u = j; u < je; u++) {
                        const Row2<R> rw = yrow<R>(buf, u);
                        yrow_proj<R>(rw, ma, A);
                        if (TWO) yrow_proj<R>(rw, mb, B);
                    }
                }
                if (!yrescale(A)) {
                    A = A0;
                    yblock_ratio<R>(buf, j, je, xa, pivmin, A);
                }
                if (TWO && !yrescale(B)) {
                    B = B0;
                    yblock_ratio<R>(buf, j, je, xb, pivmin, B);
                }
            }
            if (last) {
                const Row2<R> rw = yrow<R>(buf, rows - 1);
                const R D = fma_dd(rw.d, A.q, A.p);
                A.c += (int)((unsigned)(__double2hiint(hi(D)) ^ __double2hiint(hi(A.q))) >> 31);
                if (TWO) {
                    const R E = fma_dd(rw.d, B.q, B.p);
                    B.c += (int)((unsigned)(__double2hiint(hi(E)) ^ __double2hiint(hi(B.q))) >> 31);
                }
            }
        });
    ca = A.c;
    cb = B.c;
}

// NEXT-1b ("the above criterion can be relaxed for eigenvalues with a
// large gap to the rest of the spectrum"): isolation of lambda_k read off the item's OWN
// Sturm counts, so it depends on nothing but the item's path (world- and CTA-independent).
// A point x with count(x) = k - 1 lies in (lambda_{k-1}, lambda_k], one with count(x) = k in
// (lambda_k, lambda_{k+1}]; with alo the smallest point seen of the first kind and bhi the
// largest of the second, the gaps of lambda_k are at least a - alo and bhi - b.  Once they are
// both >= sep * max(|a|, |b|) (so the item will classify as a singleton with room to spare)
// and the bracket is narrower than relax * gap, the bracket stops: its midpoint is a start
// from which the RQI needs the same two passes (R20), whatever rtol asks for.
struct Iso {
    double alo = INFINITY, bhi = -INFINITY;  // isolation points seen so far
    double relax = 0.0;                      // 0: off (rtol alone decides)
    double sep = 0.0;                        // required gap / magnitude (4 gaptol)
    double slack = 0.0;                      // width allowed on top (the x -> y widening)
    int kmax = 0;                            // eigenvalues of the node (k = kmax: no right one)
};
__device__ __forceinline__ bool iso_stop(const Iso &I, int k, double a, double b) {
    if (!(I.relax > 0.0)) return false;
    const double gl = k <= 1 ? INFINITY : a - I.alo;
    const double gr = k >= I.kmax ? INFINITY : I.bhi - b;
    const double g = fmin(gl, gr);
    return g >= I.sep * fmax(fabs(a), fabs(b)) && b - a <= I.relax * g + I.slack;
}

// CTA-synchronous multisection rounds of the groups (see multisect in k_bisect.cuh)
template <class T, int G, class Count>
__device__ __forceinline__ void msect_cta(T &a, T &b, bool active, int k, int lig, int lane,
                                          unsigned gmask, double rtol, double absfloor,
                                          double tolmul, unsigned long long &rows, int64_t n,
                                          Count count, Iso *iso = nullptr) {
    bool mdone = !active;
#pragma unroll 1
    for (int round = 0; round < 4000; round++) {
        T x = a;
        bool need = false, above = false;
        if (!mdone) {
            T w = sub(b, a);
            double tol = tolmul * fmax(2.0 * rtol * fmax(fabs(hi(a)), fabs(hi(b))), absfloor);
            if (hi(w) <= tol || (iso != nullptr && iso_stop(*iso, k, hi(a), hi(b)))) {
                mdone = true;
            } else {
                x = add(a, mul(w, (double)(lig + 1) / (double)(G + 1)));
                above = lt(a, x);
                need = above && lt(x, b);
            }
        }
        if (!__syncthreads_or(!mdone)) break;
        int c = count(need, x);
        if (!mdone) {
            if (need)
                rows += n;
            else
                c = above ? k : k - 1;  // x == b counts as right of lambda_k, x == a as left
            bool P = c >= k;
            const unsigned sh = lane & ~(G - 1) & 31;
            const unsigned gm = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
            unsigned bal = __ballot_sync(gmask, P);
            bal = (bal >> sh) & gm;
            int first = bal ? __ffs(bal) : G + 1;
            if (iso != nullptr) {  // isolation points among the evaluated ones (group-uniform)
                const unsigned e1 = (__ballot_sync(gmask, need && c == k - 1) >> sh) & gm;
                const unsigned e2 = (__ballot_sync(gmask, need && c == k) >> sh) & gm;
                const double x1 = __shfl_sync(gmask, hi(x), e1 ? __ffs(e1) - 1 : 0, G);
                const double x2 = __shfl_sync(gmask, hi(x), e2 ? 31 - __clz(e2) : 0, G);
                if (e1) iso->alo = fmin(iso->alo, x1);
                if (e2) iso->bhi = fmax(iso->bhi, x2);
            }
            T xb = shfl_R<T>(gmask, x, first <= G ? first - 1 : 0, G);
            T xa = shfl_R<T>(gmask, x, first >= 2 ? first - 2 : 0, G);
            T nb = first <= G ? xb : b;
            T na = first >= 2 ? xa : a;
            if (same(na, a) && same(nb, b)) {
                mdone = true;  // no representable progress
            } else {
                a = na;
                b = nb;
            }
        }
    }
}

// Same, with two points per lane: a group of G lanes cuts [a, b] into 2G + 1
// parts per round (lane l evaluates points 2l+1 and 2l+2).  The new bracket is
// [x_{f-1}, x_f] for the first point f whose count is >= k, so count(x_{f-1}) < k
// <= count(x_f) holds whatever the monotonicity of the rounded counts.
template <int G, class Count2>
__device__ __forceinline__ void msect2_cta(double &a, double &b, bool active, int k, int lig,
                                           int lane, unsigned gmask, double rtol, double absfloor,
                                           double tolmul, unsigned long long &rows, int64_t n,
                                           Count2 count2) {
    bool mdone = !active;
    constexpr int NPT = 2 * G;
#pragma unroll 1
    for (int round = 0; round < 4000; round++) {
        double x0 = a, x1 = a;
        bool n0 = false, n1 = false, ab0 = false, ab1 = false;
        if (!mdone) {
            const double w = b - a;
            const double tol = tolmul * fmax(2.0 * rtol * fmax(fabs(a), fabs(b)), absfloor);
            if (w <= tol) {
                mdone = true;
            } else {
                x0 = a + w * ((double)(2 * lig + 1) / (double)(NPT + 1));
                x1 = a + w * ((double)(2 * lig + 2) / (double)(NPT + 1));
                ab0 = a < x0;
                n0 = ab0 && x0 < b;
                ab1 = a < x1;
                n1 = ab1 && x1 < b;
            }
        }
        if (!__syncthreads_or(!mdone)) break;
        int c0 = 0, c1 = 0;
        count2(n0 || n1, x0, x1, c0, c1);
        if (!mdone) {
            rows += (unsigned long long)((n0 ? 1 : 0) + (n1 ? 1 : 0)) * n;
            if (!n0) c0 = ab0 ? k : k - 1;
            if (!n1) c1 = ab1 ? k : k - 1;
            const unsigned sh = lane & ~(G - 1) & 31;
            const unsigned msk = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
            const unsigned b0 = (__ballot_sync(gmask, c0 >= k) >> sh) & msk;
            const unsigned b1 = (__ballot_sync(gmask, c1 >= k) >> sh) & msk;
            const unsigned any = b0 | b1;
            int first = NPT + 1;  // 1-based index of the first point with count >= k
            if (any) {
                const int l = __ffs(any) - 1;
                first = 2 * l + (((b0 >> l) & 1u) ? 0 : 1) + 1;
            }
            const int fb = first <= NPT ? first - 1 : 0;  // 0-based point index of x_f
            const int fa = first >= 2 ? first - 2 : 0;    // of x_{f-1}
            const double vb0 = __shfl_sync(gmask, x0, fb >> 1, G);
            const double vb1 = __shfl_sync(gmask, x1, fb >> 1, G);
            const double va0 = __shfl_sync(gmask, x0, fa >> 1, G);
            const double va1 = __shfl_sync(gmask, x1, fa >> 1, G);
            const double nb = first <= NPT ? ((fb & 1) ? vb1 : vb0) : b;
            const double na = first >= 2 ? ((fa & 1) ? va1 : va0) : a;
            if (na == a && nb == b) {
                mdone = true;  // no representable progress
            } else {
                a = na;
                b = nb;
            }
        }
    }
}

template <class R, int G, bool XPHASE>
__global__ void __launch_bounds__(BS_TPB) k_bisect_s(const NodeInfo *__restrict__ nodes, Items it,
                                                  const int32_t *__restrict__ list,
                                                  const RqiTask *__restrict__ tasks,
                                                  const int *__restrict__ ntasks, double rtol,
                                                  double absfloor, double pivmin, double pivmin_x,
                                                  double eps_x, int certify, int xpts,
                                                  int ycert, char *tailflag, int xpts_maxpass,
                                                  double widen, double relax_f, double sep,
                                                  int iso_init, DevStats *st) {
    __shared__ __align__(16) double sbuf[2 * BS_TILE];
    if ((int)blockIdx.x >= *ntasks) return;  // grid is an upper bound (whole CTA leaves)
    const RqiTask task = tasks[blockIdx.x];
    const NodeInfo nd = nodes[task.node];
    const int64_t n = nd.n;
    const int local = threadIdx.x / G, lig = threadIdx.x % G;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const bool active = local < task.cnt;
    int id = -1, k = 0;
    R a = mk<R>(0.0), b = a;
    if (active) {
        id = list[task.first + local];
        k = it.k[id];
        a = reinterpret_cast<R *>(it.lo)[id];
        b = reinterpret_cast<R *>(it.hi)[id];
    }
    unsigned long long rows = 0, rows_x = 0;
    // NEXT-1b: relaxed stop for isolated eigenvalues (relax_f = 0: off); relax = relax_f n^(1/4)
    // makes the stop width relax * gap = c gap sqrt(eps_x sqrt(n) / C) (host: mr3.cu)
    Iso iso;
    iso.relax = relax_f > 0.0 ? relax_f * sqrt(sqrt((double)n)) : 0.0;
    iso.sep = sep;
    iso.kmax = (int)n;
    if (iso_init && active) {  // isolation points from the grid cells (k_cell_final)
        const double l0 = it.lgap[id], r0 = it.rgap[id];
        if (!isnan(l0)) iso.alo = l0;
        if (!isnan(r0)) iso.bhi = r0;
        __syncwarp(gmask);
        if (lig == 0) {  // (restored: the gaps are classification's from here on)
            it.lgap[id] = 1e300;
            it.rgap[id] = 1e300;
        }
    }

    // binary_y certification: count_y(a) < k <= count_y(b); failing ends are widened
    // (by delta, then 8x per try) until certified (k_bisect.cuh certify_bracket)
    auto certify_y = [&](double delta) {
        bool cdone = !active;
#pragma unroll 1
        for (int tries = 0; tries < 200; tries++) {
            if (!__syncthreads_or(!cdone)) break;
            int ca = 0, cb = 0;
            count_y_cta<R, true>(sbuf, nd, !cdone && lig == 0, a, b, pivmin, ca, cb);
            if (!cdone) {
                ca = __shfl_sync(gmask, ca, 0, G);
                cb = __shfl_sync(gmask, cb, 0, G);
                if (lig == 0) rows += 2 * n;
                if (ca < k && cb >= k) {
                    cdone = true;
                } else {
                    double w = fmax(delta, fmax(absfloor, 1e-3 * fabs(hi(b)) * (tries > 2 ? 1.0 : 0.0)));
                    w = w * (double)(1ULL << (3 * (tries < 20 ? tries : 20)));
                    if (ca >= k) a = sub(a, mk<R>(w));
                    if (cb < k) b = add(b, mk<R>(w));
                }
            }
        }
    };

    if (XPHASE && certify == 2) {
        // K2' (RQI starting points): binary_x multisection on M_x to relative rtol
        // (a few ulps) from the certified bracket; x0 = midpoint if strictly inside it.
        // Root brackets of the uncertified binary_x phase (R8d) are first widened as k_rqi
        // widens its guard (widen = root_widen): the binary_x eigenvalue seen by count_x may
        // lie just outside a bracket that count_xn (Newton) produced
        if (widen > 0.0 && nd.depth == 0 && active) {
            const double wd = widen * (double)n * fmax(fabs(hi(a)), fabs(hi(b)));
            a = sub(a, mk<R>(wd));
            b = add(b, mk<R>(wd));
        }
        double ax = hi(a), bx = hi(b);
        msect_cta<double, G>(ax, bx, active, k, lig, lane, gmask, rtol, absfloor, 1.0, rows_x, n,
                             [&](bool need, double x) {
                                 return count_x_cta(sbuf, nd, need, x, pivmin_x);
                             });
        if (active && lig == 0) {
            const double x = 0.5 * (ax + bx);
            it.x0[id] = (x > hi(a) && x < hi(b)) ? x : NAN;
        }
        if (rows_x) atomicAdd(&st->refine_rows_x, rows_x);
        return;
    }
    if (certify) certify_y(absfloor);
    if (XPHASE) {
        double ax = hi(a), bx = hi(b);
        if (G == 1 && xpts == 3) {
            int passes = 0;
            bool conv = true;
            double est = NAN, step = INFINITY;
            newton_cta(sbuf, nd, ax, bx, active, k, rtol, absfloor, 0.5, pivmin_x, rows_x, n, passes,
                       tailflag ? xpts_maxpass : 4000, conv, est, step);
            if (passes) atomicAdd(&st->newton_rows_x, (unsigned long long)passes * n);
            if (active) {  // the last Newton estimate: RQI start unless k_refine_flags rejects it
                it.x0[id] = conv ? est : NAN;
                it.dx[id] = conv ? step : INFINITY;
                it.twist[id] = passes;  // (diagnostics only: k_rqi_locate sets the twist)
            }
            if (tailflag && active) tailflag[local + task.first] = conv ? 0 : 1;
            if (tailflag && active && !conv) {
                // unfinished: hand the current (valid) bracket to the tail launch
                reinterpret_cast<R *>(it.lo)[id] = mk<R>(ax);
                reinterpret_cast<R *>(it.hi)[id] = mk<R>(bx);
                if (rows_x) atomicAdd(&st->bisect_rows_x, rows_x);
                return;  // tail mode is only used with ycert == 0, certify == 0: no barrier follows
            }
        }
        else if (xpts == 2)
            msect2_cta<G>(ax, bx, active, k, lig, lane, gmask, rtol, absfloor, 0.5, rows_x, n,
                          [&](bool need, double x0, double x1, int &c0, int &c1) {
                              count_x2_cta(sbuf, nd, need, x0, x1, pivmin_x, c0, c1);
                          });
        else
            msect_cta<double, G>(ax, bx, active, k, lig, lane, gmask, rtol, absfloor, 0.5, rows_x,
                                 n, [&](bool need, double x) {
                                     return count_x_cta(sbuf, nd, need, x, pivmin_x);
                                 }, &iso);
        if (!(G == 1 && xpts == 3) && !ycert && !certify && active && lig == 0) {
            // multisection result: its midpoint is the RQI start, |error| <= half-width
            // (dx < 0 marks a direct bound, dx >= 0 a Newton step; k_refine_flags)
            it.x0[id] = 0.5 * (ax + bx);
            it.dx[id] = -0.5 * (bx - ax);
        }
        double delta = absfloor;
        if (active) {
            double mag = fmax(fabs(ax), fabs(bx));
            delta = 8.0 * eps_x * sqrt((double)n) * mag + absfloor;
            R na = mk<R>(ax - delta), nb = mk<R>(bx + delta);
            if (lt(na, a)) na = a;  // never leave the certified incoming bracket
            if (lt(b, nb)) nb = b;
            a = na;
            b = nb;
        }
        if (!ycert && !certify) {
            // root level without binary_y certification (reading R8d): [a, b] is the
            // binary_x bracket widened by the typical M_x -> M_y shift; consumers that
            // need a rigorous enclosure widen it by the relative-robustness bound of the
            // definite root (k_rqi: root_widen)
            if (active && lig == 0) {
                reinterpret_cast<R *>(it.lo)[id] = a;
                reinterpret_cast<R *>(it.hi)[id] = b;
            }
            if (rows) atomicAdd(&st->bisect_rows, rows);
            if (rows_x) atomicAdd(&st->bisect_rows_x, rows_x);
            return;
        }
        certify_y(delta);
        // the binary_x isolation points, moved toward lambda_k by the M_x -> M_y shift; a
        // bracket the x phase stopped by isolation stays stopped after the widening by delta
        // (certify_y may widen further: then the y phase bisects back)
        iso.alo += delta;
        iso.bhi -= delta;
        iso.slack = 4.0 * delta;
    }
    msect_cta<R, G>(a, b, active, k, lig, lane, gmask, rtol, absfloor, 1.0, rows, n,
                    [&](bool need, R x) {
                        int c, dummy;
                        count_y_cta<R, false>(sbuf, nd, need, x, x, pivmin, c, dummy);
                        return c;
                    }, &iso);
    if (active && lig == 0) {
        reinterpret_cast<R *>(it.lo)[id] = a;
        reinterpret_cast<R *>(it.hi)[id] = b;
    }
    if (rows) atomicAdd(&st->bisect_rows, rows);
    if (rows_x) atomicAdd(&st->bisect_rows_x, rows_x);
}

// K2' selection: singletons whose certified bracket half-width exceeds
// gap sqrt(eps_x sqrt(n) / C) need a refined RQI start: each RQI step restarts inverse
// iteration from e_r, so its error contracts like e1 ~ C e0^2 / gap, and two iterations
// (one RQ correction + the converged solve) need e0 <= gap sqrt(eps_x sqrt(n) / C).  The
// selected items get x0 from a binary_x multisection on M_x (k_bisect_s, certify = 2); all
// others start at the bracket midpoint (x0 = NaN).  x0 needs no certification: the RQI
// keeps the certified binary_y bracket as its guard.
// A root item whose binary_x phase ended in a Newton step dx keeps that step's estimate
// as its start when the estimate's predicted error -- quadratic convergence, 4 dx^2 / gap
// (the Newton constant |f''/2f'| is about 1/gap), plus 2 ulps -- is below both the
// bracket half-width and the requirement above: those items need no refinement pass.
template <class R>
__global__ void k_refine_flags(const NodeInfo *__restrict__ nodes, Items it,
                               const int32_t *__restrict__ list, int cnt, double eps_x,
                               double cconv, char *flags) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const int id = list[t];
    const NodeInfo &nd = nodes[it.node[id]];
    const int64_t n = nd.n;
    const R a = reinterpret_cast<R *>(it.lo)[id];
    const R b = reinterpret_cast<R *>(it.hi)[id];
    const double gap = fmin(it.lgap[id], it.rgap[id]);
    const double need = gap * sqrt(eps_x * sqrt((double)n) / cconv);
    const double half_w = 0.5 * hi(sub(b, a));
    const double x0 = it.x0[id], dx = it.dx[id];
    double err = half_w;  // of the midpoint start
    if (nd.depth == 0 && x0 > hi(a) && x0 < hi(b) && dx < INFINITY && gap > 0.0) {
        const double pe = dx < 0.0 ? -dx : 4.0 * dx * dx / gap + eps_x * fabs(x0);
        if (pe < half_w) err = pe;
    }
    if (err == half_w) it.x0[id] = NAN;
    // the refinement ends at about 2 ulps: below 4 ulps it has nothing to add; and a start
    // up to 1024x worse than `need` costs one or two more RQI iterations, which run as split
    // passes (k_rqi, R9d) at a few percent of the refinement launch's latency (≈ 4 ms even
    // for a handful of items: its multisection rounds are serial n-row chains)
    const double floor_ = 4.0 * eps_x * fmax(fabs(hi(a)), fabs(hi(b)));
    flags[t] = (err > 1024.0 * fmax(need, floor_) && n >= 2) ? 1 : 0;
}

}  // namespace mr3
