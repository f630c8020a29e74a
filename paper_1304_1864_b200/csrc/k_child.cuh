// k_child.cuh -- K4: child representations for clusters (Alg. 1 l.15-17).
#pragma once
#include "k_bisect.cuh"

namespace mr3 {

// Rows of the parent staged through shared memory (all 32 lanes read the same row: broadcast),
// double-buffered with cp.async: tiles of CH_TR rows.
constexpr int CH_TR = 32;
template <class R>
__device__ __forceinline__ void child_stage(double *buf, const double *rep, int64_t n, int64_t t0) {
    constexpr int ROWD = 4 * Prec<R>::words;  // doubles per row
    constexpr int CHK = CH_TR * ROWD / 2;      // 16-byte chunks per tile
    for (int c = threadIdx.x; c < CHK; c += 32) {
        const int r = c / (ROWD / 2), off = (c % (ROWD / 2)) * 2;
        int64_t g = t0 + r;
        g = g < n ? g : n - 1;
        const unsigned sa = (unsigned)__cvta_generic_to_shared(buf + r * ROWD + off);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(rep + g * ROWD + off));
    }
    asm volatile("cp.async.commit_group;\n" ::);
}
template <class R>
__device__ __forceinline__ Row4<R> child_row(const double *buf, int j);
template <>
__device__ __forceinline__ Row4<dd> child_row<dd>(const double *buf, int j) {
    const double2 *p = reinterpret_cast<const double2 *>(buf + j * 8);
    const double2 a = p[0], b = p[1], c = p[2], d = p[3];
    Row4<dd> r;
    r.d = mkdd(a.x, a.y);
    r.lld = mkdd(b.x, b.y);
    r.l = mkdd(c.x, c.y);
    r.ld = mkdd(d.x, d.y);
    return r;
}
template <>
__device__ __forceinline__ Row4<double> child_row<double>(const double *buf, int j) {
    const double2 *p = reinterpret_cast<const double2 *>(buf + j * 4);
    const double2 a = p[0], b = p[1];
    Row4<double> r;
    r.d = a.x;
    r.lld = a.y;
    r.l = b.x;
    r.ld = b.y;
    return r;
}

// projective dstqds row (SURVEY.md App. A in the division-free form of reading R8b):
// with s = p / q, D = d q + p (= d+ q), p' = lld p - tau D, q' = D.  The pivot guard of
// reading R6 (|d+| < pivmin -> d+ = -pivmin) in scale-invariant form: |D| < pivmin |q|.
template <class R>
__device__ __forceinline__ R child_D(const Row4<R> &rw, R p, R q, double pivmin) {
    R D = fma_dd(rw.d, q, p);
    if (!(fabs(hi(D)) >= pivmin * fabs(hi(q)))) D = mul(q, mk<R>(-pivmin));
    return D;
}
template <class R>
__device__ __forceinline__ void child_rescale(R &p, R &q) {  // by a power of two (ratio kept)
    const unsigned ex = (unsigned)__double2hiint(hi(p)) & 0x7ff00000u;
    const unsigned ey = (unsigned)__double2hiint(hi(q)) & 0x7ff00000u;
    const unsigned em = ex > ey ? ex : ey;
    if (em == 0x7ff00000u || em == 0u) return;
    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
    p = scale_pow2(p, sc);
    q = scale_pow2(q, sc);
}

// One warp per cluster.  32 candidate shifts tau (lane q: side = q & 1 -- left
// end lambda_p - delta or right end lambda_q + delta -- and back-off level q >> 1,
// delta geometric from just outside the end bracket to half the outer gap;
// PAPER.md L1047-L1054 "back off further away than usual").
// Acceptance (nearest candidate first, priority = lane):
//   1. growth <= elg1 * spdiam among the four nearest back-off levels;
//   2. growth <= elg2 * spdiam, elg2 = max(10, eps_x / (eps_y sqrt(n))): the
//      relaxed k_elg of the mixed-precision setting (Eq. (3.5)),
//      which costs no accuracy; preferring a near shift under the relaxed bound
//      over a far one under the strict bound keeps the child eigenvalues small,
//      so the cluster actually splits (glued matrices: localized vectors make
//      max|d+| large exactly where the cluster's vectors are negligible --
//      "conditional" growth, Def. 2.4);
//   3. else the smallest growth (L567-L572), counted as a robustness failure.
// Growth pass: every lane runs its candidate's dstqds over the parent's rows, staged through
// shared memory (one tile read serves all 32 candidates), in projective form (one pair FMA
// chain per row; d+ = D / q only for the growth, off the chain).
// Write pass, chunk-parallel over the 32 lanes: the projective recurrence is linear in (p, q)
// (row k: (p, q) -> ((lld_k - tau) p - tau d_k q, d_k q + p)), so lane c forms the transfer
// matrix of rows [c L, (c + 1) L) from two basis solutions, lane 0 chains the 32 matrices
// into the chunk start states, and every lane re-runs its rows from its start state writing
// d+ = D / q, l+ = ld / d+, ld+ = d+ l+, lld+ = ld+ l+.  A chunk whose re-run end state
// differs from the next chunk's start state by more than 2^-100 (dd) / 2^-50 (fp64) relative,
// as a projective point -- a pivot guard fired inside it (the guard is not linear), or the
// chained products lost accuracy (strongly graded / glued parents: measured on glued
// Wilkinson, 2^-40 let a child through whose eigenvectors came out at residual 5e-13) --
// sends the whole child to the sequential write: lane 0 runs the growth pass's projective
// recurrence over rows the warp stages through shared memory.
// (dstqds: s_1 = -tau; d+_i = d_i + s_i;
// l+_i = ld_i / d+_i; s_{i+1} = l+_i l_i s_i - tau; L+D+L+^T = LDL^T - tau I.)
template <class R>
__global__ void __launch_bounds__(32) k_child(NodeInfo *nodes, int node_base, Items it,
                                              const int32_t *__restrict__ next_active,
                                              const int32_t *__restrict__ cbeg,
                                              const int32_t *__restrict__ cend, int nclus,
                                              double *child_pool, double *childx_pool,
                                              int64_t pool_stride_rows,
                                              double spdiam, double elg1, double elg2,
                                              double pivmin, DevStats *st, double *dbg,
                                              double *cfail, int mode, int force_depth) {
    constexpr int ROWD = 4 * Prec<R>::words;
    __shared__ __align__(16) double sbuf[2][CH_TR * ROWD];
    __shared__ R sS[2 * 33];  // chunk start states (p, q)
    const int c = blockIdx.x;
    if (c >= nclus) return;
    const int lane = threadIdx.x;
    const int b = cbeg[c], e = cend[c];
    const int id0 = next_active[b], id1 = next_active[e - 1];
    // mode 0: the child of the cluster's node.  mode 1 (backtracking, PAPER.md L1190-L1197,
    // reading R22): a cluster whose child failed the acceptance tests in mode 0 (cfail[c] >= 0:
    // the failed child's growth) takes its child from the grandparent instead -- a different
    // shift at a higher level of the tree -- and keeps it if it passes or grows less.
    int pnode = it.node[id0];
    R shift_in = mk<R>(0.0);  // member brackets: + shift_in = base-node coordinates
    if (mode == 1) {
        // cfail: -1 none (or no grandparent), -2 forced by the test hook, else the growth
        if (!(cfail[c] >= 0.0 || cfail[c] == -2.0)) return;  // (uniform)
        const NodeInfo C = nodes[pnode];
        pnode = nodes[C.parent].parent;
        const NodeInfo Gn = nodes[pnode];
        shift_in = sub(mk2<R>(C.sig_hi, C.sig_lo), mk2<R>(Gn.sig_hi, Gn.sig_lo));
        if (lane == 0) atomicAdd(&st->backtrack_tries, 1);
    }
    const NodeInfo P = nodes[pnode];
    const int64_t n = P.n;
    const R *lo = reinterpret_cast<const R *>(it.lo);
    const R *hi_ = reinterpret_cast<const R *>(it.hi);
    R lamL = add(lo[id0], shift_in), lamR = add(hi_[id1], shift_in);
    double wL = hi(sub(hi_[id0], lo[id0])), wR = hi(sub(hi_[id1], lo[id1]));
    double gL = it.lgap[id0], gR = it.rgap[id1];
    const int side = lane & 1, lev = lane >> 1;
    double w = side ? wR : wL;
    double g = side ? gR : gL;
    double lam_abs = fabs(hi(side ? lamR : lamL));
    double d0 = fmax(2.0 * w, 8.0 * Prec<R>::eps * lam_abs + pivmin);
    double cap = fmax(d0, fmin(0.5 * g, spdiam));
    double delta = d0 * pow(cap / d0, (double)lev / 15.0);
    R tau = side ? add(lamR, mk<R>(delta)) : sub(lamL, mk<R>(delta));
    const R mtau = neg(tau);

    double *child = child_pool + (int64_t)c * pool_stride_rows * 4 * Prec<R>::words;
    double *childx = childx_pool + (int64_t)c * pool_stride_rows * 2;
    // ---- growth pass (staged rows, one candidate per lane); lane 0's candidate -- the nearest
    // shift, the usual winner -- writes its child rows on the way (speculative write)
    double growth = 0.0;
    bool bad = false;
    {
        R p = mtau, q = mk<R>(1.0);
        const int ntile = (int)((n + CH_TR - 1) / CH_TR);
        child_stage<R>(sbuf[0], P.rep, n, 0);
#pragma unroll 1
        for (int t = 0; t < ntile; t++) {
            if (t + 1 < ntile) {
                child_stage<R>(sbuf[(t + 1) & 1], P.rep, n, (int64_t)(t + 1) * CH_TR);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncwarp();
            const double *buf = sbuf[t & 1];
            const int jn = (int)min((int64_t)CH_TR, n - (int64_t)t * CH_TR);
#pragma unroll 4
            for (int j = 0; j < jn; j++) {
                const Row4<R> rw = child_row<R>(buf, j);
                const R D = child_D<R>(rw, p, q, pivmin);
                const double dp = fabs(hi(D) * rcp(hi(q)));  // |d+| (growth only)
                bad |= !(dp <= 1e300);
                growth = fmax(growth, dp);
                if (lane == 0 && mode == 0) {
                    const int64_t k = (int64_t)t * CH_TR + j;
                    const R dpr = div(D, q);  // d+_k
                    R lp = mk<R>(0.0);
                    if (k < n - 1) lp = div(rw.ld, dpr);
                    const R ldp = mul(dpr, lp);
                    const R lldp = mul(ldp, lp);
                    store_row4<R>(child, k, dpr, lldp, lp, ldp);
                    reinterpret_cast<double2 *>(childx)[k] = make_double2(hi(dpr), hi(lldp));
                }
                p = fma_dd(mtau, D, mul(rw.lld, p));
                q = D;
                if ((j & 7) == 7) child_rescale<R>(p, q);
            }
            child_rescale<R>(p, q);
            __syncwarp();
        }
    }
    if (bad) growth = INFINITY;
    unsigned ok1 = __ballot_sync(0xffffffffu, growth <= elg1 * spdiam) & 0xffu;
    unsigned ok2 = __ballot_sync(0xffffffffu, growth <= elg2 * spdiam);
    int win;
    bool fail = false;
    if (ok1) {
        win = __ffs(ok1) - 1;
    } else if (ok2) {
        win = __ffs(ok2) - 1;
    } else {
        double gmin = growth;
        int l = lane;
        for (int o = 16; o > 0; o >>= 1) {
            double og = __shfl_xor_sync(0xffffffffu, gmin, o);
            int ol = __shfl_xor_sync(0xffffffffu, l, o);
            if (og < gmin || (og == gmin && ol < l)) {
                gmin = og;
                l = ol;
            }
        }
        win = l;
        fail = true;
    }
    const double gwin = __shfl_sync(0xffffffffu, growth, win);
    const bool was_forced = mode == 1 && cfail[c] == -2.0;
    if (mode == 1 && !was_forced && fail && !(gwin < cfail[c])) return;  // (uniform) keep mode 0's
    // test hook (MR3_BACKTRACK = 2): children at depth >= force_depth count as failed in mode 0
    const bool forced = mode == 0 && force_depth > 0 && P.depth + 1 >= force_depth;
    const R t = shfl_R<R>(0xffffffffu, tau, win, 32);
    const R mt = neg(t);
    if (win != 0 || mode == 1) {  // (uniform) the speculative child is not the chosen one: write it

    // ---- write pass, chunk-parallel (see above)
    const int64_t L = (n + 31) / 32;
    const int64_t k0 = min((int64_t)lane * L, n), k1 = min(k0 + L, n);
    // phase 1: transfer matrix of the chunk (basis solutions u = (1, 0), v = (0, 1))
    R up = mk<R>(1.0), uq = mk<R>(0.0), vp = mk<R>(0.0), vq = mk<R>(1.0);
#pragma unroll 4
    for (int64_t k = k0; k < k1; k++) {
        const Row4<R> rw = load_row4<R>(P.rep, k);
        const R U = fma_dd(rw.d, uq, up), V = fma_dd(rw.d, vq, vp);
        up = fma_dd(mt, U, mul(rw.lld, up));
        vp = fma_dd(mt, V, mul(rw.lld, vp));
        uq = U;
        vq = V;
        if (((k - k0) & 7) == 7) {  // joint power-of-two rescale (only ratios matter)
            unsigned em = (unsigned)__double2hiint(hi(up)) & 0x7ff00000u, tt;
            tt = (unsigned)__double2hiint(hi(uq)) & 0x7ff00000u;
            em = tt > em ? tt : em;
            tt = (unsigned)__double2hiint(hi(vp)) & 0x7ff00000u;
            em = tt > em ? tt : em;
            tt = (unsigned)__double2hiint(hi(vq)) & 0x7ff00000u;
            em = tt > em ? tt : em;
            if (em != 0x7ff00000u && em != 0u) {
                const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                up = scale_pow2(up, sc);
                uq = scale_pow2(uq, sc);
                vp = scale_pow2(vp, sc);
                vq = scale_pow2(vq, sc);
            }
        }
    }
    // phase 2: chunk start states (lane 0 chains the 32 matrices)
    __shared__ R sM[4 * 32];
    sM[4 * lane] = up;
    sM[4 * lane + 1] = uq;
    sM[4 * lane + 2] = vp;
    sM[4 * lane + 3] = vq;
    __syncwarp();
    if (lane == 0) {
        R p = mt, q = mk<R>(1.0);
        for (int j = 0; j < 32; j++) {
            sS[2 * j] = p;
            sS[2 * j + 1] = q;
            const R np = add(mul(p, sM[4 * j]), mul(q, sM[4 * j + 2]));
            const R nq = add(mul(p, sM[4 * j + 1]), mul(q, sM[4 * j + 3]));
            p = np;
            q = nq;
            child_rescale<R>(p, q);
        }
        sS[64] = p;
        sS[65] = q;
    }
    __syncwarp();
    // phase 3: re-run from the start state, writing the child rows
    R p = sS[2 * lane], q = sS[2 * lane + 1];
#pragma unroll 4
    for (int64_t k = k0; k < k1; k++) {
        const Row4<R> rw = load_row4<R>(P.rep, k);
        const R D = child_D<R>(rw, p, q, pivmin);
        const R dp = div(D, q);  // d+_k
        R lp = mk<R>(0.0);
        if (k < n - 1) lp = div(rw.ld, dp);
        const R ldp = mul(dp, lp);
        const R lldp = mul(ldp, lp);
        store_row4<R>(child, k, dp, lldp, lp, ldp);
        reinterpret_cast<double2 *>(childx)[k] = make_double2(hi(dp), hi(lldp));
        p = fma_dd(mt, D, mul(rw.lld, p));
        q = D;
        if (((k - k0) & 7) == 7) child_rescale<R>(p, q);
    }
    // continuity: this chunk's end state against the next chunk's start (projective points)
    bool jump = false;
    if (k1 > k0 && lane < 31 && k1 < n) {
        const R ps = sS[2 * (lane + 1)], qs = sS[2 * (lane + 1) + 1];
        const double cross = fabs(hi(sub(mul(p, qs), mul(q, ps))));
        const double mag = (fabs(hi(p)) + fabs(hi(q))) * (fabs(hi(ps)) + fabs(hi(qs)));
        // the child must be the dstqds of the parent to working precision (an element-wise
        // O(eps_y) relative perturbation, mixed relative stability): a boundary jump delta
        // perturbs d+ there by delta |s_k| / |d_k| relative, so only rounding-level jumps pass
        const double tolj = Prec<R>::words == 2 ? 0x1p-100 : 0x1p-50;
        jump = !(cross <= tolj * mag);
    }
    if (__any_sync(0xffffffffu, jump)) {
        // sequential write: the projective recurrence of the growth pass (the same guard),
        // rows staged through shared memory by the warp, lane 0 runs the chain
        __syncwarp();
        R p = mt, q = mk<R>(1.0);
        const int ntile = (int)((n + CH_TR - 1) / CH_TR);
        child_stage<R>(sbuf[0], P.rep, n, 0);
#pragma unroll 1
        for (int ti = 0; ti < ntile; ti++) {
            if (ti + 1 < ntile) {
                child_stage<R>(sbuf[(ti + 1) & 1], P.rep, n, (int64_t)(ti + 1) * CH_TR);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncwarp();
            if (lane == 0) {
                const double *buf = sbuf[ti & 1];
                const int64_t k0t = (int64_t)ti * CH_TR;
                const int jn = (int)min((int64_t)CH_TR, n - k0t);
#pragma unroll 4
                for (int j = 0; j < jn; j++) {
                    const int64_t k = k0t + j;
                    const Row4<R> rw = child_row<R>(buf, j);
                    const R D = child_D<R>(rw, p, q, pivmin);
                    const R dp = div(D, q);  // d+_k
                    R lp = mk<R>(0.0);
                    if (k < n - 1) lp = div(rw.ld, dp);
                    const R ldp = mul(dp, lp);
                    const R lldp = mul(ldp, lp);
                    store_row4<R>(child, k, dp, lldp, lp, ldp);
                    reinterpret_cast<double2 *>(childx)[k] = make_double2(hi(dp), hi(lldp));
                    p = fma_dd(mt, D, mul(rw.lld, p));
                    q = D;
                    if ((j & 7) == 7) child_rescale<R>(p, q);
                }
                child_rescale<R>(p, q);
            }
            __syncwarp();
        }
    }
    }  // win != 0
    __syncwarp();
    if (lane == win) {
        NodeInfo ch = P;
        ch.rep = child;
        ch.repx = childx;
        R sig = add(mk2<R>(P.sig_hi, P.sig_lo), t);
        ch.sig_hi = hi(sig);
        ch.sig_lo = lo_part(sig);
        ch.depth = P.depth + 1;
        ch.parent = pnode;
        if (mode == 1) {
            ch.depth = nodes[node_base + c].depth;  // (the failed child's level)
            atomicAdd(&st->backtracks, 1);
            if (!fail && !was_forced) atomicSub(&st->robustness_failures, 1);  // (mode 0's)
            if (fail && was_forced) atomicAdd(&st->robustness_failures, 1);
        }
        nodes[node_base + c] = ch;
        if (fail && mode == 0) atomicAdd(&st->robustness_failures, 1);
        if (cfail != nullptr && mode == 0)
            cfail[c] = P.depth < 1 ? -1.0 : fail ? gwin : forced ? -2.0 : -1.0;
        if (dbg) {
            dbg[4 * c + 0] = win;
            dbg[4 * c + 1] = growth;
            dbg[4 * c + 2] = delta;
            dbg[4 * c + 3] = hi(t);
        }
    }
    __syncwarp();
    // translate the member brackets into the child's coordinates (Alg. 1 l.16)
    R *wlo = reinterpret_cast<R *>(it.lo);
    R *whi = reinterpret_cast<R *>(it.hi);
    const R tt = sub(t, shift_in);
    for (int j = b + lane; j < e; j += 32) {
        int id = next_active[j];
        wlo[id] = sub(wlo[id], tt);
        whi[id] = sub(whi[id], tt);
        it.node[id] = node_base + c;
    }
}

}  // namespace mr3
