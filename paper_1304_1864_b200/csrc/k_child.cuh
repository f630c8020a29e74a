// k_child.cuh -- K4: child representations for clusters (Alg. 1 l.15-17).
#pragma once
#include "k_bisect.cuh"

namespace mr3 {

// dstqds with shift tau:
//   s_1 = -tau ; d+_i = d_i + s_i ; l+_i = ld_i / d+_i ; s_{i+1} = l+_i l_i s_i - tau
// L+D+L+^T = LDL^T - tau I.  Returns max_i |d+_i| (element-growth surrogate,
// Def. 2.4 L542-L556 / SPEC S:130-136) or +inf if anything is not finite.
template <class R>
__device__ double dstqds_growth(const double *__restrict__ rep, int64_t n, R tau, double pivmin) {
    R s = neg(tau);
    double g = 0.0;
    bool bad = false;
#pragma unroll 1
    for (int64_t i = 0; i < n; i++) {
        Row4<R> r = load_row4<R>(rep, i);
        R dp = guard(add(r.d, s), pivmin);
        double a = fabs(hi(dp));
        if (!(a <= 1e300)) bad = true;
        g = fmax(g, a);
        if (i < n - 1) {
            R lp = div(r.ld, dp);
            s = sub(mul(mul(lp, r.l), s), tau);
        }
    }
    return bad ? INFINITY : g;
}

template <class R>
__device__ void dstqds_write(const double *__restrict__ rep, int64_t n, R tau, double pivmin,
                             double *__restrict__ child, double *__restrict__ childx) {
    R s = neg(tau);
#pragma unroll 1
    for (int64_t i = 0; i < n; i++) {
        Row4<R> r = load_row4<R>(rep, i);
        R dp = guard(add(r.d, s), pivmin);
        R lp = mk<R>(0.0);
        if (i < n - 1) {
            lp = div(r.ld, dp);
            s = sub(mul(mul(lp, r.l), s), tau);
        }
        R ldp = mul(dp, lp);
        R lldp = mul(ldp, lp);
        store_row4<R>(child, i, dp, lldp, lp, ldp);
        reinterpret_cast<double2 *>(childx)[i] = make_double2(hi(dp), hi(lldp));
    }
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
template <class R>
__global__ void __launch_bounds__(32) k_child(NodeInfo *nodes, int node_base, Items it,
                                              const int32_t *__restrict__ next_active,
                                              const int32_t *__restrict__ cbeg,
                                              const int32_t *__restrict__ cend, int nclus,
                                              double *child_pool, double *childx_pool,
                                              int64_t pool_stride_rows,
                                              double spdiam, double elg1, double elg2,
                                              double pivmin, DevStats *st, double *dbg) {
    const int c = blockIdx.x;
    if (c >= nclus) return;
    const int lane = threadIdx.x;
    const int b = cbeg[c], e = cend[c];
    const int id0 = next_active[b], id1 = next_active[e - 1];
    const int pnode = it.node[id0];
    const NodeInfo P = nodes[pnode];
    const R *lo = reinterpret_cast<const R *>(it.lo);
    const R *hi_ = reinterpret_cast<const R *>(it.hi);
    R lamL = lo[id0], lamR = hi_[id1];
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
    double growth = dstqds_growth<R>(P.rep, P.n, tau, pivmin);
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
    R t = shfl_R<R>(0xffffffffu, tau, win, 32);
    double *child = child_pool + (int64_t)c * pool_stride_rows * 4 * Prec<R>::words;
    double *childx = childx_pool + (int64_t)c * pool_stride_rows * 2;
    if (lane == win) {
        dstqds_write<R>(P.rep, P.n, t, pivmin, child, childx);
        NodeInfo ch = P;
        ch.rep = child;
        ch.repx = childx;
        R sig = add(mk2<R>(P.sig_hi, P.sig_lo), t);
        ch.sig_hi = hi(sig);
        ch.sig_lo = lo_part(sig);
        ch.depth = P.depth + 1;
        nodes[node_base + c] = ch;
        if (fail) atomicAdd(&st->robustness_failures, 1);
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
    for (int j = b + lane; j < e; j += 32) {
        int id = next_active[j];
        wlo[id] = sub(wlo[id], t);
        whi[id] = sub(whi[id], t);
        it.node[id] = node_base + c;
    }
}

}  // namespace mr3
