// k_bisect.cuh -- K2 (batched bisection / multisection) and K3 (classification).
#pragma once
#include "kernels.cuh"

namespace mr3 {

template <class R>
__device__ __forceinline__ R shfl_R(unsigned mask, R v, int src, int width);
template <>
__device__ __forceinline__ double shfl_R<double>(unsigned mask, double v, int src, int width) {
    return __shfl_sync(mask, v, src, width);
}
template <>
__device__ __forceinline__ dd shfl_R<dd>(unsigned mask, dd v, int src, int width) {
    return mkdd(__shfl_sync(mask, v.hi, src, width), __shfl_sync(mask, v.lo, src, width));
}
template <class R>
__device__ __forceinline__ bool same(R a, R b) {
    return hi(a) == hi(b) && lo_part(a) == lo_part(b);
}

__device__ __forceinline__ void warp_add_u64(unsigned long long v, unsigned long long *dst) {
    unsigned mask = __activemask();
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    // lanes of `mask` each hold a (partial) sum; only the lowest active lane adds
    // when the mask is full, otherwise every lane adds its own (unreduced) value.
    if (mask == 0xffffffffu) {
        if ((threadIdx.x & 31) == 0) atomicAdd(dst, v);
    }
}

// ---------------------------------------------------------------------------
// K2: eigenvalue approximation to relative accuracy rtol (Alg. 1 l.3
// and l.16, L302-L304, L326-L328; Eq. (2.2); rtol = 1e-2 * gaptol,
// L1294-L1295) by Sturm counts of the node's representation.
//
// A group of G lanes (G | 32) owns one eigenvalue index k: each round the
// bracket [a, b] (count(a) < k <= count(b)) is cut into G+1 equal parts and
// lane j counts at a + (b - a)(j+1)/(G+1); the new bracket is the part whose
// left count is < k and right count >= k.  G = 1 is plain bisection.
// With certify != 0 the incoming bracket (translated from the parent, Alg. 1
// l.16) is first checked and widened until count(a) < k <= count(b).
// The path of every index depends only on (representation, k, bracket, G).
// ---------------------------------------------------------------------------
// Multisection rounds of a group of G lanes on [a, b] to width <= tol.
// Count is a functor (T x) -> count; T is the bracket type (R or double).
template <class T, int G, class Count>
__device__ __forceinline__ void multisect(T &a, T &b, int k, int lig, int lane, unsigned gmask,
                                          double rtol, double absfloor, double tolmul,
                                          unsigned long long &rows, int64_t n, Count count) {
#pragma unroll 1
    for (int round = 0; round < 4000; round++) {
        T w = sub(b, a);
        double tol = tolmul * fmax(2.0 * rtol * fmax(fabs(hi(a)), fabs(hi(b))), absfloor);
        if (hi(w) <= tol) break;
        T x = add(a, mul(w, (double)(lig + 1) / (double)(G + 1)));
        bool above = lt(a, x);
        bool below = lt(x, b);
        int c;
        if (above && below) {
            c = count(x);
            rows += n;
        } else {
            c = above ? k : k - 1;  // x == b counts as "right of lambda_k", x == a as left
        }
        bool P = c >= k;
        unsigned bal = __ballot_sync(gmask, P);
        bal = (bal >> (lane & ~(G - 1) & 31)) & ((G == 32) ? 0xffffffffu : ((1u << G) - 1u));
        int first = bal ? __ffs(bal) : G + 1;  // 1-based point index of the first P
        T xb = shfl_R<T>(gmask, x, first <= G ? first - 1 : 0, G);
        T xa = shfl_R<T>(gmask, x, first >= 2 ? first - 2 : 0, G);
        T nb = first <= G ? xb : b;
        T na = first >= 2 ? xa : a;
        if (same(na, a) && same(nb, b)) break;  // no representable progress
        a = na;
        b = nb;
    }
}

// ---------------------------------------------------------------------------
// K2: eigenvalue approximation to relative accuracy rtol (Alg. 1 l.3
// and l.16, L302-L304, L326-L328; Eq. (2.2); rtol = 1e-2 * gaptol,
// L1294-L1295) by Sturm counts of the node's representation.
//
// A group of G lanes (G | 32) owns one eigenvalue index k: each round the
// bracket [a, b] (count(a) < k <= count(b)) is cut into G+1 equal parts and
// lane j counts at a + (b - a)(j+1)/(G+1); the new bracket is the part whose
// left count is < k and right count >= k.  G = 1 is plain bisection.
//
// XPHASE (fp64 I/O): the rounds run first in binary_x on the narrowed copy M_x
// (L1064-L1111: "One creates a temporary copy of M_y in binary_x"; the paper's
// double/quad solver does all approximation and refinement this way,
// L1318-L1322) to half the target width; the result is widened by
// delta = 8 eps_x sqrt(n) |lambda| (the M_y -> M_x perturbation, Eq. (3.8)) and
// certified by two Sturm counts in binary_y; failed ends are widened by 8x until
// certified, and binary_y rounds finish whatever width is left.  So every
// returned bracket satisfies count_y(a) < k <= count_y(b) regardless of the
// fp64 phase.  With certify != 0 the incoming bracket (translated from the
// parent, Alg. 1 l.16) is first checked the same way.
// The path of every index depends only on (representation, k, bracket, G).
// ---------------------------------------------------------------------------
template <class R, int G>
__device__ __forceinline__ void certify_bracket(const NodeInfo &nd, R &a, R &b, int k, int lig,
                                                unsigned gmask, double absfloor, double delta,
                                                double pivmin, unsigned long long &rows) {
    for (int tries = 0; tries < 200; tries++) {
        int ca, cb;
        if (G == 1) {
            ca = negcount<R>(nd.rep, nd.n, a, pivmin);
            cb = negcount<R>(nd.rep, nd.n, b, pivmin);
            rows += 2 * nd.n;
        } else {
            int c = 0;
            if (lig < 2) {
                c = negcount<R>(nd.rep, nd.n, lig == 0 ? a : b, pivmin);
                rows += nd.n;
            }
            ca = __shfl_sync(gmask, c, 0, G);
            cb = __shfl_sync(gmask, c, 1, G);
        }
        if (ca < k && cb >= k) break;
        double w = fmax(delta, fmax(absfloor, 1e-3 * fabs(hi(b)) * (tries > 2 ? 1.0 : 0.0)));
        w = w * (double)(1ULL << (3 * (tries < 20 ? tries : 20)));
        if (ca >= k) a = sub(a, mk<R>(w));
        if (cb < k) b = add(b, mk<R>(w));
    }
}

template <class R, int G, bool XPHASE>
__global__ void __launch_bounds__(128, 6) k_bisect(const NodeInfo *__restrict__ nodes, Items it,
                                                const int32_t *__restrict__ list, int cnt,
                                                double rtol, double absfloor, double pivmin,
                                                double pivmin_x, double eps_x, int certify,
                                                DevStats *st) {
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = gtid / G;
    const int lig = gtid % G;  // lane in group
    if (item >= cnt) return;   // a whole group leaves together (G | blockDim)
    const int lane = threadIdx.x & 31;
    const unsigned gmask =
        (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const int id = list[item];
    const NodeInfo nd = nodes[it.node[id]];
    const int k = it.k[id];
    R a = reinterpret_cast<R *>(it.lo)[id];
    R b = reinterpret_cast<R *>(it.hi)[id];
    unsigned long long rows = 0, rows_x = 0;
    const double delta0 = 8.0 * eps_x * sqrt((double)nd.n);

    if (certify) certify_bracket<R, G>(nd, a, b, k, lig, gmask, absfloor, absfloor, pivmin, rows);
    if (XPHASE) {
        double ax = hi(a), bx = hi(b);
        multisect<double, G>(ax, bx, k, lig, lane, gmask, rtol, absfloor, 0.5, rows_x, nd.n,
                             [&](double x) { return negcount_x(nd.repx, nd.n, x, pivmin_x); });
        double mag = fmax(fabs(ax), fabs(bx));
        double delta = delta0 * mag + absfloor;
        R na = mk<R>(ax - delta), nb = mk<R>(bx + delta);
        // never leave the certified incoming bracket
        if (lt(na, a)) na = a;
        if (lt(b, nb)) nb = b;
        a = na;
        b = nb;
        certify_bracket<R, G>(nd, a, b, k, lig, gmask, absfloor, delta, pivmin, rows);
    }
    multisect<R, G>(a, b, k, lig, lane, gmask, rtol, absfloor, 1.0, rows, nd.n,
                    [&](R x) { return negcount<R>(nd.rep, nd.n, x, pivmin); });
    if (lig == 0) {
        reinterpret_cast<R *>(it.lo)[id] = a;
        reinterpret_cast<R *>(it.hi)[id] = b;
    }
    if (rows) atomicAdd(&st->bisect_rows, rows);
    if (rows_x) atomicAdd(&st->bisect_rows_x, rows_x);
}

// ---------------------------------------------------------------------------
// K2': starting points for RQI.  Each RQI step restarts inverse iteration from
// e_r, so its error contracts like e1 ~ C e0^2 / gap; two iterations (one RQ
// correction + the converged solve) need e0 <= gap sqrt(eps_x sqrt(n) / C).  A
// singleton whose certified bracket is wider than that (small gaps near the
// spectrum ends) gets x0 from a binary_x multisection on M_x to a few ulps; the
// others keep x0 = NaN (bracket midpoint).  x0 needs no certification: the RQI
// keeps the certified binary_y bracket as its guard.
// ---------------------------------------------------------------------------
template <class R, int G>
__global__ void __launch_bounds__(128) k_refine_x0(const NodeInfo *__restrict__ nodes, Items it,
                                                   const int32_t *__restrict__ list, int cnt,
                                                   double eps_x, double pivmin_x, double cconv,
                                                   DevStats *st) {
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = gtid / G;
    const int lig = gtid % G;
    if (item >= cnt) return;
    const int lane = threadIdx.x & 31;
    const unsigned gmask =
        (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const int id = list[item];
    const NodeInfo nd = nodes[it.node[id]];
    const int k = it.k[id];
    const R a = reinterpret_cast<R *>(it.lo)[id];
    const R b = reinterpret_cast<R *>(it.hi)[id];
    const double gap = fmin(it.lgap[id], it.rgap[id]);
    const double need = gap * sqrt(eps_x * sqrt((double)nd.n) / cconv);
    if (!(0.5 * hi(sub(b, a)) > need) || nd.n < 2) {
        if (lig == 0) it.x0[id] = NAN;
        return;
    }
    double ax = hi(a), bx = hi(b);
    unsigned long long rows_x = 0;
    // to a few ulps: relative 4 eps_x (multisect's tol is 2 rtol max|.|)
    multisect<double, G>(ax, bx, k, lig, lane, gmask, 2.0 * eps_x, 1e-300, 1.0, rows_x, nd.n,
                         [&](double x) { return negcount_x(nd.repx, nd.n, x, pivmin_x); });
    if (lig == 0) {
        double x = 0.5 * (ax + bx);
        it.x0[id] = (x > hi(a) && x < hi(b)) ? x : NAN;
    }
    if (rows_x) atomicAdd(&st->bisect_rows_x, rows_x);
}

// ---------------------------------------------------------------------------
// K3: classification (Alg. 1 l.7, L309-L310; reldist, L593-L612):
//   reldist(j, j+1) = (lo_{j+1} - hi_j) / max(|lo_j|, |hi_j|, |lo_{j+1}|, |hi_{j+1}|)
// >= gaptol separates j and j+1 (zero denominator: separated).
// One CTA of 1024 threads walks the active list (sorted item ids) in chunks:
// segment flags -> scan -> segments -> singleton list, cluster list and the
// member list of the next level.  Also refreshes the neighbour gaps.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int block_excl_scan(int v, int *total, int *sh /* 33 */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        int nw = blockDim.x >> 5;
        int s = lane < nw ? sh[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) sh[lane] = s;  // inclusive warp totals
        if (lane == nw - 1) sh[32] = s;
    }
    __syncthreads();
    int base = w > 0 ? sh[w - 1] : 0;
    int res = base + x - v;
    *total = sh[32];
    __syncthreads();
    return res;
}

struct SegOut {
    int32_t *singles;   // item ids of wanted singletons
    int32_t *clus_beg;  // per cluster: [beg, end) into next_active
    int32_t *clus_end;
    int32_t *next_active;
    int32_t *seg_begin;  // scratch: cnt + 1
    int32_t *seg_want;   // scratch: cnt (zeroed here)
    int32_t *counts;     // [0] singles, [1] clusters, [2] members, [3] segments
    DevStats *st;
};

template <class R>
__global__ void __launch_bounds__(1024) k_classify(Items it, const int32_t *__restrict__ list,
                                                   int cnt, double gaptol, SegOut out) {
    __shared__ int sh[33];
    __shared__ int carry[4];
    if (threadIdx.x < 4) carry[threadIdx.x] = 0;
    for (int p = threadIdx.x; p < cnt; p += blockDim.x) out.seg_want[p] = 0;
    __syncthreads();
    const R *lo = reinterpret_cast<const R *>(it.lo);
    const R *hi_ = reinterpret_cast<const R *>(it.hi);
    // pass 1: segment starts and ids
    for (int base = 0; base < cnt; base += blockDim.x) {
        int p = base + threadIdx.x;
        int start = 0;
        int id = -1;
        if (p < cnt) {
            id = list[p];
            bool contiguous = p > 0 && list[p - 1] == id - 1 && it.node[id - 1] == it.node[id];
            if (!contiguous) {
                start = 1;
            } else {
                R l1 = lo[id], h0 = hi_[id - 1], l0 = lo[id - 1], h1 = hi_[id];
                double gap = hi(sub(l1, h0));
                double den = fmax(fmax(fabs(hi(l0)), fabs(hi(h0))), fmax(fabs(hi(l1)), fabs(hi(h1))));
                it.lgap[id] = gap;
                it.rgap[id - 1] = gap;
                start = (den == 0.0 || gap >= gaptol * den) ? 1 : 0;
            }
        }
        int tot;
        int ex = block_excl_scan(start, &tot, sh);
        int seg = carry[0] + ex + start - 1;  // id of the segment p belongs to
        if (p < cnt) {
            if (start) out.seg_begin[seg] = p;
            if (it.col[id] >= 0) atomicOr(&out.seg_want[seg], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) carry[0] += tot;
        __syncthreads();
    }
    const int nseg = carry[0];
    if (threadIdx.x == 0) out.seg_begin[nseg] = cnt;
    __syncthreads();
    // pass 2: singletons, clusters, members
    for (int base = 0; base < nseg; base += blockDim.x) {
        int s = base + threadIdx.x;
        int size = 0, want = 0;
        if (s < nseg) {
            size = out.seg_begin[s + 1] - out.seg_begin[s];
            want = out.seg_want[s];
        }
        int single = (s < nseg && size == 1 && want) ? 1 : 0;
        int clus = (s < nseg && size > 1 && want) ? 1 : 0;
        int t1, t2, t3;
        int ps = block_excl_scan(single, &t1, sh);
        int pc = block_excl_scan(clus, &t2, sh);
        int pm = block_excl_scan(clus ? size : 0, &t3, sh);
        if (single) out.singles[carry[1] + ps] = list[out.seg_begin[s]];
        if (clus) {
            int mb = carry[3] + pm;
            out.clus_beg[carry[2] + pc] = mb;
            out.clus_end[carry[2] + pc] = mb + size;
            for (int j = 0; j < size; j++) out.next_active[mb + j] = list[out.seg_begin[s] + j];
            atomicMax(&out.st->largest_cluster, size);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            carry[1] += t1;
            carry[2] += t2;
            carry[3] += t3;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out.counts[0] = carry[1];
        out.counts[1] = carry[2];
        out.counts[2] = carry[3];
        out.counts[3] = nseg;
        out.st->n_clusters += carry[2];
    }
}

}  // namespace mr3
