// k_grid.cuh -- K2 start: eigenvalue brackets from a shared grid of Sturm counts.
//
// Alg. 1 l.3 starts every eigenvalue's bisection from the
// root's enclosure; the first log2(m) or so halvings of all m brackets are then
// the same few points counted m times over.  Here they are counted once: a
// uniform grid of GRID_L1 points over the root enclosure [L, U] locates the
// sub-interval holding the requested indices, and a second uniform grid of M2
// (about 1.5 per requested eigenvalue) points over that sub-interval gives every
// index k the grid cell [x_j, x_{j+1}] with count(x_j) < k <= count(x_{j+1})
// (binary search; the invariant holds even if rounding made the counts locally
// non-monotone).  The multisection of k_bisect_s continues from that cell.
// Counts are binary_x (projective, on M_x) for fp64 I/O -- the brackets are then
// binary_x brackets, certified in binary_y after the binary_x phase like any
// other (k_bisect_s) -- and binary_y (= binary64) for fp32 I/O.
// Grid positions are a function of the global index set only, so every rank of
// the two-phase form sees the same points (it counts only those in its slice).
#pragma once
#include "k_bisect_s.cuh"

namespace mr3 {

constexpr int GRID_L1 = 2048;

struct GridInfo {
    double L, U;       // root enclosure: count(L) = 0, count(U) = n
    double xa, xb;     // level-2 interval of the global index set
    double sa, sb;     // this slice's sub-interval (level-1 points or L, U)
    int csa, csb;      // counts at sa, sb
    int j0, j1;        // level-2 points inside (sa, sb): j0 .. j1 (j1 < j0: none)
    int m2;            // level-2 points over (xa, xb)
    int pad;
};

__global__ void k_grid_init(GridInfo *gi, const double *brk) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        gi->L = brk[0] + brk[1];
        gi->U = brk[2] + brk[3];
    }
}

__device__ __forceinline__ double grid_pt(double a, double b, int j, int m) {
    return a + (b - a) * ((double)(j + 1) / (double)(m + 1));
}

// level 1 (level == 1): points j in [0, GRID_L1) over (L, U); level 2: j in
// [j0, j1] over (xa, xb).  One point per thread, CTA-collective staged counts.
template <class R, bool XMODE>
__global__ void __launch_bounds__(BS_TPB) k_grid_counts(const NodeInfo *__restrict__ nodes,
                                                     int node, int level,
                                                     const GridInfo *__restrict__ gi, int *cnt,
                                                     double pivmin, double pivmin_x) {
    __shared__ __align__(16) double sbuf[2 * BS_TILE];
    const GridInfo g = *gi;
    const int j = blockIdx.x * BS_TPB + threadIdx.x;
    int lo = 0, hi = GRID_L1 - 1, m = GRID_L1;
    double a = g.L, b = g.U;
    if (level == 2) {
        lo = g.j0;
        hi = g.j1;
        m = g.m2;
        a = g.xa;
        b = g.xb;
    }
    const int cta0 = blockIdx.x * BS_TPB;
    if (cta0 > hi || cta0 + BS_TPB - 1 < lo) return;  // whole CTA outside the range
    const NodeInfo nd = nodes[node];
    const bool need = j >= lo && j <= hi;
    const double x = grid_pt(a, b, j, m);
    int c;
    if (XMODE) {
        c = count_x_cta(sbuf, nd, need, x, pivmin_x);
    } else {
        int dummy;
        count_y_cta<R, false>(sbuf, nd, need, mk<R>(x), mk<R>(x), pivmin, c, dummy);
    }
    if (need) cnt[j] = c;
}

// first j in [lo, hi] with cnt[j] >= k (hi + 1 if none), on a possibly
// non-monotone array: keeps count(left) < k <= count(right) with virtual ends
__device__ __forceinline__ int grid_search(const int *cnt, int lo, int hi, int k) {
    int l = lo - 1, r = hi + 1;  // cnt[l] < k (virtual), cnt[r] >= k (virtual)
    while (r - l > 1) {
        int mid = (l + r) >> 1;
        if (cnt[mid] >= k)
            r = mid;
        else
            l = mid;
    }
    return r;
}

// level-2 plan from the level-1 counts.  k_lo..k_hi: global index set; k_first..k_last: slice.
__global__ void k_grid_setup(GridInfo *gi, const double *brk, const int *cnt1, int n, int k_lo,
                             int k_hi, int k_first, int k_last, int m2) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    GridInfo g;
    g.L = brk[0] + brk[1];
    g.U = brk[2] + brk[3];
    auto pt1 = [&](int j) -> double {
        return j < 0 ? g.L : (j >= GRID_L1 ? g.U : grid_pt(g.L, g.U, j, GRID_L1));
    };
    auto c1 = [&](int j) -> int { return j < 0 ? 0 : (j >= GRID_L1 ? n : cnt1[j]); };
    // global interval: left end = last point with count < k_lo, right end = first with count >= k_hi
    int r = grid_search(cnt1, 0, GRID_L1 - 1, k_lo);
    g.xa = pt1(r - 1);
    r = grid_search(cnt1, 0, GRID_L1 - 1, k_hi);
    g.xb = pt1(r);
    r = grid_search(cnt1, 0, GRID_L1 - 1, k_first);
    g.sa = pt1(r - 1);
    g.csa = c1(r - 1);
    r = grid_search(cnt1, 0, GRID_L1 - 1, k_last);
    g.sb = pt1(r);
    g.csb = c1(r);
    g.m2 = m2;
    // level-2 points strictly inside (sa, sb)
    const double span = g.xb - g.xa;
    int j0 = 0, j1 = m2 - 1;
    if (span > 0) {
        j0 = (int)floor((g.sa - g.xa) / span * (m2 + 1)) - 1;
        j1 = (int)ceil((g.sb - g.xa) / span * (m2 + 1)) - 1;
        j0 = max(j0, 0);
        j1 = min(j1, m2 - 1);
        while (j0 <= j1 && !(grid_pt(g.xa, g.xb, j0, m2) > g.sa)) j0++;
        while (j1 >= j0 && !(grid_pt(g.xa, g.xb, j1, m2) < g.sb)) j1--;
    } else {
        j1 = -1;
    }
    g.j0 = j0;
    g.j1 = j1;
    g.pad = 0;
    *gi = g;
}

// brackets of the slice's items [first, first + cnt) from the level-2 counts
template <class R>
__global__ void k_grid_assign(Items it, int first, int cnt, const GridInfo *__restrict__ gi,
                              const int *__restrict__ cnt2) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const GridInfo g = *gi;
    const int id = first + t;
    const int k = it.k[id];
    double lo = g.sa, hi = g.sb;
    if (g.csa < k && k <= g.csb) {
        const int r = grid_search(cnt2, g.j0, g.j1, k);
        if (r - 1 >= g.j0) lo = grid_pt(g.xa, g.xb, r - 1, g.m2);
        if (r <= g.j1) hi = grid_pt(g.xa, g.xb, r, g.m2);
    } else {
        return;  // keep the root enclosure (counts inconsistent with the slice plan)
    }
    reinterpret_cast<R *>(it.lo)[id] = mk<R>(lo);
    reinterpret_cast<R *>(it.hi)[id] = mk<R>(hi);
}

}  // namespace mr3
