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
constexpr int GRID_LEVELS = 3;  // adaptive levels after the uniform one
constexpr int CELL_PMIN = 64;   // points per subdivided cell, at least

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

// ---- adaptive levels: cells holding two or more eigenvalues are subdivided ----------
//
// After level 1 every requested index k has a cell [lo, hi] with counts clo < k <= chi.
// A cell holding c = chi - clo >= 2 eigenvalues is cut by P = 2c + 1 uniform points (at least
// 64 from the second adaptive level on, where only clusters are left); every
// index of the cell finds its sub-cell by binary search in their counts.  Repeated for a
// few levels this isolates the eigenvalues at the ends of spectra whose density grows
// there (Gauss nodes cluster quadratically at +-1), where one uniform grid cannot.
// The points of a cell are a function of (lo, hi, clo, chi) only -- global quantities --
// so every rank of the two-phase form computes the same cells for its slice.

struct CellSet {      // per slice item t (item first + t)
    double *lo, *hi;  // cell bounds
    int *clo, *chi;   // counts at lo, hi
    double *lo2, *hi2;  // next level (k_cell_assign writes here; the host swaps)
    int *clo2, *chi2;
    int *P;           // points this item's cell gets (leaders only, else 0)
    int *off;         // exclusive prefix of P
    int *lead;        // slice position of the item's cell leader
    int *total;       // device: sum of P
};

__device__ __forceinline__ double cell_pt(double lo, double hi, int i, int P) {
    return lo + (hi - lo) * ((double)(i + 1) / (double)(P + 1));
}

// level 1: cells from the uniform level-1 grid
__global__ void k_cell_init(CellSet cs, const GridInfo *__restrict__ gi, const int *__restrict__ cnt1,
                            int n, const int32_t *__restrict__ kk, int mine) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= mine) return;
    const GridInfo g = *gi;
    const int k = kk[t];
    const int r = grid_search(cnt1, 0, GRID_L1 - 1, k);
    cs.lo[t] = r - 1 < 0 ? g.L : grid_pt(g.L, g.U, r - 1, GRID_L1);
    cs.hi[t] = r >= GRID_L1 ? g.U : grid_pt(g.L, g.U, r, GRID_L1);
    cs.clo[t] = r - 1 < 0 ? 0 : cnt1[r - 1];
    cs.chi[t] = r >= GRID_L1 ? n : cnt1[r];
}

// leaders (first slice item of each cell) and their point counts
__global__ void k_cell_plan(CellSet cs, int *lead0, int mine, double rtol, double absfloor,
                            int pmin) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= mine) return;
    const double lo = cs.lo[t], hi = cs.hi[t];
    const bool lead = t == 0 || cs.lo[t - 1] != lo || cs.hi[t - 1] != hi;
    const int c = cs.chi[t] - cs.clo[t];
    const double tol = fmax(2.0 * rtol * fmax(fabs(lo), fabs(hi)), absfloor);
    cs.P[t] = (lead && c >= 2 && hi - lo > tol) ? max(2 * c + 1, pmin) : 0;
    lead0[t] = lead ? t : -1;  // (max-scanned into cs.lead)
}

__global__ void k_cell_total(CellSet cs, int mine) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *cs.total = cs.off[mine - 1] + cs.P[mine - 1];
}

// counts at the points (one per thread, CTA-collective staged counts on the root node)
template <class R, bool XMODE>
__global__ void __launch_bounds__(BS_TPB) k_cell_counts(const NodeInfo *__restrict__ nodes,
                                                        CellSet cs, int mine, int *cnt,
                                                        double pivmin, double pivmin_x) {
    __shared__ __align__(16) double sbuf[2 * BS_TILE];
    const int total = *cs.total;
    const NodeInfo nd = nodes[0];
    // grid-stride over the points (uniform trip count per CTA: the counts are collective)
    for (int base = blockIdx.x * BS_TPB; base < total; base += gridDim.x * BS_TPB) {
        const int t = base + threadIdx.x;
        const bool need = t < total;
        double x = 0.0;
        if (need) {
            int l = 0, r = mine;  // last L with off[L] <= t (it owns t: off[L] + P[L] > t)
            while (r - l > 1) {
                const int mid = (l + r) >> 1;
                if (cs.off[mid] <= t)
                    l = mid;
                else
                    r = mid;
            }
            x = cell_pt(cs.lo[l], cs.hi[l], t - cs.off[l], cs.P[l]);
        }
        int c;
        if (XMODE) {
            c = count_x_cta(sbuf, nd, need, x, pivmin_x);
        } else {
            int dummy;
            count_y_cta<R, false>(sbuf, nd, need, mk<R>(x), mk<R>(x), pivmin, c, dummy);
        }
        if (need) cnt[t] = c;
    }
}

// every item: its sub-cell in its leader's points (keeps clo < k <= chi with virtual ends)
__global__ void k_cell_assign(CellSet cs, int mine, const int32_t *__restrict__ kk,
                              const int *__restrict__ cnt) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= mine) return;
    const int L = cs.lead[t];
    const int P = cs.P[L];
    const double lo = cs.lo[t], hi = cs.hi[t];  // = the leader's (same cell)
    const int clo = cs.clo[t], chi = cs.chi[t];
    double nlo = lo, nhi = hi;
    int nclo = clo, nchi = chi;
    const int k = kk[t];
    const int *c = cnt + cs.off[L];
    const int r = P > 0 ? grid_search(c, 0, P - 1, k) : 0;
    if (P > 0 && r - 1 >= 0) {
        nlo = cell_pt(lo, hi, r - 1, P);
        nclo = c[r - 1];
    }
    if (P > 0 && r <= P - 1) {
        nhi = cell_pt(lo, hi, r, P);
        nchi = c[r];
    }
    cs.lo2[t] = nlo;
    cs.hi2[t] = nhi;
    cs.clo2[t] = nclo;
    cs.chi2[t] = nchi;
}

// final cells -> item brackets; a cell end whose count shows it isolates lambda_k (count k - 1
// on the left, k on the right) is handed to the bisection as an isolation point of NEXT-1b
// (k_bisect_s Iso; carried in lgap / rgap, which classification overwrites later)
template <class R>
__global__ void k_cell_final(Items it, int first, int mine, CellSet cs,
                             const int32_t *__restrict__ kk) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= mine) return;
    reinterpret_cast<R *>(it.lo)[first + t] = mk<R>(cs.lo[t]);
    reinterpret_cast<R *>(it.hi)[first + t] = mk<R>(cs.hi[t]);
    const int k = kk[t];
    it.lgap[first + t] = cs.clo[t] == k - 1 ? cs.lo[t] : NAN;
    it.rgap[first + t] = cs.chi[t] == k ? cs.hi[t] : NAN;
}

}  // namespace mr3
