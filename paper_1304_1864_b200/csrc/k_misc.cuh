// k_misc.cuh -- K7 (same-run FP64 peak and dd-step latency) and small helpers.
#pragma once
#include "kernels.cuh"

namespace mr3 {

// 8 independent DFMA chains per thread; every SM busy.  FP64 instructions
// executed = threads * 8 * iters (the loop counter is integer work).
__global__ void __launch_bounds__(256) k_fp64_peak(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4,
           x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 1
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            x0 = fma(x0, a, b);
            x1 = fma(x1, a, b);
            x2 = fma(x2, a, b);
            x3 = fma(x3, a, b);
            x4 = fma(x4, a, b);
            x5 = fma(x5, a, b);
            x6 = fma(x6, a, b);
            x7 = fma(x7, a, b);
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 123.456) out[0] = s;  // keep the chains alive
}

// one dependent chain of dd Sturm steps over a synthetic representation
__global__ void k_dd_latency(const double *rep, int64_t n, int reps, int *out) {
    int c = 0;
    for (int i = 0; i < reps; i++) c += negcount<dd>(rep, n, mkdd(0.25 + 1e-3 * i, 0.0), 1e-30);
    out[0] = c;
}

__global__ void k_fill_rep_test(double *rep, int64_t n) {
    for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double *p = rep + 8 * i;
        p[0] = 2.0;  // d
        p[1] = 0.0;
        p[2] = 0.5;  // lld
        p[3] = 0.0;
        p[4] = 0.5;  // l
        p[5] = 0.0;
        p[6] = 1.0;  // ld
        p[7] = 0.0;
    }
}

// initialise the items of the requested index set (no-split case):
// block-local index k = k0 + t, column = k - il (or -1 outside [il, iu])
template <class R>
__global__ void k_init_items(Items it, int cnt, int k0, int il, int iu, int node,
                             const double *brk /* lo, hi of the node's root bracket */) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    int k = k0 + t;
    it.node[t] = node;
    it.k[t] = k;
    it.col[t] = (k >= il && k <= iu) ? (int64_t)(k - il) : -1;
    reinterpret_cast<R *>(it.lo)[t] = mk2<R>(brk[0], brk[1]);
    reinterpret_cast<R *>(it.hi)[t] = mk2<R>(brk[2], brk[3]);
    it.lgap[t] = 1e300;
    it.rgap[t] = 1e300;
    it.x0[t] = NAN;
    it.dx[t] = INFINITY;
}

// split case: items for every eigenvalue of every block
template <class R>
__global__ void k_init_items_blocks(Items it, int total, const BlockDesc *blocks, int nblocks,
                                    const int64_t *item0 /* prefix over blocks */,
                                    const double *brk) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    int lo = 0, hi_ = nblocks - 1;
    while (lo < hi_) {  // block containing item t
        int mid = (lo + hi_ + 1) / 2;
        if (item0[mid] <= t)
            lo = mid;
        else
            hi_ = mid - 1;
    }
    int b = lo;
    it.node[t] = b;
    it.k[t] = (int)(t - item0[b]) + 1;
    it.col[t] = -1;
    reinterpret_cast<R *>(it.lo)[t] = mk2<R>(brk[4 * b + 0], brk[4 * b + 1]);
    reinterpret_cast<R *>(it.hi)[t] = mk2<R>(brk[4 * b + 2], brk[4 * b + 3]);
    it.lgap[t] = 1e300;
    it.rgap[t] = 1e300;
    it.x0[t] = NAN;
    it.dx[t] = INFINITY;
}

__global__ void k_iota(int32_t *list, int cnt, int start) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < cnt) list[t] = start + t;
}

// bracket exchange buffer <-> items (MR3_BRK_REC doubles per record: lo.hi lo.lo hi.hi
// hi.lo x0 dx -- the bracket and the Newton estimate behind the RQI start)
template <class R>
__global__ void k_items_to_brk(Items it, int first, int cnt, double *brk) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    R l = reinterpret_cast<R *>(it.lo)[first + t], h = reinterpret_cast<R *>(it.hi)[first + t];
    double *p = brk + MR3_BRK_REC * (int64_t)t;
    p[0] = hi(l);
    p[1] = lo_part(l);
    p[2] = hi(h);
    p[3] = lo_part(h);
    p[4] = it.x0[first + t];
    p[5] = it.dx[first + t];
}
template <class R>
__global__ void k_brk_to_items(Items it, int cnt, int slice_cap, int world, const double *brk) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    // item t lives in rank t / slice_cap's slice at offset t % slice_cap
    const double *p = brk + MR3_BRK_REC * (int64_t)t;
    reinterpret_cast<R *>(it.lo)[t] = mk2<R>(p[0], p[1]);
    reinterpret_cast<R *>(it.hi)[t] = mk2<R>(p[2], p[3]);
    it.x0[t] = p[4];
    it.dx[t] = p[5];
}

// output columns for the split case: global rank of each item by its midpoint
// (keys = order-preserving bits of the fp64 midpoint + sigma)
template <class R>
__global__ void k_item_keys(Items it, int cnt, const NodeInfo *nodes, unsigned long long *keys,
                            int32_t *vals) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const NodeInfo nd = nodes[it.node[t]];
    const R a = reinterpret_cast<R *>(it.lo)[t], b = reinterpret_cast<R *>(it.hi)[t];
    R m = half(add(a, b));
    // the bisection's last estimate (RQI start, far inside the bracket's tolerance) orders
    // eigenvalues of different blocks whose brackets overlap
    const double x0 = it.x0[t];
    if (!isnan(x0) && x0 > hi(a) && x0 < hi(b)) m = mk<R>(x0);
    double v = hi(add(m, mk2<R>(nd.sig_hi, nd.sig_lo)));
    unsigned long long u = (unsigned long long)__double_as_longlong(v);
    u = (u & 0x8000000000000000ULL) ? ~u : (u | 0x8000000000000000ULL);
    keys[t] = u;
    vals[t] = t;
}

// after sorting: rank -> column assignment for ranks in [c0, c1] (1-based il..iu)
// or values in (vl, vu]
__global__ void k_assign_cols(Items it, int cnt, const int32_t *sorted_ids,
                              const unsigned long long *sorted_keys, int mode, int64_t il,
                              int64_t iu, double vl, double vu, int64_t *mcount) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    int id = sorted_ids[t];
    int64_t rank = t + 1;
    bool want;
    if (mode == 0) {
        want = true;
    } else if (mode == 1) {
        want = rank >= il && rank <= iu;
    } else {
        unsigned long long u = sorted_keys[t];
        u = (u & 0x8000000000000000ULL) ? (u & 0x7FFFFFFFFFFFFFFFULL) : ~u;
        double v = __longlong_as_double((long long)u);
        want = v > vl && v <= vu;
    }
    it.col[id] = want ? rank : -1;  // provisional: rank (compacted below)
    if (want) atomicAdd((unsigned long long *)mcount, 1ULL);
}
__global__ void k_compact_cols(Items it, int cnt, const int32_t *sorted_ids, int64_t first_rank) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    int id = sorted_ids[t];
    if (it.col[id] >= 0) it.col[id] -= first_rank;
}

// ---- final order of a split matrix's eigenpairs (execute_impl): the columns were assigned from
// the plan's bracket order, so eigenvalues of different blocks that agree to within the bisection
// tolerance can come out of order after the RQI.  A stable sort of w and the same permutation
// of the Z columns, in place and cycle by cycle, restore "w ascending" (include/mr3.h).
template <class T>
__global__ void k_sort_keys(const T *__restrict__ w, int m, unsigned long long *keys,
                            int32_t *vals, int *ninv) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const double v = (double)w[t];
    unsigned long long u = (unsigned long long)__double_as_longlong(v);
    u = (u & 0x8000000000000000ULL) ? ~u : (u | 0x8000000000000000ULL);
    keys[t] = u;
    vals[t] = t;
    if (t + 1 < m && (double)w[t + 1] < v) atomicAdd(ninv, 1);
}
template <class T>
__global__ void k_gather_w(const T *__restrict__ w, const int32_t *__restrict__ perm, int m,
                           T *out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) out[t] = w[perm[t]];
}
// position t takes the old column perm[t]; t leads its cycle iff it is the cycle's smallest index
__global__ void k_cycle_leaders(const int32_t *__restrict__ perm, int m, char *leader) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    int j = perm[t];
    bool lead = j != t;
    while (lead && j != t) {
        if (j < t) lead = false;
        j = perm[j];
    }
    leader[t] = lead ? 1 : 0;
}
// one CTA column (blockIdx.x) per cycle leader, rows over blockIdx.y and the threads
template <class T>
__global__ void k_permute_cols(T *Z, int64_t ldz, int64_t n, const int32_t *__restrict__ perm,
                               const char *__restrict__ leader) {
    const int t = blockIdx.x;
    if (!leader[t]) return;
    for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.y * blockDim.x) {
        const T save = Z[(int64_t)t * ldz + i];
        int j = t;
        for (;;) {
            const int src = perm[j];
            if (src == t) {
                Z[(int64_t)j * ldz + i] = save;
                break;
            }
            Z[(int64_t)j * ldz + i] = Z[(int64_t)src * ldz + i];
            j = src;
        }
    }
}

}  // namespace mr3
