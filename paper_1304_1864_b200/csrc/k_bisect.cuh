// k_bisect.cuh -- K3 (classification) and helpers shared with the staged bisection
// (k_bisect_s.cuh, K2).
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
                                                   int cnt, double gaptol, SegOut out,
                                                   double absgap = 0.0) {
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
                // relative gap (Eq. (2.2)), or -- NEXT-3, absgap > 0 -- an absolute gap of at
                // least absgap ("amended by a criterion based on the
                // absolute separation"; R21)
                start = (den == 0.0 || gap >= gaptol * den || (absgap > 0.0 && gap >= absgap)) ? 1 : 0;
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
