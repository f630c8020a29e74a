// mr3.cu -- B2 (level-by-level representation-tree scheduler) and B3 (C-ABI).
//
// Algorithm 1 of PAPER.md (L287-L337) executed breadth-first, one tree level
// per round of kernel launches: every singleton of a level goes
// to K5 in one batched launch, every cluster of a level to K4 (one warp each),
// then the cluster members are refined (K2) and classified (K3) in the child
// coordinates.  The host only sizes launches (a few counters per level).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is loaded lazily (nccl_api below)
#include <cublas_v2.h>  // types only: libcublas.so.12 is loaded lazily (dense pipeline)

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/mr3.h"
#include "k_bisect.cuh"
#include "k_bisect_s.cuh"
#include "k_grid.cuh"
#include "k_child.cuh"
#include "k_misc.cuh"
#include "k_rqi.cuh"
#include "k_rqi_fb.cuh"
#include "k_rqi_chunk.cuh"
#include "k_dense.cuh"
#include "kernels.cuh"

using namespace mr3;

namespace {

struct Buf {
    void *p = nullptr;
    size_t cap = 0;
};

struct KTime {
    const char *name;
    cudaEvent_t a, b;
};

struct Cfg {  // per-mode parameters
    double v[MR3_NPARAM];
};

}  // namespace

struct mr3_ctx_s {
    double t_last = 0.0;  // host wall time of the last synchronisation point (MR3_DEBUG & 2)
    int dump = 0;         // MR3_DEBUG & 1: items to dump
    int grid_levels = 0;  // adaptive grid levels of the last plan (diagnostics)
    cudaStream_t side = nullptr;              // internal stream (root PP rows)
    cudaEvent_t ev_root = nullptr, ev_pp = nullptr;
    int fuse_scale = 1;   // K6 normalisation inside k_rqi (MR3_FUSE_SCALE=0 in the environment: k_zscale)
    size_t mem_free = 0;  // device free memory seen by the first solve (RQI scratch budget)
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int nsm = 148;
    std::map<std::string, Buf> bufs;
    Cfg cfg[2];
    std::string err;
    std::vector<KTime> kt;
    size_t kt_used = 0;
    std::vector<std::pair<std::string, std::pair<double, int>>> ktimes;

    // plan state
    bool planned = false;
    int mode = 0;
    char range = 'A';
    int64_t n = 0;
    const void *d = nullptr, *e = nullptr;
    double vl = 0, vu = 0;
    int64_t il = 1, iu = 0;
    int rank = 0, world = 1;
    int64_t m = 0;      // wanted eigenpairs (global)
    int cnt = 0;        // items (index set incl. guards, or all for splits)
    int64_t slice_cap = 0;
    bool split = false;
    int nblocks = 1;
    double scale = 1.0, norm1 = 0.0, pivmin = 0.0, spdiam = 1.0;
    int nodes_used = 0;
    int node_cap = 0;
    int G0 = 1;
    int64_t launches = 0;
    int debug = 0;
    double root_widen = 0.0;  // relative guard widening per row of a root node (R8d), 0 = certified
    mr3_stats stats;
    // ranks of the one-call solvers (mr3_create): communicator or exchange callback
    void *nccl_comm = nullptr;
    int crank = 0, cworld = 1;
    mr3_allgather_fn xfn = nullptr;
    void *xuser = nullptr;
    std::vector<int64_t> colb;  // column partition of the last execute (world + 1 entries)
    cublasHandle_t cublas = nullptr;  // dense pipeline's library GEMMs (created on first use)
    // dense reduction as one CUDA graph (2 kernels per reflector), keyed by its arguments
    cudaGraphExec_t dn_exec = nullptr;
    std::vector<const void *> dn_key;
    cudaEvent_t dn_ev[2] = {nullptr, nullptr};
};

// ------------------------------------------------------------------ NCCL (lazy)
namespace {
struct NcclApi {
    bool tried = false, ok = false;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
};
NcclApi g_nccl;
// the process's libnccl.so.2 if one is loaded already (e.g. PyTorch's), else the system one
bool nccl_load() {
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    g_nccl.GetUniqueId = (decltype(&ncclGetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(&ncclCommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.CommDestroy = (decltype(&ncclCommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.AllGather = (decltype(&ncclAllGather))dlsym(h, "ncclAllGather");
    g_nccl.GetErrorString = (decltype(&ncclGetErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy &&
                g_nccl.AllGather && g_nccl.GetErrorString;
    return g_nccl.ok;
}
}  // namespace

// ------------------------------------------------------------------ cuBLAS (lazy, dense pipeline)
namespace {
struct CublasApi {
    bool tried = false, ok = false;
    decltype(&cublasCreate_v2) Create = nullptr;
    decltype(&cublasDestroy_v2) Destroy = nullptr;
    decltype(&cublasSetStream_v2) SetStream = nullptr;
    decltype(&cublasDgemm_v2) Dgemm = nullptr;
};
CublasApi g_cublas;
bool cublas_load() {
    if (g_cublas.tried) return g_cublas.ok;
    g_cublas.tried = true;
    void *h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcublas.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    g_cublas.Create = (decltype(&cublasCreate_v2))dlsym(h, "cublasCreate_v2");
    g_cublas.Destroy = (decltype(&cublasDestroy_v2))dlsym(h, "cublasDestroy_v2");
    g_cublas.SetStream = (decltype(&cublasSetStream_v2))dlsym(h, "cublasSetStream_v2");
    g_cublas.Dgemm = (decltype(&cublasDgemm_v2))dlsym(h, "cublasDgemm_v2");
    g_cublas.ok = g_cublas.Create && g_cublas.Destroy && g_cublas.SetStream && g_cublas.Dgemm;
    return g_cublas.ok;
}
}  // namespace

// in-place all-gather of world slices of `bytes` bytes (this rank's slice valid on entry)
static int exchange_allgather(mr3_ctx ctx, void *buf, size_t bytes) {
    if (ctx->cworld <= 1 || bytes == 0) return 0;
    if (ctx->xfn) {
        const int r = ctx->xfn(ctx->xuser, buf, bytes, ctx->crank, ctx->cworld, (void *)ctx->stream);
        if (r != 0) {
            ctx->err = "exchange callback returned " + std::to_string(r);
            return MR3_ERR_NCCL;
        }
        return 0;
    }
    if (!ctx->nccl_comm) {
        ctx->err = "world > 1 without an NCCL communicator or an exchange callback";
        return MR3_ERR_NCCL;
    }
    if (!nccl_load()) {
        ctx->err = "libnccl.so.2 not found";
        return MR3_ERR_NCCL;
    }
    char *b = (char *)buf;
    const ncclResult_t r = g_nccl.AllGather(b + (size_t)ctx->crank * bytes, b, bytes, ncclUint8,
                                            (ncclComm_t)ctx->nccl_comm, ctx->stream);
    if (r != ncclSuccess) {
        ctx->err = std::string("ncclAllGather: ") + g_nccl.GetErrorString(r);
        return MR3_ERR_NCCL;
    }
    return 0;
}

// ------------------------------------------------------------------ helpers
#include <chrono>
static double host_now_ms();
static void hsync_note(mr3_ctx ctx, const char *where) {
    if (!(ctx->debug & 2)) return;
    const double t = host_now_ms();
    fprintf(stderr, "[mr3] %s: %.3f ms since last sync point\n", where, t - ctx->t_last);
    ctx->t_last = t;
}

static const double kDefaults[2][MR3_NPARAM] = {
    // GAPTOL XI                     KRS MAXRQI MAXDEPTH SEED      ELG RTOL GROUPS XPHASE REFINE GRID CTA XPTS YCERT NEWTON TWISTW SPLIT FUSE POOL DEBUG FB CHUNK RELAX ABSGAP BT
    {1e-10, 1.1102230246251565e-16, 1.0, 10, 10, 5067315.0, 8.0, -1.0, 0.0, 1.0, 4.0, 1.0, 0.0, 3.0, 0.0, 6.0, 100.0, 1.0, 1.0, 0.0, 0.0, 1.0, 8192.0, 0.5, 0.0, 1.0},
    {1e-5, 5.9604644775390625e-08, 1.0, 10, 10, 5067315.0, 8.0, -1.0, 0.0, 0.0, 4.0, 1.0, 0.0, 3.0, 0.0, 6.0, 100.0, 1.0, 1.0, 0.0, 0.0, 1.0, 8192.0, 0.5, 0.0, 1.0},
};

#define CK(call)                                                                  \
    do {                                                                          \
        cudaError_t _e = (call);                                                  \
        if (_e != cudaSuccess) {                                                  \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(_e);         \
            return _e == cudaErrorMemoryAllocation ? MR3_ERR_NOMEM : MR3_ERR_CUDA; \
        }                                                                         \
    } while (0)

#define CKL(name)                                                                         \
    do {                                                                                  \
        cudaError_t _e = cudaGetLastError();                                              \
        if (_e == cudaSuccess && (ctx->debug & 8)) /* MR3_DEBUG & 8: check every launch */ \
            _e = cudaStreamSynchronize(ctx->stream);                                      \
        if (_e != cudaSuccess) {                                                          \
            ctx->err = std::string("launch ") + name + ": " + cudaGetErrorString(_e);      \
            return MR3_ERR_CUDA;                                                          \
        }                                                                                 \
        ctx->launches++;                                                                  \
    } while (0)

// MR3_DEBUG & 2: wall time between host synchronisation points (finds device idle gaps)
#include <chrono>
static double host_now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
static void hsync_note(mr3_ctx ctx, const char *where);

static void *getbuf(mr3_ctx ctx, const std::string &name, size_t bytes, int *rc) {
    Buf &b = ctx->bufs[name];
    if (bytes == 0) bytes = 16;
    if (b.cap < bytes) {
        if (b.p) {
            cudaStreamSynchronize(ctx->stream);
            cudaFree(b.p);
            b.p = nullptr;
            b.cap = 0;
        }
        size_t want = bytes + bytes / 8;
        if (ctx->debug & 2) fprintf(stderr, "[mr3] cudaMalloc %s %zu\n", name.c_str(), want);
        cudaError_t e = cudaMalloc(&b.p, want);
        if (e != cudaSuccess) {
            e = cudaMalloc(&b.p, bytes);
            want = bytes;
        }
        if (e != cudaSuccess) {
            cudaGetLastError();
            ctx->err = "cudaMalloc(" + name + ", " + std::to_string(bytes) + ") failed";
            *rc = MR3_ERR_NOMEM;
            return nullptr;
        }
        b.cap = want;
    }
    return b.p;
}

static KTime *kt_begin(mr3_ctx ctx, const char *name) {
    if (ctx->kt_used == ctx->kt.size()) {
        KTime t;
        cudaEventCreate(&t.a);
        cudaEventCreate(&t.b);
        ctx->kt.push_back(t);
    }
    KTime *t = &ctx->kt[ctx->kt_used++];
    t->name = name;
    cudaEventRecord(t->a, ctx->stream);
    return t;
}
static void kt_end(mr3_ctx ctx, KTime *t) { cudaEventRecord(t->b, ctx->stream); }

static void kt_collect(mr3_ctx ctx) {
    cudaStreamSynchronize(ctx->stream);
    for (size_t i = 0; i < ctx->kt_used; i++) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->kt[i].a, ctx->kt[i].b);
        if (ctx->debug & 4) {  // device timeline of the timed regions (finds idle gaps)
            float st = 0.f;
            cudaEventElapsedTime(&st, ctx->kt[0].a, ctx->kt[i].a);
            fprintf(stderr, "[mr3] timeline %-14s start %9.3f ms  dur %8.3f ms\n", ctx->kt[i].name,
                    st, ms);
        }
        std::string nm = ctx->kt[i].name;
        bool found = false;
        for (auto &p : ctx->ktimes)
            if (p.first == nm) {
                p.second.first += ms;
                p.second.second += 1;
                found = true;
            }
        if (!found) ctx->ktimes.push_back({nm, {ms, 1}});
    }
    ctx->kt_used = 0;
}

static inline double hi_of(double x) { return x; }
static inline double lo_of(double) { return 0.0; }
static inline double hi_of(const dd &x) { return x.hi; }
static inline double lo_of(const dd &x) { return x.lo; }

template <class R>
struct Work {
    Items it;
    NodeInfo *nodes;
    DevStats *st;
    double *rep_pool;
};

// lanes per eigenvalue of the multisection: enough independent Sturm chains to
// cover the dependent-step latency (about 4 warps per SM; measured sweep), as few as possible
// beyond that (a round of G points buys log2(G+1) bits).  A function of the
// global item count only, so every rank takes the same path (determinism).
static int choose_groups(mr3_ctx ctx, int cnt, int forced) {
    if (forced > 0) {
        int g = 1;
        while (g * 2 <= forced && g < 32) g *= 2;
        return g;
    }
    const long long target = (long long)ctx->nsm * 4 * 32;
    int g = 1;
    while (g < 32 && (long long)cnt * g < target) g *= 2;
    return g;
}

// Threads per CTA of k_bisect_s: tpb_max
// unless MR3_CTA forces 32..128.  (Measured on config 5: 128-thread CTAs beat
// SM-balanced smaller ones -- k_rqi 76 vs 82 (64) vs 87 ms (32) -- the per-CTA
// staging and barrier costs outweigh the 3-vs-2 CTAs-per-SM imbalance.)
static int choose_tpb(mr3_ctx ctx, int64_t thr, int tpb_max) {
    (void)thr;
    const double forced = ctx->cfg[ctx->mode].v[MR3_CTA];
    if (forced > 0) return (int)std::min<double>(tpb_max, std::max(32.0, 32.0 * std::floor(forced / 32)));
    return tpb_max;
}

template <class R>
static int launch_bisect(mr3_ctx ctx, Work<R> &W, const int32_t *list, int cnt, int G, double rtol,
                         double absfloor, int certify, bool xphase, double eps_x,
                         const char *tname = "k_bisect", int ycert = 1, char *tailflag = nullptr,
                         double widen = 0.0, bool relax_ok = true, int iso_init = 0) {
    if (cnt <= 0) return 0;
    int rc = 0;
    // NEXT-1b (R20): relaxed stop of isolated eigenvalues at width c gap sqrt(eps_x sqrt(n) / C)
    // (the kernel multiplies by n^(1/4)); not for the RQI-start refinement and the Newton tail,
    // whose targets are a few ulps
    const double *Pm = ctx->cfg[ctx->mode].v;
    const double eps_xm = ctx->mode ? 5.9604644775390625e-08 : 1.1102230246251565e-16;
    const double Cref = Pm[MR3_REFINE] > 0 ? Pm[MR3_REFINE] : 4.0;
    const double relax_f =
        (relax_ok && certify != 2 && Pm[MR3_RELAX] > 0) ? Pm[MR3_RELAX] * std::sqrt(eps_xm / Cref) : 0.0;
    const double sep = 4.0 * Pm[MR3_GAPTOL];
    const int tpb = choose_tpb(ctx, (int64_t)cnt * G, BS_TPB);
    int xpts = (int)ctx->cfg[ctx->mode].v[MR3_XPTS];
    if (xpts == 3 && (G != 1 || !xphase || certify || ycert)) xpts = 1;  // Newton: G = 1 root x-phase only
    if (xpts != 3) tailflag = nullptr;
    const int maxpass = ctx->cfg[ctx->mode].v[MR3_NEWTON] > 0 ? (int)ctx->cfg[ctx->mode].v[MR3_NEWTON]
                                                               : NEWTON_MAXPASS_DEFAULT;
    const int per = tpb / G;
    // CTA tasks: runs of <= per items of one node; the grid is an upper bound on
    // their number (the kernel reads the exact count), so no host round trip
    const int64_t bound = (cnt + per - 1) / per + std::max(1, ctx->nodes_used);
    RqiTask *dtasks = (RqiTask *)getbuf(ctx, "bis_tasks", (size_t)bound * sizeof(RqiTask), &rc);
    int32_t *dseg = (int32_t *)getbuf(ctx, "bis_seg", (size_t)(cnt + 1) * 4, &rc);
    int *dnt = (int *)getbuf(ctx, "bis_ntasks", 16, &rc);
    if (rc) return rc;
    k_rqi_tasks<<<1, 1024, 0, ctx->stream>>>(list, cnt, W.it.node, dseg, dtasks, dnt, per);
    CKL("k_rqi_tasks");
    const int grid = (int)bound;
    const double pivmin_x = 0x1p-900;
    KTime *t = certify == 2 ? nullptr : kt_begin(ctx, tname);
#define BIS(GG)                                                                               \
    case GG:                                                                                  \
        if (xphase)                                                                           \
            k_bisect_s<R, GG, true><<<grid, tpb, 0, ctx->stream>>>(                           \
                W.nodes, W.it, list, dtasks, dnt, rtol, absfloor, ctx->pivmin, pivmin_x, eps_x, \
                certify, xpts, ycert, tailflag, maxpass, widen, relax_f, sep, iso_init, W.st);    \
        else                                                                                  \
            k_bisect_s<R, GG, false><<<grid, tpb, 0, ctx->stream>>>(                          \
                W.nodes, W.it, list, dtasks, dnt, rtol, absfloor, ctx->pivmin, pivmin_x, eps_x, \
                certify, xpts, ycert, tailflag, maxpass, widen, relax_f, sep, iso_init, W.st);    \
        break;
    switch (G) {
        BIS(1)
        BIS(2)
        BIS(4)
        BIS(8)
        BIS(16)
        BIS(32)
        default:
            return MR3_ERR_STATE;
    }
#undef BIS
    if (t) kt_end(ctx, t);
    CKL("k_bisect");
    return 0;
}

// ------------------------------------------------------------------ plan

template <class R, class T>
static int plan_impl(mr3_ctx ctx, char range, int64_t n, const T *d, const T *e, double vl,
                     double vu, int64_t il, int64_t iu, int rank, int world, int64_t *m,
                     double **brk, int64_t *slice_cap, int64_t *slice_cnt) {
    const int mode = std::is_same<T, float>::value ? 1 : 0;
    const double *P = ctx->cfg[mode].v;
    const double eps_x = mode ? 5.9604644775390625e-08 : 1.1102230246251565e-16;
    const double eps_y = Prec<R>::eps;
    int rc = 0;
    ctx->planned = false;
    memset(&ctx->stats, 0, sizeof(ctx->stats));
    ctx->ktimes.clear();
    ctx->kt_used = 0;
    ctx->launches = 0;
    if (range != 'A' && range != 'I' && range != 'V') return -2;
    if (n < 0) return -3;
    if (range == 'I' && n > 0 && (il < 1 || iu < il - 1 || iu > n)) return -8;
    if (range == 'V' && !(vl < vu)) return -6;
    if (world < 1 || rank < 0 || rank >= world) return -11;
    if (n > 0x7fffffffLL) return -3;
    ctx->mode = mode;
    // MR3_DEBUG bits: 1 = dumps and histograms, 2 = host sync points, 4 = device timeline,
    // 8 = synchronise after every launch
    ctx->debug = (int)P[MR3_DEBUG];
    ctx->dump = (ctx->debug & 1) ? (ctx->debug > 15 ? ctx->debug : 40) : 0;
    ctx->fuse_scale = P[MR3_FUSE_SCALE] != 0.0 ? 1 : 0;
    ctx->range = range;
    ctx->n = n;
    ctx->d = d;
    ctx->e = e;
    ctx->rank = rank;
    ctx->world = world;
    *m = 0;
    *slice_cap = 0;
    *slice_cnt = 0;
    *brk = nullptr;
    if (n == 0 || (range == 'I' && iu < il)) {
        ctx->m = 0;
        ctx->cnt = 0;
        ctx->planned = true;
        return 0;
    }
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    // the previous solve's side-stream work (root PP rows) reads rep_pool and writes nodes[]:
    // it must be complete before this plan rewrites them
    CK(cudaStreamWaitEvent(s, ctx->ev_pp, 0));
    KTime *t_root = kt_begin(ctx, "k_root");

    // K1a: norm, Gershgorin, finiteness
    ScanInfo *dscan = (ScanInfo *)getbuf(ctx, "scan", sizeof(ScanInfo), &rc);
    unsigned long long *dcnt = (unsigned long long *)getbuf(ctx, "cnt64", 64, &rc);
    if (rc) return rc;
    k_scan_input<T><<<1, 1024, 0, s>>>(d, e, n, dscan);
    CKL("k_scan_input");
    ScanInfo info;
    CK(cudaMemcpyAsync(&info, dscan, sizeof(info), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#1");
    if (info.nonfinite) return MR3_ERR_NONFINITE;
    ctx->norm1 = info.norm1;
    int ex = 0;
    if (info.norm1 > 0) frexp(info.norm1, &ex);
    // scaled ||T||_1 in [0.5, 1); the exponent is clamped so that the scale and its inverse are
    // both normal numbers (a subnormal ||T||_1 gave scale = inf, ||T||_1 >= 2^1023 unscale = inf)
    ex = std::min(std::max(ex, -1021), 1022);
    ctx->scale = info.norm1 > 0 ? ldexp(1.0, -ex) : 1.0;
    const double nrm_s = info.norm1 * ctx->scale;
    ctx->pivmin = eps_y * (info.norm1 > 0 ? nrm_s : 1.0);
    ctx->spdiam = fmax((info.gu - info.gl) * ctx->scale, 1e-300);

    // splitting: |e_i| <= eps_x ||T||
    std::vector<BlockDesc> blocks;
    const double thr = eps_x * info.norm1;
    CK(cudaMemsetAsync(dcnt, 0, 8, s));
    if (n > 1) {
        k_split_count<T><<<std::min<int64_t>(1024, (n + 255) / 256), 256, 0, s>>>(e, n, thr, dcnt);
        CKL("k_split_count");
    }
    unsigned long long nsplit = 0;
    CK(cudaMemcpyAsync(&nsplit, dcnt, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#2");
    if (nsplit == 0) {
        blocks.push_back({0, n});
    } else {
        int64_t *dpos = (int64_t *)getbuf(ctx, "splitpos", nsplit * 8, &rc);
        if (rc) return rc;
        CK(cudaMemsetAsync(dcnt, 0, 8, s));
        k_split_list<T><<<std::min<int64_t>(1024, (n + 255) / 256), 256, 0, s>>>(e, n, thr, dpos,
                                                                                 dcnt);
        CKL("k_split_list");
        std::vector<int64_t> pos(nsplit);
        CK(cudaMemcpyAsync(pos.data(), dpos, nsplit * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#3");
        std::sort(pos.begin(), pos.end());
        int64_t r0 = 0;
        for (int64_t p : pos) {
            blocks.push_back({r0, p + 1 - r0});
            r0 = p + 1;
        }
        blocks.push_back({r0, n - r0});
    }
    ctx->nblocks = (int)blocks.size();
    ctx->split = ctx->nblocks > 1;
    ctx->stats.n_blocks = ctx->nblocks;

    // K1b: root representations (chunk-parallel LDL^T + perturbation)
    const int words = Prec<R>::words;
    std::vector<ChunkDesc> chunks;
    std::vector<int> blk_chunk0(blocks.size() + 1);
    for (size_t bi = 0; bi < blocks.size(); bi++) {
        blk_chunk0[bi] = (int)chunks.size();
        for (int64_t r = 0; r < blocks[bi].n; r += RT_CH)
            chunks.push_back({blocks[bi].row0 + r, (int32_t)std::min<int64_t>(RT_CH, blocks[bi].n - r),
                              (int32_t)bi});
    }
    blk_chunk0[blocks.size()] = (int)chunks.size();
    const int nch = (int)chunks.size();
    double *rep_pool = (double *)getbuf(ctx, "rep_root", (size_t)n * 4 * words * 8, &rc);
    double *repx_pool = (double *)getbuf(ctx, "repx_root", (size_t)(n + XPAD) * 16, &rc);
    BlockDesc *dblocks = (BlockDesc *)getbuf(ctx, "blocks", blocks.size() * sizeof(BlockDesc), &rc);
    ChunkDesc *dchunks = (ChunkDesc *)getbuf(ctx, "chunks", chunks.size() * sizeof(ChunkDesc), &rc);
    int *dbc0 = (int *)getbuf(ctx, "blk_chunk0", blk_chunk0.size() * 4, &rc);
    Mat2<R> *dmats = (Mat2<R> *)getbuf(ctx, "root_mats", (size_t)nch * sizeof(Mat2<R>), &rc);
    R *dstates = (R *)getbuf(ctx, "root_states", (size_t)nch * 2 * sizeof(R), &rc);
    double *dmu = (double *)getbuf(ctx, "root_mu", blocks.size() * 8, &rc);
    double *dbrk0 = (double *)getbuf(ctx, "brk_root", blocks.size() * 4 * 8, &rc);
    int *dfail = (int *)getbuf(ctx, "fail", 16, &rc);
    ctx->node_cap = std::max<int>(1024, ctx->nblocks * 2 + 64);
    NodeInfo *dnodes = (NodeInfo *)getbuf(ctx, "nodes", ctx->node_cap * sizeof(NodeInfo), &rc);
    if (rc) return rc;
    CK(cudaMemsetAsync(repx_pool + 2 * n, 0, XPAD * 16, s));  // prefetch padding (negcount_x)
    CK(cudaMemcpyAsync(dblocks, blocks.data(), blocks.size() * sizeof(BlockDesc),
                       cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dchunks, chunks.data(), chunks.size() * sizeof(ChunkDesc),
                       cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dbc0, blk_chunk0.data(), blk_chunk0.size() * 4, cudaMemcpyHostToDevice, s));
    int right = 0;
    if (!ctx->split) {
        if (range == 'I' && (il + iu) > n + 1) right = 1;
        if (range == 'V' && 0.5 * (vl + vu) > 0.5 * (info.gl + info.gu)) right = 1;
    }
    const double xi = P[MR3_XI];
    const uint64_t seed = (uint64_t)P[MR3_SEED];
    double padmul = 1.0;
    for (int attempt = 0; attempt < 12; attempt++, padmul *= 16.0) {
        CK(cudaMemsetAsync(dfail, 0, 4, s));
        k_root_gersh<R, T><<<ctx->nblocks, 256, 0, s>>>(d, e, dblocks, ctx->scale, right, padmul,
                                                         ctx->pivmin, dmu, dbrk0);
        CKL("k_root_gersh");
        k_root_chunkmat<R, T><<<(nch + 127) / 128, 128, 0, s>>>(d, e, dchunks, nch, dblocks,
                                                                 ctx->scale, dmu, dmats);
        CKL("k_root_chunkmat");
        k_root_scan<R><<<ctx->nblocks, RS_TPB, 0, s>>>(dbc0, ctx->nblocks, dmats, dstates);
        CKL("k_root_scan");
        k_root_factor<R, T><<<(nch + 127) / 128, 128, 0, s>>>(d, e, dchunks, nch, dblocks,
                                                               ctx->scale, dmu, dstates, right, xi,
                                                               seed, rep_pool, repx_pool, dfail);
        CKL("k_root_factor");
        int hfail = 0;
        CK(cudaMemcpyAsync(&hfail, dfail, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#4");
        if (!hfail) break;
        if (attempt == 11) {
            ctx->err = "root representation: no definite shift found";
            return MR3_ERR_CUDA;
        }
    }
    k_root_nodes<R><<<(ctx->nblocks + 63) / 64, 64, 0, s>>>(dblocks, ctx->nblocks, dmu, rep_pool,
                                                             repx_pool, dnodes);
    CKL("k_root_nodes");
    {  // prod_{j<k} (-ld_j) per root (product-form eigenvectors, k_zprod.cuh)
        double *pp = (double *)getbuf(ctx, "pp_root", (size_t)n * PP_STRIDE * 8, &rc);
        if (rc) return rc;
        // on the side stream: nothing before the RQI phase reads PP, so it overlaps the grid
        // and bisection (joined in run_rqi)
        CK(cudaEventRecord(ctx->ev_root, s));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_root, 0));
        k_node_pp<R><<<ctx->nblocks, 256, 0, ctx->side>>>(dnodes, 0, pp, 0, 1);
        CKL("k_node_pp");
        CK(cudaEventRecord(ctx->ev_pp, ctx->side));
    }
    ctx->nodes_used = ctx->nblocks;

    // index set
    int64_t ilw = il, iuw = iu;
    if (range == 'A') {
        ilw = 1;
        iuw = n;
    }
    if (!ctx->split && range == 'V') {
        int *dc = (int *)getbuf(ctx, "cnt2", 16, &rc);
        if (rc) return rc;
        k_count_at<R><<<1, 32, 0, s>>>(dnodes, 0, vl * ctx->scale, vu * ctx->scale, ctx->pivmin,
                                       dc);
        CKL("k_count_at");
        int hc[2];
        CK(cudaMemcpyAsync(hc, dc, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#5");
        ilw = hc[0] + 1;
        iuw = hc[1];
    }
    kt_end(ctx, t_root);
    ctx->vl = vl;
    ctx->vu = vu;
    ctx->il = ilw;
    ctx->iu = iuw;
    int cnt;
    if (!ctx->split) {
        if (iuw < ilw) {
            ctx->m = 0;
            ctx->cnt = 0;
            ctx->planned = true;
            return 0;
        }
        int64_t k_lo = std::max<int64_t>(1, ilw - 1), k_hi = std::min<int64_t>(n, iuw + 1);
        cnt = (int)(k_hi - k_lo + 1);
        ctx->m = iuw - ilw + 1;
        ctx->cnt = cnt;
        // allocate items
        Items it;
        it.node = (int32_t *)getbuf(ctx, "it_node", cnt * 4, &rc);
        it.k = (int32_t *)getbuf(ctx, "it_k", cnt * 4, &rc);
        it.col = (int64_t *)getbuf(ctx, "it_col", cnt * 8, &rc);
        it.lo = getbuf(ctx, "it_lo", (size_t)cnt * sizeof(R), &rc);
        it.hi = getbuf(ctx, "it_hi", (size_t)cnt * sizeof(R), &rc);
        it.lgap = (double *)getbuf(ctx, "it_lgap", cnt * 8, &rc);
        it.rgap = (double *)getbuf(ctx, "it_rgap", cnt * 8, &rc);
        it.x0 = (double *)getbuf(ctx, "it_x0", cnt * 8, &rc);
        it.dx = (double *)getbuf(ctx, "it_dx", cnt * 8, &rc);
        it.twist = (int32_t *)getbuf(ctx, "it_twist", cnt * 4, &rc);
        if (rc) return rc;
        k_init_items<R><<<(cnt + 255) / 256, 256, 0, s>>>(it, cnt, (int)k_lo, (int)ilw, (int)iuw, 0,
                                                          dbrk0);
        CKL("k_init_items");
    } else {
        cnt = (int)n;
        ctx->cnt = cnt;
        ctx->m = -1;  // known after the global ordering in execute
        std::vector<int64_t> item0(blocks.size());
        int64_t acc = 0;
        for (size_t b = 0; b < blocks.size(); b++) {
            item0[b] = acc;
            acc += blocks[b].n;
        }
        int64_t *ditem0 = (int64_t *)getbuf(ctx, "item0", item0.size() * 8, &rc);
        Items it;
        it.node = (int32_t *)getbuf(ctx, "it_node", cnt * 4, &rc);
        it.k = (int32_t *)getbuf(ctx, "it_k", cnt * 4, &rc);
        it.col = (int64_t *)getbuf(ctx, "it_col", cnt * 8, &rc);
        it.lo = getbuf(ctx, "it_lo", (size_t)cnt * sizeof(R), &rc);
        it.hi = getbuf(ctx, "it_hi", (size_t)cnt * sizeof(R), &rc);
        it.lgap = (double *)getbuf(ctx, "it_lgap", cnt * 8, &rc);
        it.rgap = (double *)getbuf(ctx, "it_rgap", cnt * 8, &rc);
        it.x0 = (double *)getbuf(ctx, "it_x0", cnt * 8, &rc);
        it.dx = (double *)getbuf(ctx, "it_dx", cnt * 8, &rc);
        it.twist = (int32_t *)getbuf(ctx, "it_twist", cnt * 4, &rc);
        if (rc) return rc;
        CK(cudaMemcpyAsync(ditem0, item0.data(), item0.size() * 8, cudaMemcpyHostToDevice, s));
        k_init_items_blocks<R><<<(cnt + 255) / 256, 256, 0, s>>>(it, cnt, dblocks, ctx->nblocks,
                                                                 ditem0, dbrk0);
        CKL("k_init_items_blocks");
    }

    // K2 on this rank's static slice (Alg. 1 l.3)
    int64_t cap = (cnt + world - 1) / world;
    int64_t first = std::min<int64_t>((int64_t)rank * cap, cnt);
    int64_t mine = std::min<int64_t>(cap, cnt - first);
    ctx->slice_cap = cap;
    double *dbrk = (double *)getbuf(ctx, "brk", (size_t)world * cap * MR3_BRK_REC * 8, &rc);
    int32_t *list = (int32_t *)getbuf(ctx, "list0", (size_t)cnt * 4, &rc);
    DevStats *dst = (DevStats *)getbuf(ctx, "devstats", sizeof(DevStats), &rc);
    if (rc) return rc;
    CK(cudaMemsetAsync(dst, 0, sizeof(DevStats), s));
    Work<R> W;
    W.it.node = (int32_t *)ctx->bufs["it_node"].p;
    W.it.k = (int32_t *)ctx->bufs["it_k"].p;
    W.it.col = (int64_t *)ctx->bufs["it_col"].p;
    W.it.lo = ctx->bufs["it_lo"].p;
    W.it.hi = ctx->bufs["it_hi"].p;
    W.it.lgap = (double *)ctx->bufs["it_lgap"].p;
    W.it.rgap = (double *)ctx->bufs["it_rgap"].p;
    W.it.x0 = (double *)ctx->bufs["it_x0"].p;
    W.it.dx = (double *)ctx->bufs["it_dx"].p;
    W.it.twist = (int32_t *)ctx->bufs["it_twist"].p;
    W.nodes = dnodes;
    W.st = dst;
    double rtol = P[MR3_RTOL] > 0 ? P[MR3_RTOL] : 1e-2 * P[MR3_GAPTOL];
    double absfloor = 4.0 * eps_y * ctx->spdiam;
    if (mine > 0) {
        k_iota<<<(int)((mine + 255) / 256), 256, 0, s>>>(list, (int)mine, (int)first);
        CKL("k_iota");
        ctx->G0 = choose_groups(ctx, cnt, (int)P[MR3_GROUPS]);
        const bool xphase = words == 2 && P[MR3_XPHASE] != 0;
        // the Newton/Laguerre phase (R8e) runs on the binary64 copy of the representation: in
        // dd mode that is the binary_x phase (brackets widened by R8d), in fp32-I/O mode the
        // binary64 counts are the binary_y counts themselves (no widening, no certification).
        // It needs one lane per eigenvalue (G0 = 1: automatic above ~19k items, or forced by
        // MR3_GROUPS = 1).  Measured on the small configs: 4-lane to 8-lane multisection is
        // faster than Newton below that size except on config 3 (profiles/r02_ab_groups.log)
        const int ycert0 = P[MR3_YCERT] != 0 ? 1 : 0;
        const bool newton_ok = (xphase || words == 1) && !ycert0 && P[MR3_XPTS] == 3;
        const bool xkern = xphase || (words == 1 && newton_ok && ctx->G0 == 1);
        const double eps_xw = xphase ? eps_x : 0.0;   // M_x -> M_y widening of the x phase
        const double eps_xt = words == 2 ? eps_x : 1.1102230246251565e-16;  // tail: 2 ulps
        int grid_iso = 0;  // the grid left isolation points in lgap / rgap (NEXT-1b)
        if (!ctx->split && P[MR3_GRID] != 0 && cnt >= 512) {
            // shared top of the bisection tree: a uniform grid of counts, then cells with
            // two or more eigenvalues subdivided level by level (k_grid.cuh)
            GridInfo *gi = (GridInfo *)getbuf(ctx, "grid_info", sizeof(GridInfo), &rc);
            int *c1 = (int *)getbuf(ctx, "grid_c1", GRID_L1 * 4, &rc);
            // points of one level: sum over cells of max(2c + 1, CELL_PMIN), c <= n for the
            // (at most two) cells reaching past the slice, one leader per slice item at most
            const int64_t bound = (2 + CELL_PMIN + 1) * mine + 4 * n + 64;
            int *cp = (int *)getbuf(ctx, "grid_cp", (size_t)bound * 4, &rc);
            CellSet cs;
            cs.lo = (double *)getbuf(ctx, "cell_lo", (size_t)mine * 8, &rc);
            cs.hi = (double *)getbuf(ctx, "cell_hi", (size_t)mine * 8, &rc);
            cs.lo2 = (double *)getbuf(ctx, "cell_lo2", (size_t)mine * 8, &rc);
            cs.hi2 = (double *)getbuf(ctx, "cell_hi2", (size_t)mine * 8, &rc);
            cs.clo = (int *)getbuf(ctx, "cell_clo", (size_t)mine * 4, &rc);
            cs.chi = (int *)getbuf(ctx, "cell_chi", (size_t)mine * 4, &rc);
            cs.clo2 = (int *)getbuf(ctx, "cell_clo2", (size_t)mine * 4, &rc);
            cs.chi2 = (int *)getbuf(ctx, "cell_chi2", (size_t)mine * 4, &rc);
            cs.P = (int *)getbuf(ctx, "cell_P", (size_t)mine * 4, &rc);
            cs.off = (int *)getbuf(ctx, "cell_off", (size_t)mine * 4, &rc);
            cs.lead = (int *)getbuf(ctx, "cell_lead", (size_t)mine * 4, &rc);
            cs.total = (int *)getbuf(ctx, "cell_total", 16, &rc);
            if (rc) return rc;
            size_t tb1 = 0, tb2 = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb1, cs.P, cs.off, (int)mine, s);
            int *lead0 = (int *)getbuf(ctx, "cell_lead0", (size_t)mine * 4, &rc);
            cub::DeviceScan::InclusiveScan(nullptr, tb2, lead0, cs.lead, cub::Max(), (int)mine, s);
            void *ctmp = getbuf(ctx, "cubtmp_cell", std::max(tb1, tb2), &rc);
            if (rc) return rc;
            const int32_t *kslice = W.it.k + first;
            const int ib = (int)((mine + 255) / 256);
            KTime *tg = kt_begin(ctx, "k_grid");
            k_grid_init<<<1, 32, 0, s>>>(gi, dbrk0);
            CKL("k_grid_init");
            if (xphase)
                k_grid_counts<R, true><<<GRID_L1 / BS_TPB, BS_TPB, 0, s>>>(dnodes, 0, 1, gi, c1,
                                                                         ctx->pivmin, 0x1p-900);
            else
                k_grid_counts<R, false><<<GRID_L1 / BS_TPB, BS_TPB, 0, s>>>(dnodes, 0, 1, gi, c1,
                                                                          ctx->pivmin, 0x1p-900);
            CKL("k_grid_counts");
            k_cell_init<<<ib, 256, 0, s>>>(cs, gi, c1, (int)n, kslice, (int)mine);
            CKL("k_cell_init");
            // MR3_GRID = 1: GRID_LEVELS adaptive levels; v >= 2: v - 2 adaptive levels
            const int levels = P[MR3_GRID] >= 2.0 ? (int)P[MR3_GRID] - 2 : GRID_LEVELS;
            ctx->grid_levels = levels;
            for (int lev = 0; lev < levels; lev++) {
                // first adaptive level: 2c + 1 points per cell (about 2 per eigenvalue, one
                // wave of counts); later levels: at least CELL_PMIN (the dense ends)
                k_cell_plan<<<ib, 256, 0, s>>>(cs, lead0, (int)mine, rtol, absfloor,
                                               lev == 0 ? 3 : CELL_PMIN);
                CKL("k_cell_plan");
                size_t t1 = tb1, t2 = tb2;
                cub::DeviceScan::ExclusiveSum(ctmp, t1, cs.P, cs.off, (int)mine, s);
                cub::DeviceScan::InclusiveScan(ctmp, t2, lead0, cs.lead, cub::Max(), (int)mine, s);
                CKL("cell scans");
                k_cell_total<<<1, 32, 0, s>>>(cs, (int)mine);
                CKL("k_cell_total");
                const int g = (int)std::min<int64_t>((bound + BS_TPB - 1) / BS_TPB,
                                                     (int64_t)ctx->nsm * 8);
                if (xphase)
                    k_cell_counts<R, true><<<g, BS_TPB, 0, s>>>(dnodes, cs, (int)mine, cp,
                                                               ctx->pivmin, 0x1p-900);
                else
                    k_cell_counts<R, false><<<g, BS_TPB, 0, s>>>(dnodes, cs, (int)mine, cp,
                                                                ctx->pivmin, 0x1p-900);
                CKL("k_cell_counts");
                k_cell_assign<<<ib, 256, 0, s>>>(cs, (int)mine, kslice, cp);
                CKL("k_cell_assign");
                std::swap(cs.lo, cs.lo2);
                std::swap(cs.hi, cs.hi2);
                std::swap(cs.clo, cs.clo2);
                std::swap(cs.chi, cs.chi2);
            }
            k_cell_final<R><<<ib, 256, 0, s>>>(W.it, (int)first, (int)mine, cs, kslice);
            grid_iso = 1;
            CKL("k_cell_final");
            kt_end(ctx, tg);
        }
        // definite roots: binary_x brackets are enclosed rigorously after widening by the
        // relative-robustness bound (R8d); binary_y certification only if MR3_YCERT
        const int ycert = ycert0;
        ctx->root_widen = (xphase && !ycert) ? 10.0 * eps_x : 0.0;
        char *tail = nullptr;
        const bool newton = newton_ok && ctx->G0 == 1;
        if (newton) {
            tail = (char *)getbuf(ctx, "bis_tailflag", (size_t)mine, &rc);
            if (rc) return rc;
        }
        rc = launch_bisect<R>(ctx, W, list, (int)mine, ctx->G0, rtol, absfloor, 0, xkern, eps_xw,
                              "k_bisect", ycert, tail, 0.0, true, grid_iso);
        if (rc) return rc;
        if (newton) {
            // items whose Newton phase did not finish in NEWTON_MAXPASS passes: multisection
            // with many lanes per item from their current brackets
            int32_t *tl = (int32_t *)getbuf(ctx, "bis_taillist", (size_t)mine * 4, &rc);
            int *tc = (int *)getbuf(ctx, "bis_tailcnt", 16, &rc);
            if (rc) return rc;
            size_t tmpb = 0;
            cub::DeviceSelect::Flagged(nullptr, tmpb, list, tail, tl, tc, (int)mine, s);
            void *tmp = getbuf(ctx, "cubtmp_tail", tmpb, &rc);
            if (rc) return rc;
            cub::DeviceSelect::Flagged(tmp, tmpb, list, tail, tl, tc, (int)mine, s);
            CKL("select (tail)");
            int ht = 0;
            CK(cudaMemcpyAsync(&ht, tc, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#6");
            if (ctx->dump) {
                std::vector<int32_t> ps(mine);
                cudaMemcpy(ps.data(), W.it.twist + first, mine * 4, cudaMemcpyDeviceToHost);
                int hist[64] = {0}, chist[64] = {0};
                for (int64_t i = 0; i < mine; i++) hist[std::min(63, std::max(0, ps[i]))]++;
                for (int64_t b0 = 0; b0 < mine; b0 += 128) {
                    int mx = 0;
                    for (int64_t i = b0; i < std::min<int64_t>(mine, b0 + 128); i++) mx = std::max(mx, ps[i]);
                    chist[std::min(63, mx)]++;
                }
                fprintf(stderr, "[mr3] Newton passes (items):");
                for (int i = 0; i < 64; i++)
                    if (hist[i]) fprintf(stderr, " %d:%d", i, hist[i]);
                fprintf(stderr, "\n[mr3] items with >= 5 passes:");
                for (int64_t i = 0; i < mine; i++)
                    if (ps[i] >= 5) fprintf(stderr, " %lld", (long long)(first + i));
                fprintf(stderr, "\n[mr3] Newton passes (CTA max, 128-item groups):");
                for (int i = 0; i < 64; i++)
                    if (chist[i]) fprintf(stderr, " %d:%d", i, chist[i]);
                fprintf(stderr, "\n");
                fprintf(stderr, "[mr3] Newton tail: %d of %d items:", ht, (int)mine);
                std::vector<int32_t> htl(ht);
                cudaMemcpy(htl.data(), tl, ht * 4, cudaMemcpyDeviceToHost);
                std::vector<int> hclo(mine), hchi(mine);
                if (ctx->bufs.count("cell_clo")) {
                    // final cells: after GRID_LEVELS swaps the current arrays alternate
                    const char *a = (ctx->grid_levels % 2) ? "cell_clo2" : "cell_clo";
                    const char *b = (ctx->grid_levels % 2) ? "cell_chi2" : "cell_chi";
                    cudaMemcpy(hclo.data(), ctx->bufs[a].p, mine * 4, cudaMemcpyDeviceToHost);
                    cudaMemcpy(hchi.data(), ctx->bufs[b].p, mine * 4, cudaMemcpyDeviceToHost);
                }
                for (int i = 0; i < ht; i++)
                    fprintf(stderr, " %d(%d)", htl[i], hchi[htl[i] - first] - hclo[htl[i] - first]);
                fprintf(stderr, "\n");
            }
            if (ht > 0) {
                // to the RQI-start precision (2 ulps) at once: the midpoints are the starts
                // and the refinement pass (K2') has nothing left to do for these items
                // (a fixed lane count: the bits of a bracket must not depend on how many
                // items this rank's slice sent to the tail)
                const int G = 32;
                rc = launch_bisect<R>(ctx, W, tl, ht, G, std::min(rtol, 2.0 * eps_xt), absfloor,
                                      0, true, eps_xw, "k_bisect", 0, nullptr, 0.0, false);
            }
        }
        if (rc) return rc;
        k_items_to_brk<R><<<(int)((mine + 255) / 256), 256, 0, s>>>(W.it, (int)first, (int)mine,
                                                                    dbrk + MR3_BRK_REC * first);
        CKL("k_items_to_brk");
    }
    CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#7");
    *m = ctx->m;
    *brk = dbrk;
    *slice_cap = cap;
    *slice_cnt = mine;
    ctx->planned = true;
    return 0;
}

// ------------------------------------------------------------------ execute

template <class R, class OutT>
static int execute_impl(mr3_ctx ctx, char jobz, OutT *w, OutT *Z, int64_t ldz, int64_t zcap,
                        int64_t *zcol_begin, int64_t *zcol_end, mr3_stats *stats) {
    if (!ctx->planned) return MR3_ERR_STATE;
    const int mode = ctx->mode;
    const double *P = ctx->cfg[mode].v;
    const double eps_x = mode ? 5.9604644775390625e-08 : 1.1102230246251565e-16;
    const double eps_y = Prec<R>::eps;
    int rc = 0;
    cudaStream_t s = ctx->stream;
    *zcol_begin = 0;
    *zcol_end = 0;
    if (jobz != 'V' && jobz != 'N') return -2;
    const int cnt = ctx->cnt;
    if (cnt == 0) {
        ctx->planned = false;
        if (stats) *stats = ctx->stats;
        return 0;
    }
    if (jobz == 'V' && ldz < ctx->n) return -4;
    const int words = Prec<R>::words;
    Work<R> W;
    W.it.node = (int32_t *)ctx->bufs["it_node"].p;
    W.it.k = (int32_t *)ctx->bufs["it_k"].p;
    W.it.col = (int64_t *)ctx->bufs["it_col"].p;
    W.it.lo = ctx->bufs["it_lo"].p;
    W.it.hi = ctx->bufs["it_hi"].p;
    W.it.lgap = (double *)ctx->bufs["it_lgap"].p;
    W.it.rgap = (double *)ctx->bufs["it_rgap"].p;
    W.it.x0 = (double *)ctx->bufs["it_x0"].p;
    W.it.dx = (double *)ctx->bufs["it_dx"].p;
    W.it.twist = (int32_t *)ctx->bufs["it_twist"].p;
    W.nodes = (NodeInfo *)ctx->bufs["nodes"].p;
    W.st = (DevStats *)ctx->bufs["devstats"].p;
    double *dbrk = (double *)ctx->bufs["brk"].p;
    // the root's PP rows (side stream, overlapping the plan's grid and bisection) are joined
    // here: everything below may read or copy nodes[] (node-table growth, RQI)
    CK(cudaStreamWaitEvent(s, ctx->ev_pp, 0));
    // per-execute counters (bisect_rows of the plan is kept)
    CK(cudaMemsetAsync((char *)W.st + offsetof(DevStats, rqi_rows), 0,
                       sizeof(DevStats) - offsetof(DevStats, rqi_rows), s));
    if (ctx->world > 1) {
        k_brk_to_items<R><<<(cnt + 255) / 256, 256, 0, s>>>(W.it, cnt, (int)ctx->slice_cap,
                                                            ctx->world, dbrk);
        CKL("k_brk_to_items");
    }
    double rtol = P[MR3_RTOL] > 0 ? P[MR3_RTOL] : 1e-2 * P[MR3_GAPTOL];
    double absfloor = 4.0 * eps_y * ctx->spdiam;
    const double gaptol = P[MR3_GAPTOL];

    // split case: global order of all block eigenvalues -> output columns
    if (ctx->split) {
        unsigned long long *keys = (unsigned long long *)getbuf(ctx, "keys", cnt * 8, &rc);
        unsigned long long *keys2 = (unsigned long long *)getbuf(ctx, "keys2", cnt * 8, &rc);
        int32_t *vals = (int32_t *)getbuf(ctx, "vals", cnt * 4, &rc);
        int32_t *vals2 = (int32_t *)getbuf(ctx, "vals2", cnt * 4, &rc);
        int64_t *mc = (int64_t *)getbuf(ctx, "mcount", 16, &rc);
        if (rc) return rc;
        k_item_keys<R><<<(cnt + 255) / 256, 256, 0, s>>>(W.it, cnt, W.nodes, keys, vals);
        CKL("k_item_keys");
        size_t tmpb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmpb, keys, keys2, vals, vals2, cnt, 0, 64, s);
        void *tmp = getbuf(ctx, "cubtmp", tmpb, &rc);
        if (rc) return rc;
        cub::DeviceRadixSort::SortPairs(tmp, tmpb, keys, keys2, vals, vals2, cnt, 0, 64, s);
        CKL("radix sort");
        int64_t init[2] = {0, 0x7fffffffffffffffLL};
        CK(cudaMemcpyAsync(mc, init, 16, cudaMemcpyHostToDevice, s));
        int md = ctx->range == 'A' ? 0 : (ctx->range == 'I' ? 1 : 2);
        k_assign_cols<<<(cnt + 255) / 256, 256, 0, s>>>(W.it, cnt, vals2, keys2, md, ctx->il,
                                                        ctx->iu, ctx->vl * ctx->scale,
                                                        ctx->vu * ctx->scale, mc);
        CKL("k_assign_cols");
        int64_t hm = 0;
        CK(cudaMemcpyAsync(&hm, mc, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#8");
        ctx->m = hm;
        int64_t first_rank = md == 1 ? ctx->il : 1;
        if (md == 2) {
            // first wanted rank = 1 + #items at or below vl: ranks are contiguous
            std::vector<int64_t> cols(cnt);
            CK(cudaMemcpyAsync(cols.data(), W.it.col, cnt * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#9");
            int64_t mn = INT64_MAX;
            for (auto c : cols)
                if (c >= 0) mn = std::min(mn, c);
            first_rank = mn == INT64_MAX ? 1 : mn;
        }
        k_compact_cols<<<(cnt + 255) / 256, 256, 0, s>>>(W.it, cnt, vals2, first_rank);
        CKL("k_compact_cols");
    }
    const int64_t m = ctx->m;
    if (m <= 0) {
        ctx->planned = false;
        if (stats) *stats = ctx->stats;
        return 0;
    }

    // level-0 classification of the whole index set (identical on every rank)
    int32_t *listA = (int32_t *)getbuf(ctx, "listA", (size_t)cnt * 4, &rc);
    int32_t *listB = (int32_t *)getbuf(ctx, "listB", (size_t)cnt * 4, &rc);
    int32_t *singles = (int32_t *)getbuf(ctx, "singles", (size_t)cnt * 4, &rc);
    int32_t *cbeg = (int32_t *)getbuf(ctx, "cbeg", (size_t)cnt * 4, &rc);
    int32_t *cend = (int32_t *)getbuf(ctx, "cend", (size_t)cnt * 4, &rc);
    int32_t *segb = (int32_t *)getbuf(ctx, "segb", (size_t)(cnt + 1) * 4, &rc);
    int32_t *segw = (int32_t *)getbuf(ctx, "segw", (size_t)cnt * 4, &rc);
    int32_t *dcounts = (int32_t *)getbuf(ctx, "counts", 16, &rc);
    if (rc) return rc;
    k_iota<<<(cnt + 255) / 256, 256, 0, s>>>(listA, cnt, 0);
    CKL("k_iota");
    SegOut so;
    so.singles = singles;
    so.clus_beg = cbeg;
    so.clus_end = cend;
    so.next_active = listB;
    so.seg_begin = segb;
    so.seg_want = segw;
    so.counts = dcounts;
    so.st = W.st;
    KTime *tc = kt_begin(ctx, "k_classify");
    k_classify<R><<<1, 1024, 0, s>>>(W.it, listA, cnt, gaptol, so,
                                                   P[MR3_ABSGAP] * ctx->norm1 * ctx->scale);
    kt_end(ctx, tc);
    CKL("k_classify");
    int hc[4];
    CK(cudaMemcpyAsync(hc, dcounts, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#10");
    int nsing = hc[0], nclus = hc[1], nmem = hc[2];
    if (ctx->dump) fprintf(stderr, "[mr3] level 0: %d singles %d clusters %d members\n", nsing, nclus, nmem);

    // multi-rank: cluster-whole partition of the output columns
    int64_t c0 = 0, c1 = m;
    if (ctx->world > 1) {
        std::vector<int32_t> hs(nsing), hb(nclus), he(nclus), hm(nmem);
        std::vector<int64_t> cols(cnt);
        if (nsing) CK(cudaMemcpyAsync(hs.data(), singles, nsing * 4, cudaMemcpyDeviceToHost, s));
        if (nclus) {
            CK(cudaMemcpyAsync(hb.data(), cbeg, nclus * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(he.data(), cend, nclus * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(hm.data(), listB, nmem * 4, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaMemcpyAsync(cols.data(), W.it.col, cnt * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#11");
        // segments: (first column, cost, kind, index)
        struct Seg {
            int64_t c0;
            double cost;
            int kind, idx;
        };
        std::vector<Seg> segs;
        for (int i = 0; i < nsing; i++) segs.push_back({cols[hs[i]], 1.0, 0, i});
        for (int i = 0; i < nclus; i++) {
            int64_t cmin = INT64_MAX;
            int wanted = 0;
            for (int j = hb[i]; j < he[i]; j++)
                if (cols[hm[j]] >= 0) {
                    cmin = std::min(cmin, cols[hm[j]]);
                    wanted++;
                }
            segs.push_back({cmin, 3.0 * wanted, 1, i});
        }
        std::sort(segs.begin(), segs.end(), [](const Seg &a, const Seg &b) { return a.c0 < b.c0; });
        std::vector<int64_t> sb(segs.size() + 1);
        std::vector<double> cost(segs.size());
        for (size_t i = 0; i < segs.size(); i++) {
            sb[i] = segs[i].c0;
            cost[i] = segs[i].cost;
        }
        sb[segs.size()] = m;
        std::vector<int64_t> cb(ctx->world + 1);
        mr3_partition_columns((int64_t)segs.size(), sb.data(), cost.data(), ctx->world, cb.data());
        c0 = cb[ctx->rank];
        c1 = cb[ctx->rank + 1];
        ctx->colb = cb;
        // keep this rank's singletons and clusters
        std::vector<int32_t> ns, nb, ne, nm;
        for (auto &sg : segs) {
            if (sg.c0 < c0 || sg.c0 >= c1) continue;
            if (sg.kind == 0) {
                ns.push_back(hs[sg.idx]);
            } else {
                int b0 = (int)nm.size();
                for (int j = hb[sg.idx]; j < he[sg.idx]; j++) nm.push_back(hm[j]);
                nb.push_back(b0);
                ne.push_back((int)nm.size());
            }
        }
        // clusters must stay in item order for the child pool layout: they are
        nsing = (int)ns.size();
        nclus = (int)nb.size();
        nmem = (int)nm.size();
        if (nsing) CK(cudaMemcpyAsync(singles, ns.data(), nsing * 4, cudaMemcpyHostToDevice, s));
        if (nclus) {
            CK(cudaMemcpyAsync(cbeg, nb.data(), nclus * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(cend, ne.data(), nclus * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(listB, nm.data(), nmem * 4, cudaMemcpyHostToDevice, s));
        }
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#12");
    }
    if (ctx->world <= 1) ctx->colb = {0, m};
    *zcol_begin = c0;
    *zcol_end = c1;
    bool zfail = jobz == 'V' && zcap < c1 - c0;
    if (ctx->cworld > 1 && ctx->world > 1) {
        // one-call multi-rank solve: the ranks agree on MR3_ERR_ZCAP before any of them starts
        // the RQI phase (a rank that returned alone would leave the others waiting in the
        // eigenvalue all-gather)
        int32_t *zf = (int32_t *)getbuf(ctx, "zcap_flags", (size_t)ctx->cworld * 4, &rc);
        if (rc) return rc;
        std::vector<int32_t> hf(ctx->cworld, 0);
        hf[ctx->crank] = zfail ? 1 : 0;
        CK(cudaMemcpyAsync(zf + ctx->crank, &hf[ctx->crank], 4, cudaMemcpyHostToDevice, s));
        if ((rc = exchange_allgather(ctx, zf, 4))) return rc;
        CK(cudaMemcpyAsync(hf.data(), zf, (size_t)ctx->cworld * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int r = 0; r < ctx->cworld; r++) zfail = zfail || hf[r] != 0;
    }
    if (zfail) return MR3_ERR_ZCAP;
    if (jobz == 'V' && ctx->split && c1 > c0) {
        CK(cudaMemset2DAsync(Z, ldz * sizeof(OutT), 0, ctx->n * sizeof(OutT), c1 - c0, s));
    }

    // RQI scratch sizing: checkpoints of (s, W, p) every RQ_C rows per eigenpair
    // (cudaMemGetInfo once per context: the call can stall the host for tens of ms
    // while the device works; a failed allocation below halves the chunk instead)
    if (ctx->mem_free == 0) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        ctx->mem_free = std::max<size_t>(fr, 1);
    }
    const size_t freeb = ctx->mem_free;
    const int64_t nmaxb = ctx->n;
    const int64_t nblk = (nmaxb + RQ_C - 1) / RQ_C;
    size_t budget = std::min<size_t>((size_t)(freeb * 0.6), (size_t)48 << 30);
    int64_t per_thread = nblk * (2 * (int64_t)sizeof(R) + 8);
    int64_t Smax = std::max<int64_t>(RQ_TPB, (int64_t)(budget / std::max<int64_t>(per_thread, 1)));
    Smax = (Smax / RQ_TPB) * RQ_TPB;
    ZCol *dzc = nullptr;  // per local column: factors for k_zscale (written by k_rqi)
    if (jobz == 'V' && c1 > c0) {
        dzc = (ZCol *)getbuf(ctx, "zcol_info", (size_t)(c1 - c0) * sizeof(ZCol), &rc);
        if (rc) return rc;
        CK(cudaMemsetAsync(dzc, 0, (size_t)(c1 - c0) * sizeof(ZCol), s));
    }

    auto run_rqi = [&](const int32_t *list, int ncount) -> int {
        if (ncount <= 0) return 0;
        int rc2 = 0;
        if (P[MR3_REFINE] > 0) {  // K2': binary_x starting points for small-gap singletons
            char *flags = (char *)getbuf(ctx, "ref_flags", (size_t)ncount, &rc2);
            int32_t *rlist = (int32_t *)getbuf(ctx, "ref_list", (size_t)ncount * 4, &rc2);
            int *rcnt = (int *)getbuf(ctx, "ref_cnt", 16, &rc2);
            if (rc2) return rc2;
            KTime *tr = kt_begin(ctx, "k_refine_x0");
            k_refine_flags<R><<<(ncount + 255) / 256, 256, 0, s>>>(W.nodes, W.it, list, ncount,
                                                                  eps_x, P[MR3_REFINE], flags);
            CKL("k_refine_flags");
            size_t tmpb = 0;
            cub::DeviceSelect::Flagged(nullptr, tmpb, list, flags, rlist, rcnt, ncount, s);
            void *tmp = getbuf(ctx, "cubtmp_ref", tmpb, &rc2);
            if (rc2) return rc2;
            cub::DeviceSelect::Flagged(tmp, tmpb, list, flags, rlist, rcnt, ncount, s);
            CKL("select (refine)");
            int hr = 0;
            CK(cudaMemcpyAsync(&hr, rcnt, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#13");
            if (ctx->dump) fprintf(stderr, "[mr3] refine: %d of %d singletons\n", hr, ncount);
            if (hr > 0) {
                // many lanes per item: few items, short dependent chains (log2(G+1) bits/round)
                // (fixed lane count: independent of the rank-local number of items)
                const int G = 32;
                rc2 = launch_bisect<R>(ctx, W, rlist, hr, G, 2.0 * eps_x, 1e-300, 2, true, eps_x,
                                       "k_refine_x0", 1, nullptr, ctx->root_widen);
                if (rc2) return rc2;
                if (ctx->dump) {
                    cudaStreamSynchronize(s);
                    std::vector<int32_t> hl(hr);
                    cudaMemcpy(hl.data(), rlist, hr * 4, cudaMemcpyDeviceToHost);
                    int mid = 0;
                    for (int i = 0; i < hr; i++) mid = std::max(mid, hl[i]);
                    std::vector<double> hx(mid + 1), hd(mid + 1), hg(mid + 1);
                    cudaMemcpy(hx.data(), W.it.x0, hx.size() * 8, cudaMemcpyDeviceToHost);
                    cudaMemcpy(hd.data(), W.it.dx, hd.size() * 8, cudaMemcpyDeviceToHost);
                    cudaMemcpy(hg.data(), W.it.lgap, hg.size() * 8, cudaMemcpyDeviceToHost);
                    int nn = 0, ninf = 0;
                    for (int i = 0; i < hr; i++) {
                        nn += std::isnan(hx[hl[i]]) ? 1 : 0;
                        ninf += std::isinf(hd[hl[i]]) ? 1 : 0;
                    }
                    fprintf(stderr, "[mr3] refine: %d NaN x0 of %d, %d without a Newton step; dx/lgap:", nn, hr, ninf);
                    for (int i = 0; i < hr; i += std::max(1, hr / 40))
                        fprintf(stderr, " %d:%.2g/%.2g", hl[i], hd[hl[i]], hg[hl[i]]);
                    fprintf(stderr, "\n[mr3] ids:");
                    for (int i = 0; i < hr; i++)
                        if (hl[i] >= 49500) fprintf(stderr, " %d%s", hl[i], std::isnan(hx[hl[i]]) ? "n" : "");
                    fprintf(stderr, "\n");
                }
            }
            kt_end(ctx, tr);
        } else {
            CK(cudaMemsetAsync(W.it.x0, 0xff, (size_t)cnt * 8, s));  // NaN: midpoints
        }
        // CTA tasks: runs of <= rtpb singletons of one node (smem staging)
        const int rtpb = RQ_TPB;  // k_rqi* are written for full 128-thread CTAs
        RqiTask *dtasks = (RqiTask *)getbuf(ctx, "rqi_tasks", (size_t)(ncount + 1) * sizeof(RqiTask),
                                            &rc2);
        int32_t *dseg = (int32_t *)getbuf(ctx, "rqi_seg", (size_t)(ncount + 1) * 4, &rc2);
        int *dnt = (int *)getbuf(ctx, "rqi_ntasks", 16, &rc2);
        unsigned long long *tkeys =
            (unsigned long long *)getbuf(ctx, "rqi_keys", (size_t)ncount * 8 * 2, &rc2);
        int32_t *tvals = (int32_t *)getbuf(ctx, "rqi_vals", (size_t)ncount * 4, &rc2);
        int32_t *slist = (int32_t *)getbuf(ctx, "rqi_sorted", (size_t)ncount * 4, &rc2);
        if (rc2) return rc2;
        // few eigenpairs (fewer than ~16 per SM): one per CTA, every RQI iteration a split
        // pass of all 128 threads (R9d) -- the serial n-row chains would leave the GPU idle
        const bool split_all = P[MR3_SPLIT] >= 2 && ncount <= ctx->nsm * 16;
        bool rqi_split_all = false;  // (set for the k_rqi launch, read by launch_chunks)
        const RqiResume<R> *rqi_resume_in = nullptr;  // (k_rqi continuing after k_rqi_fb)
        const char *rqi_tname = "k_rqi";
        bool rqi_nosplit = false;  // (serial passes only: the eigenpairs k_rqi_chunk could not split)
        int rqi_iter0 = 0;
        auto make_tasks = [&](const int32_t *lst, int *nt, int per, int count) -> int {
            k_rqi_tasks<<<1, 1024, 0, s>>>(lst, count, W.it.node, dseg, dtasks, dnt, per);
            cudaError_t e2 = cudaGetLastError();
            if (e2 != cudaSuccess) {
                ctx->err = std::string("k_rqi_tasks: ") + cudaGetErrorString(e2);
                return MR3_ERR_CUDA;
            }
            ctx->launches++;
            if (cudaMemcpyAsync(nt, dnt, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess) {
                ctx->err = "k_rqi_tasks: copy";
                return MR3_ERR_CUDA;
            }
            return 0;
        };
        int64_t tmax = std::max<int64_t>(1, Smax / rtpb);
        auto launch_chunks = [&](bool locate, const int32_t *lst, int ntasks) -> int {
            for (int off = 0; off < ntasks;) {
                const int nb = (int)std::min<int64_t>(tmax, ntasks - off);
                const int64_t S = (int64_t)nb * rtpb;
                int rc3 = 0;
                char *ck =
                    (char *)getbuf(ctx, "rqi_ck", (size_t)nblk * S * (2 * sizeof(R) + 8), &rc3);
                if (rc3 == MR3_ERR_NOMEM && tmax > 1) {  // memory got tighter: smaller chunks
                    tmax = std::max<int64_t>(1, tmax / 2);
                    ctx->mem_free = 0;
                    continue;
                }
                if (rc3) return rc3;
                RqiArgs<R> A;
                A.nodes = W.nodes;
                A.it = W.it;
                A.list = lst;
                A.tasks = dtasks + off;
                A.ck_s = (R *)ck;
                A.ck_p = (R *)(ck + nblk * S * sizeof(R));
                A.ck_W = (double *)(ck + 2 * nblk * S * sizeof(R));
                A.zc = dzc;
                A.S = S;
                A.pivmin = ctx->pivmin;
                A.krs = P[MR3_KRS];
                A.eps_x = eps_x;
                A.gaptol = gaptol;
                A.root_widen = ctx->root_widen;
                A.twist_w = P[MR3_TWISTW];
                A.split = (P[MR3_SPLIT] != 0 && !rqi_nosplit) ? (rqi_split_all && !locate ? 2 : 1) : 0;
                A.fuse_scale = ctx->fuse_scale;
                A.maxit = (int)P[MR3_MAX_RQI];
                A.jobz_v = jobz == 'V';
                A.w = w;
                A.Z = Z;
                A.ldz = ldz;
                A.zcol0 = c0;
                A.unscale = 1.0 / ctx->scale;
                A.st = W.st;
                A.dbg_iters = nullptr;
                A.dbg_trace = nullptr;
                A.dbg_clk = nullptr;
                A.left = nullptr;
                A.resume = nullptr;
                A.resume_in = locate ? nullptr : rqi_resume_in;
                A.iter0 = locate ? 0 : rqi_iter0;
                if (ctx->dump && !locate) {
                    A.dbg_clk = (unsigned long long *)getbuf(ctx, "dbg_clk", (size_t)nb * 32, &rc3);
                    cudaMemsetAsync(A.dbg_clk, 0, (size_t)nb * 32, s);
                }
                if (ctx->dump) {
                    A.dbg_iters = (int32_t *)getbuf(ctx, "dbg_iters", (size_t)cnt * 4, &rc3);
                    A.dbg_trace = (double *)getbuf(ctx, "dbg_trace", (size_t)cnt * 64, &rc3);
                }
                KTime *t = kt_begin(ctx, locate ? "k_rqi_locate" : rqi_tname);
                if (locate)
                    k_rqi_locate<R><<<nb, rtpb, 0, s>>>(A);
                else
                {
                    constexpr size_t smem = rqi_smem_bytes<R, OutT>();
                    static bool attr_set = false;  // per instantiation, once per process
                    if (!attr_set) {
                        cudaFuncSetAttribute(k_rqi<R, OutT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                        attr_set = true;
                    }
                    k_rqi<R, OutT><<<nb, rtpb, smem, s>>>(A);
                }
                kt_end(ctx, t);
                if (A.dbg_clk) {  // per-CTA durations against the CTA's sweep length
                    std::vector<unsigned long long> hc((size_t)nb * 4);
                    cudaMemcpyAsync(hc.data(), A.dbg_clk, (size_t)nb * 32, cudaMemcpyDeviceToHost, s);
                    cudaStreamSynchronize(s);
                    unsigned long long t0 = ~0ull, t1 = 0;
                    for (int b = 0; b < nb; b++) {
                        t0 = std::min(t0, hc[4 * b]);
                        t1 = std::max(t1, hc[4 * b + 1]);
                    }
                    std::map<unsigned long long, int> per_sm;
                    for (int b = 0; b < nb; b++) per_sm[hc[4 * b + 2] & 0xff]++;
                    {  // the slowest CTAs
                        std::vector<std::pair<double, int>> dv;
                        for (int b = 0; b < nb; b++)
                            dv.push_back({1e-6 * (double)(hc[4 * b + 1] - hc[4 * b]), b});
                        std::sort(dv.rbegin(), dv.rend());
                        for (int q = 0; q < std::min(nb, 12); q++) {
                            const int b = dv[q].second;
                            const unsigned long long w2 = hc[4 * b + 2], w3 = hc[4 * b + 3];
                            fprintf(stderr, "[mr3]   slow CTA %d: %.2f ms sm %llu (%d CTAs) twist %llu..%llu iters %llu first item %llu\n",
                                    b, dv[q].first, w2 & 0xff, per_sm[w2 & 0xff], (w2 >> 8) & 0xffffff,
                                    (w2 >> 32) & 0xffffff, w3 & 0xff, w3 >> 8);
                        }
                    }
                    // duration histogram (2 ms bins) split by CTAs on the SM and max iterations
                    std::map<std::pair<int, int>, std::vector<double>> grp;
                    double busy = 0;
                    for (int b = 0; b < nb; b++) {
                        const double dur = 1e-6 * (double)(hc[4 * b + 1] - hc[4 * b]);
                        grp[{per_sm[hc[4 * b + 2] & 0xff], (int)(hc[4 * b + 3] & 0xff)}].push_back(dur);
                        busy += dur;
                    }
                    fprintf(stderr, "[mr3] k_rqi CTAs %d on %zu SMs span %.3f ms mean %.3f ms\n", nb,
                            per_sm.size(), 1e-6 * (double)(t1 - t0), busy / std::max(nb, 1));
                    for (auto &g : grp) {
                        auto v = g.second;
                        std::sort(v.begin(), v.end());
                        fprintf(stderr, "[mr3]   %d CTAs/SM, iters %d: %zu CTAs, min %.2f med %.2f max %.2f ms\n",
                                g.first.first, g.first.second, v.size(), v.front(), v[v.size() / 2],
                                v.back());
                    }
                }
                cudaError_t e2 = cudaGetLastError();
                if (e2 != cudaSuccess) {
                    ctx->err = std::string(locate ? "k_rqi_locate: " : "k_rqi: ") +
                               cudaGetErrorString(e2);
                    return MR3_ERR_CUDA;
                }
                ctx->launches++;
                off += nb;
            }
            return 0;
        };
        // K5a: twist indices in binary_x, then group the singletons by (node, r) so
        // that the CTAs of the fixed-twist iterations sweep nearly equal row ranges
        int ntasks = 0;
        if ((rc2 = make_tasks(list, &ntasks, rtpb, ncount))) return rc2;
        if ((rc2 = launch_chunks(true, list, ntasks))) return rc2;
        if (ctx->dump) {  // located twists of the first and last singletons
            std::vector<int32_t> hl(ncount), ht(cnt);
            cudaMemcpy(hl.data(), list, (size_t)ncount * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(ht.data(), W.it.twist, (size_t)cnt * 4, cudaMemcpyDeviceToHost);
            fprintf(stderr, "[mr3] twists (item:r):");
            for (int i = 0; i < ncount; i++)
                if (i < 6 || i >= ncount - 6) fprintf(stderr, " %d:%d", hl[i], ht[hl[i]]);
            fprintf(stderr, "\n");
        }
        k_twist_keys<<<(ncount + 255) / 256, 256, 0, s>>>(list, ncount, W.it.node, W.it.twist,
                                                          tkeys, tvals);
        CKL("k_twist_keys");
        {
            size_t tmpb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmpb, tkeys, tkeys + ncount, tvals, slist,
                                            ncount, 0, 64, s);
            void *tmp = getbuf(ctx, "cubtmp_rqi", tmpb, &rc2);
            if (rc2) return rc2;
            cub::DeviceRadixSort::SortPairs(tmp, tmpb, tkeys, tkeys + ncount, tvals, slist,
                                            ncount, 0, 64, s);
            CKL("radix sort (twist)");
        }
        if (split_all || P[MR3_RQI_FB] == 0) {  // every iteration in k_rqi
            if ((rc2 = make_tasks(slist, &ntasks, split_all ? 1 : rtpb, ncount))) return rc2;
            rqi_split_all = split_all;
            return launch_chunks(false, slist, ntasks);
        }
        // small index sets: every iteration chunk-parallel, one eigenpair per CTA (k_rqi_chunk)
        // (decided by the global number of wanted eigenpairs, not this rank's or this level's
        // singletons: the path, hence every bit, must not depend on the world size)
        const bool small = P[MR3_RQI_CHUNK] > 0 && ctx->m <= (int64_t)P[MR3_RQI_CHUNK];
        char *leftc = (char *)getbuf(ctx, "rqi_leftc", (size_t)ncount, &rc2);
        int32_t *llc = (int32_t *)getbuf(ctx, "rqi_llc", (size_t)ncount * 4, &rc2);
        RqiResume<R> *resume0 =
            (RqiResume<R> *)getbuf(ctx, "rqi_resume", (size_t)cnt * sizeof(RqiResume<R>), &rc2);
        if (rc2) return rc2;
        auto rqi_args = [&](const int32_t *lst, char *lf, const RqiResume<R> *rin) {
            RqiArgs<R> A;
            memset(&A, 0, sizeof(A));
            A.nodes = W.nodes;
            A.it = W.it;
            A.list = lst;
            A.zc = dzc;
            A.pivmin = ctx->pivmin;
            A.krs = P[MR3_KRS];
            A.eps_x = eps_x;
            A.gaptol = gaptol;
            A.root_widen = ctx->root_widen;
            A.twist_w = P[MR3_TWISTW];
            A.fuse_scale = ctx->fuse_scale;
            A.maxit = (int)P[MR3_MAX_RQI];
            A.jobz_v = jobz == 'V';
            A.w = w;
            A.Z = Z;
            A.ldz = ldz;
            A.zcol0 = c0;
            A.unscale = 1.0 / ctx->scale;
            A.st = W.st;
            A.left = lf;
            A.resume = resume0;
            A.resume_in = rin;
            return A;
        };
        // k_rqi_chunk over `lst` (count cntl), then the eigenpairs it leaves continue serially
        // in k_rqi from their state (bisection fallback after max_rqi)
        auto run_chunked = [&](const int32_t *lst, int cntl, const RqiResume<R> *rin) -> int {
            if (cntl <= 0) return 0;
            RqiArgs<R> A = rqi_args(lst, leftc, rin);
            if (ctx->dump) {
                A.dbg_trace = (double *)getbuf(ctx, "dbg_trace", (size_t)cnt * 64, &rc2);
                if (rc2) return rc2;
                CK(cudaMemsetAsync(A.dbg_trace, 0, (size_t)cnt * 64, s));
            }
            const int tpb = ctx->n >= 4096 ? 128 : (ctx->n >= 2048 ? 64 : 32);
            KTime *t = kt_begin(ctx, rin ? "k_rqi_tail" : "k_rqi");
            k_rqi_chunk<R, OutT><<<cntl, tpb, 0, s>>>(A);
            kt_end(ctx, t);
            CKL("k_rqi_chunk");
            int *lcnt2 = (int *)getbuf(ctx, "rqi_lcnt2", 16, &rc2);
            if (rc2) return rc2;
            size_t tmpl = 0;
            cub::DeviceSelect::Flagged(nullptr, tmpl, lst, leftc, llc, lcnt2, cntl, s);
            void *tmp = getbuf(ctx, "cubtmp_leftc", tmpl, &rc2);
            if (rc2) return rc2;
            cub::DeviceSelect::Flagged(tmp, tmpl, lst, leftc, llc, lcnt2, cntl, s);
            CKL("select (chunk left)");
            int hl = 0;
            CK(cudaMemcpyAsync(&hl, lcnt2, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#13c");
            if (ctx->dump) {
                fprintf(stderr, "[mr3] k_rqi_chunk left %d of %d eigenpairs\n", hl, cntl);
                std::vector<int32_t> hll(hl);
                std::vector<double> tr((size_t)cnt * 8);
                cudaMemcpy(hll.data(), llc, (size_t)hl * 4, cudaMemcpyDeviceToHost);
                cudaMemcpy(tr.data(), A.dbg_trace, (size_t)cnt * 64, cudaMemcpyDeviceToHost);
                for (int i = 0; i < hl && i < 24; i++) {
                    const double *t = &tr[8 * (size_t)hll[i]];
                    fprintf(stderr, "[mr3]   item %d: log2 rel %.1f jr/tol %.3g iter %g r %g n %g bad %g\n",
                            hll[i], t[0], t[1], t[2], t[3], t[4], t[5]);
                }
            }
            if (hl == 0) return 0;
            if ((rc2 = make_tasks(llc, &ntasks, rtpb, hl))) return rc2;
            rqi_resume_in = resume0;
            rqi_iter0 = 0;
            rqi_tname = "k_rqi_serial";
            rqi_nosplit = true;
            rc2 = launch_chunks(false, llc, ntasks);
            rqi_nosplit = false;
            rqi_tname = "k_rqi";
            rqi_resume_in = nullptr;
            return rc2;
        };
        if (small) return run_chunked(slist, ncount, nullptr);
        // K5 main phase: iterations 1-2 with the F and B halves in two threads (k_rqi_fb);
        // the eigenpairs it leaves continue in k_rqi from their saved state
        char *left = (char *)getbuf(ctx, "rqi_left", (size_t)ncount, &rc2);
        int32_t *llist = (int32_t *)getbuf(ctx, "rqi_llist", (size_t)ncount * 4, &rc2);
        int *lcnt = (int *)getbuf(ctx, "rqi_lcnt", 16, &rc2);
        RqiResume<R> *resume =
            (RqiResume<R> *)getbuf(ctx, "rqi_resume", (size_t)cnt * sizeof(RqiResume<R>), &rc2);
        if (rc2) return rc2;
        if ((rc2 = make_tasks(slist, &ntasks, FB_NP, ncount))) return rc2;
        {
            RqiArgs<R> A;
            memset(&A, 0, sizeof(A));
            A.nodes = W.nodes;
            A.it = W.it;
            A.list = slist;
            A.tasks = dtasks;
            A.zc = dzc;
            A.pivmin = ctx->pivmin;
            A.krs = P[MR3_KRS];
            A.eps_x = eps_x;
            A.gaptol = gaptol;
            A.root_widen = ctx->root_widen;
            A.twist_w = P[MR3_TWISTW];
            A.fuse_scale = ctx->fuse_scale;
            A.maxit = (int)P[MR3_MAX_RQI];
            A.jobz_v = jobz == 'V';
            A.w = w;
            A.Z = Z;
            A.ldz = ldz;
            A.zcol0 = c0;
            A.unscale = 1.0 / ctx->scale;
            A.st = W.st;
            A.left = left;
            A.resume = resume;
            if (ctx->dump) A.dbg_iters = (int32_t *)getbuf(ctx, "dbg_iters", (size_t)cnt * 4, &rc2);
            constexpr size_t smem = fb_smem_bytes<R, OutT>();
            static bool attr_fb = false;  // per instantiation, once per process
            if (!attr_fb) {
                for (auto fk : {k_rqi_fb<R, OutT, false>, k_rqi_fb<R, OutT, true>}) {
                    cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    cudaFuncSetAttribute(fk, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         (int)cudaSharedmemCarveoutMaxShared);
                }
                attr_fb = true;
            }
            KTime *t = kt_begin(ctx, "k_rqi");
            if (P[MR3_RQI_FB] >= 2)
                k_rqi_fb<R, OutT, true><<<ntasks, FB_TPB, smem, s>>>(A);
            else
                k_rqi_fb<R, OutT, false><<<ntasks, FB_TPB, smem, s>>>(A);
            kt_end(ctx, t);
            CKL("k_rqi_fb");
        }
        size_t tmpl = 0;
        cub::DeviceSelect::Flagged(nullptr, tmpl, slist, left, llist, lcnt, ncount, s);
        void *tmp = getbuf(ctx, "cubtmp_left", tmpl, &rc2);
        if (rc2) return rc2;
        cub::DeviceSelect::Flagged(tmp, tmpl, slist, left, llist, lcnt, ncount, s);
        CKL("select (rqi left)");
        int hl = 0;
        CK(cudaMemcpyAsync(&hl, lcnt, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#13b");
        if (ctx->dump) fprintf(stderr, "[mr3] k_rqi_fb left %d of %d eigenpairs\n", hl, ncount);
        if (hl == 0) return 0;
        if (P[MR3_RQI_CHUNK] > 0)  // the stragglers: chunk-parallel, one CTA each
            return run_chunked(llist, hl, resume);
        if ((rc2 = make_tasks(llist, &ntasks, rtpb, hl))) return rc2;
        rqi_resume_in = resume;
        rqi_iter0 = std::min(2, (int)P[MR3_MAX_RQI]);
        rqi_tname = "k_rqi_tail";
        rc2 = launch_chunks(false, llist, ntasks);
        rqi_tname = "k_rqi";
        rqi_resume_in = nullptr;
        rqi_iter0 = 0;
        return rc2;
    };

    auto dump = [&](const char *tag, const int32_t *list, int cntl, int lvl) {
        if (!ctx->dump) return;
        cudaStreamSynchronize(ctx->stream);
        std::vector<int32_t> ids(cntl);
        std::vector<R> lo(cnt), hi(cnt);
        std::vector<int32_t> nodev(cnt), kv(cnt);
        std::vector<double> lg(cnt), rg(cnt);
        cudaMemcpy(ids.data(), list, cntl * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(lo.data(), W.it.lo, cnt * sizeof(R), cudaMemcpyDeviceToHost);
        cudaMemcpy(hi.data(), W.it.hi, cnt * sizeof(R), cudaMemcpyDeviceToHost);
        cudaMemcpy(nodev.data(), W.it.node, cnt * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(kv.data(), W.it.k, cnt * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(lg.data(), W.it.lgap, cnt * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(rg.data(), W.it.rgap, cnt * 8, cudaMemcpyDeviceToHost);
        std::vector<NodeInfo> nds(ctx->nodes_used);
        cudaMemcpy(nds.data(), W.nodes, ctx->nodes_used * sizeof(NodeInfo), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[mr3] level %d %s: %d items\n", lvl, tag, cntl);
        for (int i = 0; i < cntl && i < ctx->dump; i++) {
            int id = ids[i];
            const NodeInfo &nd = nds[nodev[id]];
            fprintf(stderr, "  id %d k %d node %d depth %d sig %.17g lo %.17g%+.3g hi %.17g%+.3g w %.3g lg %.3g rg %.3g\n",
                    id, kv[id], nodev[id], nd.depth, nd.sig_hi, hi_of(lo[id]), lo_of(lo[id]),
                    hi_of(hi[id]), lo_of(hi[id]), hi_of(hi[id]) - hi_of(lo[id]), lg[id], rg[id]);
        }
    };

    // Tree traversal (Alg. 1 l.5-17).  Level 0 is one batch; the clusters of a level are
    // processed breadth-first in batches (one launch per kernel for all clusters of a batch,
    // reading R12) whose child representations fit the pool budget (MR3_POOL_MB); batches
    // are taken depth-first from a stack, so a batch's subtree is finished before the next
    // batch of its level reuses the level's pool (depth-first keeps the
    // memory at O((depth + batch) n) instead of O(clusters n), SPEC memory contract).
    struct Frontier {
        int level;                       // depth of the member items' nodes
        std::vector<int32_t> cb, ce, mem;  // clusters [cb, ce) into mem (item ids)
    };
    std::vector<Frontier> stack;
    auto push_clusters = [&](int lvl, int nc, int nm) -> int {
        if (nc <= 0) return 0;
        Frontier F;
        F.level = lvl;
        F.cb.resize(nc);
        F.ce.resize(nc);
        F.mem.resize(nm);
        CK(cudaMemcpyAsync(F.cb.data(), cbeg, nc * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(F.ce.data(), cend, nc * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(F.mem.data(), listB, nm * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        hsync_note(ctx, "sync#14");
        stack.push_back(std::move(F));
        return 0;
    };
    const int maxdepth = (int)P[MR3_MAX_DEPTH];
    const double elg1 = P[MR3_ELG_MAX];
    const double elg2 = std::max(10.0, eps_x / (eps_y * std::sqrt((double)ctx->n)));
    const int Gc = P[MR3_GROUPS] > 0 ? choose_groups(ctx, 0, (int)P[MR3_GROUPS]) : 8;
    // child pool budget: rep (4 R) + M_x (2 doubles) + PP rows per row and cluster
    const size_t row_bytes = (size_t)4 * words * 8 + 16 + (size_t)PP_STRIDE * 8;
    size_t pool_budget = P[MR3_POOL_MB] > 0 ? (size_t)(P[MR3_POOL_MB] * 1048576.0)
                                            : std::min<size_t>((size_t)8 << 30, (size_t)(freeb * 0.15));
    const int64_t batch_max =
        std::max<int64_t>(1, (int64_t)(pool_budget / std::max<size_t>(1, row_bytes * (size_t)ctx->n)));
    int dmax = 0;
    if (nsing > 0) {
        rc = run_rqi(singles, nsing);
        if (rc) return rc;
    }
    if ((rc = push_clusters(0, nclus, nmem))) return rc;
    while (!stack.empty()) {
        Frontier F = std::move(stack.back());
        stack.pop_back();
        const int nc = (int)F.cb.size();
        if (nc > batch_max) {  // split into batches (pushed in reverse: taken in order)
            std::vector<Frontier> parts;
            for (int c0b = 0; c0b < nc; c0b += (int)batch_max) {
                const int c1b = (int)std::min<int64_t>(nc, c0b + batch_max);
                Frontier Q;
                Q.level = F.level;
                const int m0 = F.cb[c0b];
                for (int c = c0b; c < c1b; c++) {
                    Q.cb.push_back(F.cb[c] - m0);
                    Q.ce.push_back(F.ce[c] - m0);
                }
                Q.mem.assign(F.mem.begin() + m0, F.mem.begin() + F.ce[c1b - 1]);
                parts.push_back(std::move(Q));
            }
            for (auto it2 = parts.rbegin(); it2 != parts.rend(); ++it2) stack.push_back(std::move(*it2));
            continue;
        }
        const int nm = (int)F.mem.size();
        CK(cudaMemcpyAsync(listB, F.mem.data(), nm * 4, cudaMemcpyHostToDevice, s));
        if (F.level + 1 > maxdepth) {
            // depth cap: the members get the bisection fallback + one solve each (the RQI
            // kernel's fallback path)
            double saved = ctx->cfg[mode].v[MR3_MAX_RQI];
            ctx->cfg[mode].v[MR3_MAX_RQI] = 0;
            P = ctx->cfg[mode].v;
            rc = run_rqi(listB, nm);
            ctx->cfg[mode].v[MR3_MAX_RQI] = saved;
            P = ctx->cfg[mode].v;
            if (rc) return rc;
            continue;
        }
        CK(cudaMemcpyAsync(cbeg, F.cb.data(), nc * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(cend, F.ce.data(), nc * 4, cudaMemcpyHostToDevice, s));
        // K4: child representations (new nodes)
        if (ctx->nodes_used + nc > ctx->node_cap) {
            // grow the node table (keep contents)
            int newcap = std::max(ctx->node_cap * 2, ctx->nodes_used + nc + 64);
            NodeInfo *nn = nullptr;
            CK(cudaMalloc(&nn, newcap * sizeof(NodeInfo)));
            CK(cudaMemcpyAsync(nn, W.nodes, ctx->nodes_used * sizeof(NodeInfo),
                               cudaMemcpyDeviceToDevice, s));
            CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#15");
            cudaFree(ctx->bufs["nodes"].p);
            ctx->bufs["nodes"].p = nn;
            ctx->bufs["nodes"].cap = newcap * sizeof(NodeInfo);
            ctx->node_cap = newcap;
            W.nodes = nn;
        }
        // pool of this level (children of depth level + 1); reused by the level's later batches
        std::string pname = "child_pool" + std::to_string(F.level);
        double *pool = (double *)getbuf(ctx, pname, (size_t)nc * ctx->n * 4 * words * 8, &rc);
        double *poolx = (double *)getbuf(ctx, pname + "x", ((size_t)nc * ctx->n + XPAD) * 16, &rc);
        double *ppc = (double *)getbuf(ctx, pname + "pp", (size_t)nc * ctx->n * PP_STRIDE * 8, &rc);
        if (rc) return rc;
        CK(cudaMemsetAsync(poolx + 2 * (size_t)nc * ctx->n, 0, XPAD * 16, s));
        double *cdbg = nullptr;
        if (ctx->dump) cdbg = (double *)getbuf(ctx, "child_dbg", (size_t)nc * 32, &rc);
        KTime *tch = kt_begin(ctx, "k_child");
        // backtracking (R22): children at depth >= 2 that fail the acceptance tests are redone
        // from their grandparent (MR3_BACKTRACK = 2: a test hook that fails every child at
        // depth >= 2 in the first launch)
        const int bt = (int)P[MR3_BACKTRACK];
        double *cfail = nullptr;
        if (bt && F.level >= 1) {
            cfail = (double *)getbuf(ctx, "child_fail", (size_t)nc * 8, &rc);
            if (rc) return rc;
        }
        k_child<R><<<nc, 32, 0, s>>>(W.nodes, ctx->nodes_used, W.it, listB, cbeg, cend, nc, pool,
                                     poolx, ctx->n, ctx->spdiam, elg1, elg2, ctx->pivmin, W.st,
                                     cdbg, cfail, 0, bt == 2 ? 2 : 0);
        CKL("k_child");
        if (cfail) {
            k_child<R><<<nc, 32, 0, s>>>(W.nodes, ctx->nodes_used, W.it, listB, cbeg, cend, nc,
                                         pool, poolx, ctx->n, ctx->spdiam, elg1, elg2, ctx->pivmin,
                                         W.st, cdbg, cfail, 1, 0);
            CKL("k_child (backtrack)");
        }
        kt_end(ctx, tch);
        if (ctx->dump) {
            std::vector<double> hd(4 * nc);
            cudaStreamSynchronize(s);
            cudaMemcpy(hd.data(), cdbg, nc * 32, cudaMemcpyDeviceToHost);
            for (int c = 0; c < nc && c < ctx->dump; c++)
                fprintf(stderr, "[mr3] child %d: lane %g growth %.3g delta %.3g tau %.17g\n", c,
                        hd[4 * c], hd[4 * c + 1], hd[4 * c + 2], hd[4 * c + 3]);
        }
        k_node_pp<R><<<nc, 256, 0, s>>>(W.nodes, ctx->nodes_used, ppc, ctx->n, 0);
        CKL("k_node_pp");
        ctx->nodes_used += nc;
        dump("after child", listB, nm, F.level + 1);
        // K2: refine in the child coordinates (certified)
        rc = launch_bisect<R>(ctx, W, listB, nm, Gc, rtol, absfloor, 1,
                              words == 2 && P[MR3_XPHASE] != 0, eps_x);
        if (rc) return rc;
        dump("after refine", listB, nm, F.level + 1);
        // K3: classify the members (singletons, clusters with members in listB)
        CK(cudaMemcpyAsync(listA, listB, nm * 4, cudaMemcpyDeviceToDevice, s));
        so.next_active = listB;
        KTime *tc2 = kt_begin(ctx, "k_classify");
        k_classify<R><<<1, 1024, 0, s>>>(W.it, listA, nm, gaptol, so,
                                                   P[MR3_ABSGAP] * ctx->norm1 * ctx->scale);
        kt_end(ctx, tc2);
        CKL("k_classify");
        CK(cudaMemcpyAsync(hc, dcounts, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#16");
        const int ns2 = hc[0], nc2 = hc[1], nm2 = hc[2];
        dmax = std::max(dmax, F.level + 1);
        if (ctx->dump)
            fprintf(stderr, "[mr3] level %d batch: %d singles %d clusters %d members\n",
                    F.level + 1, ns2, nc2, nm2);
        if (ns2 > 0) {
            rc = run_rqi(singles, ns2);
            if (rc) return rc;
        }
        if ((rc = push_clusters(F.level + 1, nc2, nm2))) return rc;
    }
    const int level = dmax;
    ctx->stats.levels = dmax + 1;
    if (ctx->dump && ctx->bufs.count("rqi_sorted") && ctx->n > 1) {
        // twist-index distribution (r / n in 10 bins) and spread per 128-run of the sorted list
        cudaStreamSynchronize(s);
        std::vector<int32_t> tw(cnt), nodev(cnt);
        cudaMemcpy(tw.data(), W.it.twist, cnt * 4, cudaMemcpyDeviceToHost);
        int hist[10] = {0};
        for (int i = 0; i < cnt; i++) hist[std::min(9, std::max(0, (int)(10.0 * tw[i] / ctx->n)))]++;
        fprintf(stderr, "[mr3] twist r/n histogram:");
        for (int i = 0; i < 10; i++) fprintf(stderr, " %d", hist[i]);
        fprintf(stderr, "\n");
    }
    if (ctx->dump && ctx->bufs.count("dbg_iters")) {
        cudaStreamSynchronize(s);
        std::vector<int32_t> itv(cnt);
        std::vector<double> lg(cnt), rg(cnt);
        std::vector<R> lam(cnt);
        cudaMemcpy(itv.data(), ctx->bufs["dbg_iters"].p, cnt * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(lg.data(), W.it.lgap, cnt * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(rg.data(), W.it.rgap, cnt * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(lam.data(), W.it.lo, cnt * sizeof(R), cudaMemcpyDeviceToHost);
        int hist[16] = {0};
        for (int i = 0; i < cnt; i++) hist[std::min(15, std::max(0, itv[i]))]++;
        fprintf(stderr, "[mr3] rqi iteration histogram:");
        for (int i = 0; i < 16; i++)
            if (hist[i]) fprintf(stderr, " %d:%d", i, hist[i]);
        fprintf(stderr, "\n");
        int shown = 0;
        for (int i = 0; i < cnt && shown < 40; i++) {
            double tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (itv[i] >= 4)
                cudaMemcpy(tr, (double *)ctx->bufs["dbg_trace"].p + 8 * (size_t)i, 64,
                           cudaMemcpyDeviceToHost);
            if (itv[i] >= 4 && tr[5] != 0.0) {
                fprintf(stderr,
                        "  item %d iters %d lam %.17g lgap %.3g rgap %.3g | x0 %g gap %.3g r %g "
                        "res/tol %.3g %.3g %.3g %.3g | split log2 rel %.1f\n",
                        i, itv[i], hi_of(lam[i]), lg[i], rg[i], tr[0], tr[1], tr[2], tr[3], tr[4],
                        tr[5], tr[6], tr[7]);
                shown++;
            }
        }
        cudaMemset(ctx->bufs["dbg_iters"].p, 0, cnt * 4);
        cudaMemset(ctx->bufs["dbg_trace"].p, 0, (size_t)cnt * 64);
    }
    if (dzc && !ctx->fuse_scale) {  // K6 epilogue: per-column factors and exact normalisation (k_zprod.cuh)
        KTime *tf = kt_begin(ctx, "k_zscale");
        const int64_t nc = c1 - c0;
        k_zscale<OutT><<<ctx->nsm * 16, 256, 0, s>>>(Z, ldz, nc, dzc, ctx->n);
        kt_end(ctx, tf);
        CKL("k_zscale");
    }
    // split matrices: restore "w ascending" over this rank's columns (k_misc.cuh)
    if (ctx->split && c1 - c0 > 1) {
        const int mm = (int)(c1 - c0);
        OutT *wl = w + c0;
        unsigned long long *sk = (unsigned long long *)getbuf(ctx, "srt_keys", (size_t)mm * 8, &rc);
        unsigned long long *sk2 = (unsigned long long *)getbuf(ctx, "srt_keys2", (size_t)mm * 8, &rc);
        int32_t *sv = (int32_t *)getbuf(ctx, "srt_vals", (size_t)mm * 4, &rc);
        int32_t *perm = (int32_t *)getbuf(ctx, "srt_perm", (size_t)mm * 4, &rc);
        int *ninv = (int *)getbuf(ctx, "srt_ninv", 16, &rc);
        if (rc) return rc;
        CK(cudaMemsetAsync(ninv, 0, 4, s));
        k_sort_keys<OutT><<<(mm + 255) / 256, 256, 0, s>>>(wl, mm, sk, sv, ninv);
        CKL("k_sort_keys");
        int hinv = 0;
        CK(cudaMemcpyAsync(&hinv, ninv, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#15b");
        if (hinv > 0) {
            size_t tmpb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmpb, sk, sk2, sv, perm, mm, 0, 64, s);
            void *tmp = getbuf(ctx, "cubtmp", tmpb, &rc);
            OutT *wt = (OutT *)getbuf(ctx, "srt_w", (size_t)mm * sizeof(OutT), &rc);
            char *lead = (char *)getbuf(ctx, "srt_lead", (size_t)mm, &rc);
            if (rc) return rc;
            cub::DeviceRadixSort::SortPairs(tmp, tmpb, sk, sk2, sv, perm, mm, 0, 64, s);
            CKL("radix sort (w)");
            k_gather_w<OutT><<<(mm + 255) / 256, 256, 0, s>>>(wl, perm, mm, wt);
            CKL("k_gather_w");
            CK(cudaMemcpyAsync(wl, wt, (size_t)mm * sizeof(OutT), cudaMemcpyDeviceToDevice, s));
            if (jobz == 'V' && Z != nullptr) {
                k_cycle_leaders<<<(mm + 255) / 256, 256, 0, s>>>(perm, mm, lead);
                CKL("k_cycle_leaders");
                const int gy = (int)std::min<int64_t>(64, (ctx->n + 255) / 256);
                k_permute_cols<OutT><<<dim3(mm, gy), 256, 0, s>>>(Z, ldz, ctx->n, perm, lead);
                CKL("k_permute_cols");
            }
        }
    }
    ctx->stats.d_max = level;
    DevStats hst;
    CK(cudaMemcpyAsync(&hst, W.st, sizeof(hst), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#16");
    kt_collect(ctx);
    ctx->stats.n_clusters = hst.n_clusters;
    ctx->stats.largest_cluster = std::max(1, hst.largest_cluster);
    ctx->stats.rho = (double)ctx->stats.largest_cluster / (double)ctx->n;
    ctx->stats.robustness_failures = hst.robustness_failures;
    ctx->stats.backtracks = hst.backtracks;
    ctx->stats.backtrack_tries = hst.backtrack_tries;
    ctx->stats.rqi_fallbacks = hst.rqi_fallbacks;
    ctx->stats.rqi_iters_max = hst.rqi_iters_max;
    ctx->stats.bisect_rows = (double)hst.bisect_rows;
    ctx->stats.bisect_rows_x = (double)hst.bisect_rows_x;
    ctx->stats.newton_rows_x = (double)hst.newton_rows_x;
    ctx->stats.rqi_rows = (double)hst.rqi_rows;
    for (auto &p : ctx->ktimes) {
        const std::string &nm = p.first;
        int slot = nm == "k_root" ? 0 : nm == "k_bisect" ? 1 : nm == "k_classify" ? 2
                                     : nm == "k_child"  ? 3 : (nm == "k_rqi" || nm == "k_rqi_tail" || nm == "k_rqi_serial") ? 4 : 6;
        ctx->stats.t_ms[slot] += p.second.first;
        ctx->stats.t_ms[5] += p.second.first;
    }
    if (stats) *stats = ctx->stats;
    ctx->planned = false;
    return 0;
}

// ------------------------------------------------------------------ C-ABI

extern "C" {

int mr3_create(mr3_ctx *out, int device, void *cuda_stream, void *nccl_comm, int rank,
               int world) {
    if (!out) return -1;
    if (world < 1 || rank < 0 || rank >= world) return -5;
    mr3_ctx ctx = new mr3_ctx_s();
    ctx->device = device;
    ctx->nccl_comm = nccl_comm;
    ctx->crank = rank;
    ctx->cworld = world;
    for (int m = 0; m < 2; m++)
        for (int i = 0; i < MR3_NPARAM; i++) ctx->cfg[m].v[i] = kDefaults[m][i];
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return MR3_ERR_CUDA;
    }
    if (cuda_stream) {
        ctx->stream = (cudaStream_t)cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete ctx;
            return MR3_ERR_CUDA;
        }
        ctx->own_stream = true;
    }
    if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_root, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_pp, cudaEventDisableTiming) != cudaSuccess) {
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        delete ctx;
        return MR3_ERR_CUDA;
    }
    cudaEventRecord(ctx->ev_pp, ctx->side);  // (completed: nothing to wait for before a plan)
    cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, device);
    *out = ctx;
    return 0;
}

int mr3_destroy(mr3_ctx ctx) {
    if (!ctx) return 0;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->side);  // (its kernels read the buffers freed below)
    for (auto &b : ctx->bufs)
        if (b.second.p) cudaFree(b.second.p);
    for (auto &t : ctx->kt) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    if (ctx->cublas && cublas_load()) g_cublas.Destroy(ctx->cublas);
    if (ctx->dn_exec) cudaGraphExecDestroy(ctx->dn_exec);
    for (auto &ev : ctx->dn_ev)
        if (ev) cudaEventDestroy(ev);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->ev_root);
    cudaEventDestroy(ctx->ev_pp);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return 0;
}

int mr3_set_param(mr3_ctx ctx, int mode, int which, double value) {
    if (!ctx || mode < 0 || mode > 1 || which < 0 || which >= MR3_NPARAM) return -1;
    ctx->cfg[mode].v[which] = value < 0 && which != MR3_RTOL ? kDefaults[mode][which] : value;
    return 0;
}

double mr3_get_param(mr3_ctx ctx, int mode, int which) {
    if (!ctx || mode < 0 || mode > 1 || which < 0 || which >= MR3_NPARAM) return NAN;
    return ctx->cfg[mode].v[which];
}

int mr3_plan(mr3_ctx ctx, int mode, char range, int64_t n, const void *d, const void *e, double vl,
             double vu, int64_t il, int64_t iu, int rank, int world, int64_t *m, double **brk,
             int64_t *slice_cap, int64_t *slice_cnt) {
    if (!ctx) return -1;
    if (!m || !brk || !slice_cap || !slice_cnt) return -13;
    if (n > 0 && (!d || (n > 1 && !e))) return -5;
    if (mode == 0)
        return plan_impl<dd, double>(ctx, range, n, (const double *)d, (const double *)e, vl, vu,
                                     il, iu, rank, world, m, brk, slice_cap, slice_cnt);
    if (mode == 1)
        return plan_impl<double, float>(ctx, range, n, (const float *)d, (const float *)e, vl, vu,
                                        il, iu, rank, world, m, brk, slice_cap, slice_cnt);
    return -2;
}

int mr3_execute(mr3_ctx ctx, char jobz, void *w, void *Z, int64_t ldz, int64_t zcap,
                int64_t *zcol_begin, int64_t *zcol_end, mr3_stats *stats) {
    if (!ctx) return -1;
    if (!zcol_begin || !zcol_end) return -7;
    if (ctx->mode == 0)
        return execute_impl<dd, double>(ctx, jobz, (double *)w, (double *)Z, ldz, zcap, zcol_begin,
                                        zcol_end, stats);
    return execute_impl<double, float>(ctx, jobz, (float *)w, (float *)Z, ldz, zcap, zcol_begin,
                                       zcol_end, stats);
}

// the one-call solve: plan, all-gather of the bracket records, execute, all-gather of w
static int solve_common(mr3_ctx ctx, int mode, char jobz, char range, int64_t n, const void *d,
                        const void *e, double vl, double vu, int64_t il, int64_t iu, int64_t *m,
                        void *w, void *Z, int64_t ldz, int64_t zcap, int64_t *zcol_begin,
                        int64_t *zcol_end, mr3_stats *stats) {
    if (!ctx) return -1;
    if (jobz != 'V' && jobz != 'N') return -2;
    if (range != 'A' && range != 'I' && range != 'V') return -3;
    if (n < 0) return -4;
    if (!m) return -11;
    if (n > 0 && !w) return -12;
    if (jobz == 'V' && n > 0 && (!Z || ldz < n)) return -14;
    if (!zcol_begin || !zcol_end) return -16;
    *zcol_begin = 0;
    *zcol_end = 0;
    double *brk = nullptr;
    int64_t cap = 0, cntm = 0;
    int rc = mr3_plan(ctx, mode, range, n, d, e, vl, vu, il, iu, ctx->crank, ctx->cworld, m, &brk,
                      &cap, &cntm);
    if (rc) {
        if (stats) *stats = ctx->stats;
        return rc;
    }
    if (ctx->cworld > 1 && brk != nullptr) {
        rc = exchange_allgather(ctx, brk, (size_t)cap * MR3_BRK_REC * sizeof(double));
        if (rc) return rc;
    }
    rc = mr3_execute(ctx, jobz, w, Z, ldz, zcap, zcol_begin, zcol_end, stats);
    *m = ctx->m < 0 ? 0 : ctx->m;
    if (rc || ctx->cworld <= 1 || *m == 0) return rc;
    // w: every rank holds its own columns' eigenvalues; padded all-gather of the slices
    const std::vector<int64_t> cb = ctx->colb;
    if ((int)cb.size() != ctx->cworld + 1) {
        ctx->err = "column partition missing";
        return MR3_ERR_STATE;
    }
    int64_t wcap = 1;
    for (int r = 0; r < ctx->cworld; r++) wcap = std::max(wcap, cb[r + 1] - cb[r]);
    const size_t es = mode ? 4 : 8;
    char *wg = (char *)getbuf(ctx, "w_gather", (size_t)ctx->cworld * wcap * es, &rc);
    if (rc) return rc;
    cudaStream_t s = ctx->stream;
    const int me = ctx->crank;
    if (cb[me + 1] > cb[me])
        CK(cudaMemcpyAsync(wg + (size_t)me * wcap * es, (char *)w + cb[me] * es,
                           (size_t)(cb[me + 1] - cb[me]) * es, cudaMemcpyDeviceToDevice, s));
    rc = exchange_allgather(ctx, wg, (size_t)wcap * es);
    if (rc) return rc;
    for (int r = 0; r < ctx->cworld; r++)
        if (r != me && cb[r + 1] > cb[r])
            CK(cudaMemcpyAsync((char *)w + cb[r] * es, wg + (size_t)r * wcap * es,
                               (size_t)(cb[r + 1] - cb[r]) * es, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    return 0;
}

int mr3_dstemr_dd(mr3_ctx ctx, char jobz, char range, int64_t n, const double *d, const double *e,
                  double vl, double vu, int64_t il, int64_t iu, int64_t *m, double *w, double *Z,
                  int64_t ldz, int64_t zcap, int64_t *zcol_begin, int64_t *zcol_end,
                  mr3_stats *stats) {
    return solve_common(ctx, 0, jobz, range, n, d, e, vl, vu, il, iu, m, w, Z, ldz, zcap,
                        zcol_begin, zcol_end, stats);
}

int mr3_sstemr_d(mr3_ctx ctx, char jobz, char range, int64_t n, const float *d, const float *e,
                 float vl, float vu, int64_t il, int64_t iu, int64_t *m, float *w, float *Z,
                 int64_t ldz, int64_t zcap, int64_t *zcol_begin, int64_t *zcol_end,
                 mr3_stats *stats) {
    return solve_common(ctx, 1, jobz, range, n, d, e, vl, vu, il, iu, m, w, Z, ldz, zcap,
                        zcol_begin, zcol_end, stats);
}

// ------------------------------------------------------------------ dense pipeline (NEXT-4)
// A = Q T Q^T (k_sytd_col + k_sytd_fused per reflector), the tridiagonal solve of T, and
// Z <- Q Z in blocks of DN_NB reflectors (library GEMMs).  PAPER.md L1506-L1550; k_dense.cuh.
int mr3_dsyevr_dd(mr3_ctx ctx, char jobz, char range, int64_t n, double *A, int64_t lda,
                  double vl, double vu, int64_t il, int64_t iu, int64_t *m, double *w, double *Z,
                  int64_t ldz, mr3_stats *stats) {
    if (!ctx) return -1;
    if (jobz != 'V' && jobz != 'N') return -2;
    if (range != 'A' && range != 'I' && range != 'V') return -3;
    if (n < 0 || n > 0x7fffffffLL) return -4;
    if (n > 0 && !A) return -5;
    if (lda < std::max<int64_t>(1, n)) return -6;
    if (n > 1024 * DN_KE) {  // k_sytd_col keeps a column in registers of one CTA
        ctx->err = "mr3_dsyevr_dd: n > 8192";
        return -4;
    }
    if (!m) return -11;
    if (n > 0 && !w) return -12;
    if (jobz == 'V' && n > 0 && (!Z || ldz < n)) return -13;
    if (ctx->cworld > 1) {
        ctx->err = "mr3_dsyevr_dd: single-rank contexts only";
        return MR3_ERR_STATE;
    }
    *m = 0;
    if (n == 0) return 0;
    int rc = 0;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int nn = (int)n;
    double *dd_ = (double *)getbuf(ctx, "dn_d", (size_t)n * 8, &rc);
    double *de_ = (double *)getbuf(ctx, "dn_e", (size_t)n * 8, &rc);
    double *tau = (double *)getbuf(ctx, "dn_tau", (size_t)n * 8, &rc);
    double *vb = (double *)getbuf(ctx, "dn_v", (size_t)2 * n * 8, &rc);
    double *wv = (double *)getbuf(ctx, "dn_w", (size_t)n * 8, &rc);
    double *yv = (double *)getbuf(ctx, "dn_y", (size_t)n * 8, &rc);
    if (rc) return rc;
    // max |a_ij| far from 1: scale A by a power of 2 first (the reflector norms square the
    // entries: 1e-200 underflows, 1e200 overflows), w back at the end (as LAPACK's dsyevr scales
    // outside [sqrt(smallest), sqrt(largest)]); nothing is touched in between, so the usual
    // inputs keep their bits
    double dn_unscale = 1.0;
    {
        unsigned long long *amx = (unsigned long long *)getbuf(ctx, "dn_amax", 16, &rc);
        if (rc) return rc;
        CK(cudaMemsetAsync(amx, 0, 8, s));
        k_dense_absmax<<<ctx->nsm * 4, 256, 0, s>>>(A, lda, nn, amx);
        CKL("k_dense_absmax");
        unsigned long long hb = 0;
        CK(cudaMemcpyAsync(&hb, amx, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double amax;
        memcpy(&amax, &hb, 8);
        if (amax > 0.0 && amax < INFINITY && (amax < ldexp(1.0, -400) || amax > ldexp(1.0, 400))) {
            int ex = 0;
            frexp(amax, &ex);
            // two exact steps where one power of 2 would leave the double range
            const int e1 = -ex / 2, e2 = -ex - e1;
            k_dense_scale<<<ctx->nsm * 4, 256, 0, s>>>(A, lda, nn, ldexp(1.0, e1));
            k_dense_scale<<<ctx->nsm * 4, 256, 0, s>>>(A, lda, nn, ldexp(1.0, e2));
            CKL("k_dense_scale");
            vl = ldexp(ldexp(vl, e1), e2);
            vu = ldexp(ldexp(vu, e1), e2);
            dn_unscale = (double)ex;  // w <- w 2^ex (applied in two steps below)
        }
    }
    cudaEvent_t ev[2];
    CK(cudaEventCreate(&ev[0]));
    CK(cudaEventCreate(&ev[1]));
    CK(cudaEventRecord(ev[0], s));
    // reduction: per reflector the O(n) column step and one sweep of the trailing block --
    // 2n - 1 launches, captured once into a CUDA graph (per argument set) and replayed on the
    // internal stream, ordered after / before the caller's stream by events
    int64_t launches = 0;
    auto issue = [&](cudaStream_t st) {
        for (int j = 0; j < nn; j++) {
            double *vcur = vb + (size_t)(j & 1) * n, *vprev = vb + (size_t)((j + 1) & 1) * n;
            k_sytd_col<<<1, 1024, 0, st>>>(A, lda, nn, j, vprev, yv, wv, vcur, tau, dd_, de_);
            launches++;
            if (j > nn - 2) break;
            const int cols = nn - j - 1;
            k_sytd_fused<<<(cols + DN_CPB - 1) / DN_CPB, DN_COLTPB, 0, st>>>(A, lda, nn, j, vprev, wv,
                                                                              vcur, tau, yv);
            launches++;
        }
    };
    const std::vector<const void *> key = {A, (const void *)(intptr_t)lda, (const void *)(intptr_t)n,
                                           dd_, de_, tau, vb, wv, yv};
    if (ctx->dn_exec == nullptr || ctx->dn_key != key) {
        if (ctx->dn_exec) cudaGraphExecDestroy(ctx->dn_exec);
        ctx->dn_exec = nullptr;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(ctx->side, cudaStreamCaptureModeThreadLocal));
        issue(ctx->side);
        CK(cudaStreamEndCapture(ctx->side, &g));
        const cudaError_t ie = cudaGraphInstantiate(&ctx->dn_exec, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) {
            ctx->dn_exec = nullptr;
            ctx->err = std::string("dense reduction graph: ") + cudaGetErrorString(ie);
            return MR3_ERR_CUDA;
        }
        ctx->dn_key = key;
    } else {
        launches = 2 * n - 1;
    }
    if (!ctx->dn_ev[0]) {
        CK(cudaEventCreateWithFlags(&ctx->dn_ev[0], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->dn_ev[1], cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ctx->dn_ev[0], s));
    CK(cudaStreamWaitEvent(ctx->side, ctx->dn_ev[0], 0));
    CK(cudaGraphLaunch(ctx->dn_exec, ctx->side));
    CK(cudaEventRecord(ctx->dn_ev[1], ctx->side));
    CK(cudaStreamWaitEvent(s, ctx->dn_ev[1], 0));
    CK(cudaEventRecord(ev[1], s));
    // the tridiagonal eigenproblem of T (the paper's mixed-precision solver)
    int64_t zb = 0, ze = 0;
    rc = mr3_dstemr_dd(ctx, jobz, range, n, dd_, de_, vl, vu, il, iu, m, w, Z, ldz,
                       jobz == 'V' ? n : 0, &zb, &ze, stats);
    if (rc) return rc;
    if (dn_unscale != 1.0 && *m > 0) {
        const int ex = (int)dn_unscale, e1 = ex / 2, e2 = ex - e1;
        k_vec_scale<<<(int)((*m + 255) / 256), 256, 0, s>>>(w, *m, ldexp(1.0, e1));
        k_vec_scale<<<(int)((*m + 255) / 256), 256, 0, s>>>(w, *m, ldexp(1.0, e2));
        CKL("k_vec_scale");
    }
    ctx->launches += launches;
    float ms_red = 0.f;
    CK(cudaEventSynchronize(ev[1]));
    CK(cudaEventElapsedTime(&ms_red, ev[0], ev[1]));
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    ctx->ktimes.push_back({"k_sytrd", {(double)ms_red, (int)launches}});
    const int64_t mcols = *m;
    if (jobz == 'V' && mcols > 0 && n > 2) {
        // back-transformation, blocks of reflectors from the last to the first
        if (!cublas_load()) {
            ctx->err = "libcublas.so.12 not found (dense back-transformation)";
            return MR3_ERR_CUDA;
        }
        if (!ctx->cublas && g_cublas.Create(&ctx->cublas) != CUBLAS_STATUS_SUCCESS) {
            ctx->cublas = nullptr;
            ctx->err = "cublasCreate failed";
            return MR3_ERR_CUDA;
        }
        g_cublas.SetStream(ctx->cublas, s);
        double *V = (double *)getbuf(ctx, "dn_V", (size_t)n * DN_NB * 8, &rc);
        double *G = (double *)getbuf(ctx, "dn_G", (size_t)DN_NB * DN_NB * 8, &rc);
        double *Tm = (double *)getbuf(ctx, "dn_T", (size_t)DN_NB * DN_NB * 8, &rc);
        double *W1 = (double *)getbuf(ctx, "dn_W1", (size_t)DN_NB * mcols * 8, &rc);
        double *W2 = (double *)getbuf(ctx, "dn_W2", (size_t)DN_NB * mcols * 8, &rc);
        if (rc) return rc;
        KTime *tb = kt_begin(ctx, "k_ormtr");
        const int nref = nn - 2;  // reflectors 0 .. n - 3 (the last one of the reduction is I)
        const double one = 1.0, zero = 0.0, mone = -1.0;
        auto gemm = [&](cublasOperation_t ta, cublasOperation_t tb_, int M, int N, int K,
                        const double *al, const double *Am, int64_t la, const double *Bm,
                        int64_t lb, const double *be, double *Cm, int64_t lc) -> int {
            if (g_cublas.Dgemm(ctx->cublas, ta, tb_, M, N, K, al, Am, (int)la, Bm, (int)lb, be, Cm,
                               (int)lc) != CUBLAS_STATUS_SUCCESS) {
                ctx->err = "cublasDgemm failed";
                return MR3_ERR_CUDA;
            }
            return 0;
        };
        const int nblk = (nref + DN_NB - 1) / DN_NB;
        for (int b = nblk - 1; b >= 0; b--) {
            const int j0 = b * DN_NB, kb = std::min(DN_NB, nref - j0);
            const int mr = nn - j0 - 1;  // rows j0 + 1 .. n - 1
            const int64_t tot = (int64_t)mr * kb;
            k_build_v<<<(int)((tot + 255) / 256), 256, 0, s>>>(A, lda, nn, j0, kb, V, n);
            CKL("k_build_v");
            if ((rc = gemm(CUBLAS_OP_T, CUBLAS_OP_N, kb, kb, mr, &one, V, n, V, n, &zero, G, kb)))
                return rc;
            k_larft<<<1, DN_NB, 0, s>>>(G, kb, tau, j0, Tm);
            CKL("k_larft");
            double *Zs = Z + j0 + 1;
            // W1 = V^T Z(j0+1:, :), W2 = T W1, Z(j0+1:, :) -= V W2
            if ((rc = gemm(CUBLAS_OP_T, CUBLAS_OP_N, kb, (int)mcols, mr, &one, V, n, Zs, ldz, &zero,
                           W1, kb)))
                return rc;
            if ((rc = gemm(CUBLAS_OP_N, CUBLAS_OP_N, kb, (int)mcols, kb, &one, Tm, kb, W1, kb, &zero,
                           W2, kb)))
                return rc;
            if ((rc = gemm(CUBLAS_OP_N, CUBLAS_OP_N, mr, (int)mcols, kb, &mone, V, n, W2, kb, &one,
                           Zs, ldz)))
                return rc;
            ctx->launches += 3;
        }
        kt_end(ctx, tb);
        kt_collect(ctx);
    }
    CK(cudaStreamSynchronize(s));
    if (stats) {
        *stats = ctx->stats;
        for (auto &p : ctx->ktimes) {
            if (p.first == "k_sytrd") stats->t_ms[6] = p.second.first;
            if (p.first == "k_ormtr") stats->t_ms[7] = p.second.first;
        }
    }
    return 0;
}

int mr3_set_exchange(mr3_ctx ctx, mr3_allgather_fn fn, void *user) {
    if (!ctx) return -1;
    ctx->xfn = fn;
    ctx->xuser = user;
    return 0;
}

int mr3_nccl_unique_id(void *id128) {
    if (!id128) return -1;
    if (!nccl_load()) return MR3_ERR_NCCL;
    ncclUniqueId id;
    if (g_nccl.GetUniqueId(&id) != ncclSuccess) return MR3_ERR_NCCL;
    memcpy(id128, &id, sizeof(id));
    return 0;
}

int mr3_nccl_comm_init(void **comm, const void *id128, int rank, int world, int device) {
    if (!comm || !id128) return -1;
    if (world < 1 || rank < 0 || rank >= world) return -3;
    if (!nccl_load()) return MR3_ERR_NCCL;
    if (cudaSetDevice(device) != cudaSuccess) return MR3_ERR_CUDA;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    if (g_nccl.CommInitRank(&c, world, id, rank) != ncclSuccess) return MR3_ERR_NCCL;
    *comm = (void *)c;
    return 0;
}

int mr3_nccl_comm_destroy(void *comm) {
    if (!comm) return 0;
    if (!nccl_load()) return MR3_ERR_NCCL;
    return g_nccl.CommDestroy((ncclComm_t)comm) == ncclSuccess ? 0 : MR3_ERR_NCCL;
}

static int solve_host_common(mr3_ctx ctx, int mode, char jobz, char range, int64_t n,
                             const void *d, const void *e, double vl, double vu, int64_t il,
                             int64_t iu, int64_t *m, void *w, void *Z, int64_t ldz, int64_t zcap,
                             int64_t *zcol_begin, int64_t *zcol_end, mr3_stats *stats) {
    if (!ctx) return -1;
    if (jobz != 'V' && jobz != 'N') return -2;
    if (range != 'A' && range != 'I' && range != 'V') return -3;
    if (n < 0) return -4;
    if (!m) return -11;
    if (n > 0 && (!d || (n > 1 && !e))) return -5;
    if (n > 0 && !w) return -12;
    if (jobz == 'V' && n > 0 && (!Z || ldz < n)) return -14;
    if (!zcol_begin || !zcol_end) return -16;
    *m = 0;
    if (n == 0) return solve_common(ctx, mode, jobz, range, n, d, e, vl, vu, il, iu, m, w, Z, ldz,
                                    zcap, zcol_begin, zcol_end, stats);
    const size_t es = mode ? 4 : 8;
    int rc = 0;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    // device columns: at most what the host Z holds (zcap) and what the solve can produce
    int64_t mcap = n;
    if (range == 'I') mcap = std::max<int64_t>(0, std::min<int64_t>(iu, n) - std::max<int64_t>(il, 1) + 1);
    mcap = std::min(mcap, std::max<int64_t>(zcap, 0));
    char *dd_ = (char *)getbuf(ctx, "host_d", (size_t)n * es, &rc);
    char *de_ = (char *)getbuf(ctx, "host_e", (size_t)std::max<int64_t>(n - 1, 1) * es, &rc);
    char *dw = (char *)getbuf(ctx, "host_w", (size_t)n * es, &rc);
    char *dZ = jobz == 'V' ? (char *)getbuf(ctx, "host_Z", (size_t)n * std::max<int64_t>(mcap, 1) * es, &rc)
                           : nullptr;
    if (rc) return rc;
    CK(cudaMemcpyAsync(dd_, d, (size_t)n * es, cudaMemcpyHostToDevice, s));
    if (n > 1) CK(cudaMemcpyAsync(de_, e, (size_t)(n - 1) * es, cudaMemcpyHostToDevice, s));
    rc = solve_common(ctx, mode, jobz, range, n, dd_, de_, vl, vu, il, iu, m, dw, dZ, n, mcap,
                      zcol_begin, zcol_end, stats);
    if (rc) return rc;
    const int64_t mm = *m, nc = *zcol_end - *zcol_begin;
    if (mm > 0) {
        CK(cudaMemcpyAsync(w, dw, (size_t)mm * es, cudaMemcpyDeviceToHost, s));
        if (jobz == 'V' && nc > 0)
            CK(cudaMemcpy2DAsync(Z, (size_t)ldz * es, dZ, (size_t)n * es, (size_t)n * es, (size_t)nc,
                                 cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s)); hsync_note(ctx, "sync#17");
    return 0;
}

int mr3_dstemr_dd_host(mr3_ctx ctx, char jobz, char range, int64_t n, const double *d,
                       const double *e, double vl, double vu, int64_t il, int64_t iu, int64_t *m,
                       double *w, double *Z, int64_t ldz, int64_t zcap, int64_t *zcol_begin,
                       int64_t *zcol_end, mr3_stats *stats) {
    return solve_host_common(ctx, 0, jobz, range, n, d, e, vl, vu, il, iu, m, w, Z, ldz, zcap,
                             zcol_begin, zcol_end, stats);
}

int mr3_sstemr_d_host(mr3_ctx ctx, char jobz, char range, int64_t n, const float *d,
                      const float *e, float vl, float vu, int64_t il, int64_t iu, int64_t *m,
                      float *w, float *Z, int64_t ldz, int64_t zcap, int64_t *zcol_begin,
                      int64_t *zcol_end, mr3_stats *stats) {
    return solve_host_common(ctx, 1, jobz, range, n, d, e, vl, vu, il, iu, m, w, Z, ldz, zcap,
                             zcol_begin, zcol_end, stats);
}

int mr3_partition_columns(int64_t nseg, const int64_t *seg_begin, const double *cost, int world,
                          int64_t *col_begin) {
    if (world < 1 || nseg < 0 || !seg_begin || !col_begin || (nseg > 0 && !cost)) return -1;
    const int64_t m = seg_begin[nseg];
    double total = 0;
    for (int64_t i = 0; i < nseg; i++) total += cost[i];
    col_begin[0] = 0;
    int r = 1;
    double acc = 0;
    for (int64_t i = 0; i < nseg && r < world; i++) {
        acc += cost[i];
        // cut after segment i once this rank's share is reached
        while (r < world && acc >= total * r / world) {
            col_begin[r] = (i + 1 < nseg) ? seg_begin[i + 1] : m;
            r++;
        }
    }
    for (; r < world; r++) col_begin[r] = m;
    col_begin[world] = m;
    for (int i = 1; i <= world; i++)
        if (col_begin[i] < col_begin[i - 1]) col_begin[i] = col_begin[i - 1];
    return 0;
}

int mr3_fp64_peak(mr3_ctx ctx, double *fp64_inst_per_s, double *dd_step_ns) {
    if (!ctx) return -1;
    cudaSetDevice(ctx->device);
    int rc = 0;
    double *out = (double *)getbuf(ctx, "peak_out", 64, &rc);
    double *rep = (double *)getbuf(ctx, "peak_rep", 4096 * 64, &rc);
    if (rc) return rc;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096, grid = ctx->nsm * 8, tpb = 256;
    k_fp64_peak<<<grid, tpb, 0, ctx->stream>>>(out, 64, 1.0000001, 1e-9);  // warm-up
    cudaEventRecord(a, ctx->stream);
    k_fp64_peak<<<grid, tpb, 0, ctx->stream>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(b, ctx->stream);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (fp64_inst_per_s)
        *fp64_inst_per_s = (double)grid * tpb * iters * 64.0 / (ms * 1e-3);
    k_fill_rep_test<<<16, 256, 0, ctx->stream>>>(rep, 4096);
    int *ic = (int *)out;
    const int reps = 8;
    k_dd_latency<<<1, 1, 0, ctx->stream>>>(rep, 4096, 1, ic);
    cudaEventRecord(a, ctx->stream);
    k_dd_latency<<<1, 1, 0, ctx->stream>>>(rep, 4096, reps, ic);
    cudaEventRecord(b, ctx->stream);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (dd_step_ns) *dd_step_ns = ms * 1e6 / (4096.0 * reps);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        ctx->err = cudaGetErrorString(e);
        return MR3_ERR_CUDA;
    }
    return 0;
}

int mr3_last_kernel_times(mr3_ctx ctx, int *count, const char **names, double *ms,
                          int *launches) {
    if (!ctx || !count) return -1;
    int c = 0;
    for (auto &p : ctx->ktimes) {
        if (c >= 16) break;
        if (names) names[c] = p.first.c_str();
        if (ms) ms[c] = p.second.first;
        if (launches) launches[c] = p.second.second;
        c++;
    }
    *count = c;
    return 0;
}

int64_t mr3_last_launch_count(mr3_ctx ctx) { return ctx ? ctx->launches : 0; }

const char *mr3_strerror(int code) {
    switch (code) {
        case 0:
            return "ok";
        case MR3_ERR_NONFINITE:
            return "NaN or Inf in d or e";
        case MR3_ERR_CUDA:
            return "CUDA error";
        case MR3_ERR_NCCL:
            return "collective (NCCL / exchange) error";
        case MR3_ERR_NOMEM:
            return "device allocation failed";
        case MR3_ERR_NOCONV:
            return "no convergence";
        case MR3_ERR_ZCAP:
            return "Z has too few columns";
        case MR3_ERR_STATE:
            return "execute without plan";
        default:
            return code < 0 ? "invalid argument" : "unknown error";
    }
}

const char *mr3_last_error_string(mr3_ctx ctx) { return ctx ? ctx->err.c_str() : ""; }

const char *mr3_version(void) {
    return "mr3-b200 sm_100a; dd (fp64 I/O) and fp64 (fp32 I/O) internal precision";
}

}  // extern "C"
