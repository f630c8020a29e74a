/*
 * mr3.h -- C-ABI of the B200-native mixed-precision MRRR hot path.
 *
 * Operation (§1 "the real symmetric tridiagonal eigenproblem
 * (STEP)", and Algorithm 1): given T = tridiag(e, d, e) with d[n],
 * e[n-1] and an index range il..iu or a value range (vl, vu], compute eigenvalues
 * w (ascending) and unit eigenvectors Z with T z = lambda z.  Input and output
 * are in binary_x (fp64 or fp32); all per-eigenpair work runs in binary_y
 * (double-double resp. fp64) -- the mixed-precision approach of §3
 * (L746-L1197) with the parameters of §4 (L1291-L1326).
 *
 * Conventions (all calls):
 *  - Pointers named d_*, w, Z and the `d`, `e` inputs are DEVICE pointers
 *    (e.g. PyTorch CUDA tensors), caller-allocated and caller-owned.  Inputs are
 *    never modified; outputs must not alias inputs.
 *  - Z is column-major with leading dimension ldz >= n; column j holds the
 *    eigenvector of w[j].  Each column is fully written (zeros outside the
 *    eigenvector's irreducible block).
 *  - Calls are stream-ordered on the context's stream and synchronous on return
 *    (the call waits for its own work).  A context is not thread-safe.
 *  - Return codes (LAPACK-like): 0 OK; -k: argument k invalid; positive codes
 *    MR3_ERR_* below.  On error the outputs are undefined and *stats is filled as
 *    far as the solve got.  n = 0 returns OK with *m = 0.
 *  - Results are bitwise deterministic for given (d, e, range, params) and do not
 *    depend on the number of ranks of the two-phase multi-GPU form.
 *  - The library owns its scratch (stream-ordered allocations, cached in the
 *    context, released by mr3_destroy).  Z is never used as workspace
 *    (§3.3).
 */
#ifndef MR3_H
#define MR3_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mr3_ctx_s *mr3_ctx;

/* error codes (positive) */
#define MR3_OK 0
#define MR3_ERR_NONFINITE 1 /* NaN or Inf in d or e */
#define MR3_ERR_CUDA 2      /* a CUDA runtime error (mr3_last_error_string) */
#define MR3_ERR_NCCL 3      /* a collective failed (NCCL error, exchange callback error, or
                               world > 1 with neither a communicator nor a callback) */
#define MR3_ERR_NOMEM 4     /* device allocation failed */
#define MR3_ERR_NOCONV 5    /* reserved: the fallbacks are total */
#define MR3_ERR_ZCAP 6      /* two-phase form: Z has fewer columns than needed */
#define MR3_ERR_STATE 7     /* two-phase form: execute without a matching plan */

#define MR3_BRK_REC 6 /* doubles per bracket record of the two-phase form (mr3_plan) */

/*
 * Statistics of one solve (PAPER.md L425 d_max, L961 rho).
 * t_ms: device time per phase {root, bisect, classify, child, rqi, total, -, -}.
 */
typedef struct {
    int32_t d_max;               /* depth of the representation tree (L425) */
    int32_t n_clusters;          /* clusters processed, all levels */
    int32_t largest_cluster;     /* largest cluster size; rho = largest/n (L961) */
    int32_t robustness_failures; /* child RRR accepted without passing the test (L567-L572) */
    int32_t rqi_fallbacks;       /* RQI -> bisection + one solve (L724-L727, L1154-L1163) */
    int32_t n_blocks;            /* irreducible blocks after splitting (L862-L876) */
    int32_t rqi_iters_max;       /* most RQI iterations any eigenpair took */
    int32_t levels;              /* tree levels processed (d_max + 1 when m > 0) */
    double rho;                  /* clustering: largest cluster / n, in [1/n, 1] */
    double bisect_rows;          /* Sturm-count rows executed (dstqds steps) */
    double rqi_rows;             /* twisted-factorisation rows executed */
    double bisect_rows_x;        /* Sturm-count rows executed in binary_x (fp64 phase) */
    double newton_rows_x;        /* of which Newton passes (count + derivative, R8e) */
    double t_ms[8];
    int32_t backtracks;          /* clusters whose child came from the grandparent (R22) */
    int32_t backtrack_tries;     /* clusters re-processed from the grandparent */
} mr3_stats;

/* tunable parameters (mr3_set_param / mr3_get_param); defaults per PAPER.md §4 */
enum mr3_param {
    MR3_GAPTOL = 0,    /* classification gaptol; default 1e-10 (dd, L1325) / 1e-5 (fp64, L1293) */
    MR3_XI = 1,        /* root perturbation xi; default eps_x (L906-L909) */
    MR3_KRS = 2,       /* RQI stopping constant k_rs; default 1 (L1150) */
    MR3_MAX_RQI = 3,   /* RQI iterations before the bisection fallback; default 10 */
    MR3_MAX_DEPTH = 4, /* representation-tree depth cap; default 10 */
    MR3_SEED = 5,      /* perturbation seed (counter-based generator key); default 0x4D5233 */
    MR3_ELG_MAX = 6,   /* element-growth acceptance k_elg (first pass); default 8 */
    MR3_RTOL = 7,      /* bisection relative tolerance; default 1e-2 * gaptol (L1294-L1295) */
    MR3_GROUPS = 8,    /* lanes per eigenvalue in the multisection (0 = automatic) */
    MR3_XPHASE = 9,    /* fp64 I/O: approximate eigenvalues in binary_x first (L1064-L1111); 1 */
    MR3_REFINE = 10,   /* RQI start refinement constant C (0 = off): singletons whose bracket
                          half-width exceeds gap*sqrt(eps_x sqrt(n)/C) get a binary_x start; 4 */
    MR3_GRID = 11,     /* 0: no shared grid; 1: uniform grid + 3 adaptive levels (k_grid);
                          v >= 2: v - 2 adaptive levels; 1 */
    MR3_CTA = 12,      /* threads per CTA of the staged kernels, 32..128 (0 = 128) */
    MR3_XPTS = 13,     /* binary_x root phase: 1 bisection / multisection, 2 two points per lane,
                          3 Newton-accelerated bisection (G = 1; R8e); 3 */
    MR3_YCERT = 14,    /* 1: certify the root brackets of the binary_x phase by binary_y Sturm
                          counts; 0: rigorous widening by the definite root's relative
                          robustness bound instead (R8d); 0 */
    MR3_NEWTON = 15,   /* Newton passes per item before the many-lane multisection tail; 6 */
    MR3_TWISTW = 16,   /* twist weight slope w: r = argmin |gamma_k| (1 + w |2k - n| / n); 100 */
    MR3_SPLIT = 17,    /* split (chunked) RQI passes, reading R9d: 0 none, 1 iterations >= 3,
                          2 also every iteration of small sets (one eigenpair per CTA); 1 */
    MR3_FUSE_SCALE = 18, /* 1: every RQI CTA normalises its own Z columns when it is done;
                            0: one k_zscale launch after the RQI phase (same arithmetic); 1 */
    MR3_POOL_MB = 19,  /* budget for the child representations of one batch of clusters, MB
                          (0 = automatic: min(8 GB, 15% of free memory)); clusters beyond it are
                          processed in depth-first batches */
    MR3_DEBUG = 20,    /* diagnostics to stderr: bit 1 dumps/histograms, 2 host sync points,
                          4 device timeline, 8 check every launch; 0 */
    MR3_RQI_FB = 21,   /* 1: RQI iterations 1-2 with the two halves of every factorization in
                          two threads (k_rqi_fb), later iterations in k_rqi; 2: the same with the
                          row update in two-dot-product form (shorter dependent chain);
                          0: all in k_rqi; 1 */
    MR3_RQI_CHUNK = 22, /* solves of at most this many wanted eigenpairs (globally) run every
                           RQI iteration chunk-parallel, one eigenpair per CTA (k_rqi_chunk;
                           it also takes the stragglers of k_rqi_fb); 0 = off; 8192 */
    MR3_RELAX = 23,    /* NEXT-1b: bisection of an eigenvalue whose own
                          Sturm counts isolate it by gaps >= 4 gaptol |lambda| stops once its
                          bracket is narrower than c gap sqrt(eps_x sqrt(n) / C) (C = MR3_REFINE),
                          c = this value, instead of going to rtol (R20); 0 = off; 0.5 */
    MR3_ABSGAP = 24,   /* absolute-gap splitting: neighbours
                          whose bracket gap is >= this value * ||T||_1 are separated even when
                          their relative gap is below gaptol (R21); 0 = off */
    MR3_BACKTRACK = 25, /* 1: a child at depth >= 2 that fails the acceptance tests is redone
                           from its grandparent and kept if it passes or grows less (PAPER.md
                           L1190-L1197, R22); 0: off; 2: test hook (every child at
                           depth >= 2 counts as failed first); 1 */
    MR3_NPARAM = 26
};

/*
 * One context per (device, stream, rank).
 *   cuda_stream: the cudaStream_t all work is ordered on (cudaStreamLegacy = (void *)1 for the
 *                legacy default stream); NULL = a non-blocking stream owned by the context,
 *                which is NOT ordered after the caller's other work -- the caller must
 *                synchronise its inputs first.
 *   nccl_comm:   an ncclComm_t spanning `world` ranks (one GPU each; this process is `rank`)
 *                or NULL.  With world > 1 the one-call solvers below exchange the bracket
 *                records and the eigenvalues with ncclAllGather on it (NCCL is loaded
 *                lazily, libnccl.so.2, the first time a communicator is used), unless an
 *                exchange callback is installed (mr3_set_exchange).  world = 1: single GPU.
 * Errors: -1 ctx NULL, -5 rank/world invalid, MR3_ERR_CUDA.
 */
int mr3_create(mr3_ctx *ctx, int device, void *cuda_stream, void *nccl_comm, int rank, int world);
int mr3_destroy(mr3_ctx ctx);
/* mode 0: fp64 I/O (double-double internal), mode 1: fp32 I/O (fp64 internal).
 * Parameters are stored per mode; a negative value restores the default. */
int mr3_set_param(mr3_ctx ctx, int mode, int which, double value);
double mr3_get_param(mr3_ctx ctx, int mode, int which);

/*
 * In-place all-gather used by the one-call solvers when world > 1 (instead of NCCL): buf is a
 * DEVICE buffer of world slices of bytes_per_rank bytes; this rank's slice (offset
 * rank * bytes_per_rank) is valid on entry, all slices on return.  Work before the call is
 * ordered on `stream` (cudaStream_t); the callback must leave buf complete in stream order
 * (e.g. synchronise, copy through the host, or enqueue its own collective).  Returns 0 or
 * nonzero (-> MR3_ERR_NCCL).  fn = NULL removes the callback.
 */
typedef int (*mr3_allgather_fn)(void *user, void *buf, size_t bytes_per_rank, int rank, int world,
                                void *stream);
int mr3_set_exchange(mr3_ctx ctx, mr3_allgather_fn fn, void *user);

/* NCCL helpers (libnccl.so.2 loaded lazily): a unique id (128 bytes, rank 0 creates it and
 * the caller broadcasts it), a communicator of `world` ranks on `device`, and its release.
 * Return 0 or MR3_ERR_NCCL. */
int mr3_nccl_unique_id(void *id128);
int mr3_nccl_comm_init(void **comm, const void *id128, int rank, int world, int device);
int mr3_nccl_comm_destroy(void *comm);

/*
 * fp64 I/O, double-double internal (the "double/quadruple" solver of L1318-L1326).
 *   jobz : 'V' eigenvalues and eigenvectors, 'N' eigenvalues only
 *   range: 'A' all; 'I' indices il..iu (1-based, inclusive); 'V' vl < lambda <= vu
 *   d[n], e[n-1]: device inputs (the same on every rank).
 *   *m: number of eigenvalues found (globally).
 *   w[n]: device output, the first *m entries ascending -- all of them on every rank.
 *   (A matrix that splits into blocks gets its columns from the order of the blocks'
 *   bisection estimates; after the eigenpairs are final, w is sorted stably and the Z columns
 *   are permuted with it, over this rank's column range.  With world > 1 two eigenvalues of
 *   different blocks that agree to within the bisection tolerance may therefore still be
 *   exchanged across a rank boundary; with world = 1 w is ascending without exception.)
 *   Z: device output, column-major, ldz >= n, zcap columns allocated (may be NULL when
 *   jobz = 'N'): this rank's columns [*zcol_begin, *zcol_end) of the global m, at local
 *   positions 0 .. *zcol_end - *zcol_begin - 1.  Single GPU (world = 1): all m columns.
 *   With world > 1 the index set is partitioned over the ranks of the context (SURVEY.md
 *   8(e): replicated root, static-slice bisection, all-gather of the bracket records,
 *   identical classification, cluster-whole column ranges, all-gather of w); zcap below the
 *   rank's column count returns MR3_ERR_ZCAP with the range filled in (size Z from it, or
 *   use the two-phase form mr3_plan / mr3_execute).
 */
int mr3_dstemr_dd(mr3_ctx ctx, char jobz, char range, int64_t n, const double *d, const double *e,
                  double vl, double vu, int64_t il, int64_t iu, int64_t *m, double *w, double *Z,
                  int64_t ldz, int64_t zcap, int64_t *zcol_begin, int64_t *zcol_end,
                  mr3_stats *stats);

/* fp32 I/O, fp64 internal (the "single/double" solver of L1291-L1304); same contract. */
int mr3_sstemr_d(mr3_ctx ctx, char jobz, char range, int64_t n, const float *d, const float *e,
                 float vl, float vu, int64_t il, int64_t iu, int64_t *m, float *w, float *Z,
                 int64_t ldz, int64_t zcap, int64_t *zcol_begin, int64_t *zcol_end,
                 mr3_stats *stats);

/*
 * Dense symmetric eigenproblem, fp64 I/O (Fig. 3):
 * reduction A = Q T Q^T by Householder reflectors (LAPACK dsytrd's lower storage), the
 * tridiagonal eigenpairs of T by mr3_dstemr_dd (double-double internal), Z <- Q Z.
 *   A: device, column-major n x n, lda >= n; both triangles must hold the symmetric matrix
 *      (only the reduction's updates are read); OVERWRITTEN: on return the diagonal and
 *      subdiagonal hold T's d and e, the reflectors v_j (v_j(j+1) = 1 implicit) lie below the
 *      subdiagonal, the strict upper triangle holds reduction intermediates.
 *   jobz, range, vl, vu, il, iu, *m, w: as mr3_dstemr_dd.
 *   Z: device, column-major, ldz >= n, >= *m columns (may be NULL when jobz = 'N'): the
 *      eigenvectors of A.
 *   stats: as mr3_dstemr_dd's, plus t_ms[6] = reduction ms, t_ms[7] = back-transformation ms.
 * Single-rank contexts only (world = 1, else MR3_ERR_STATE).  The back-transformation's GEMMs
 * are cuBLAS (libcublas.so.12, loaded on first use; missing -> MR3_ERR_CUDA).
 * n <= 8192 (the reduction's column step keeps a column in the registers of one CTA).
 * Errors: -1 ctx NULL, -2 jobz, -3 range, -4 n < 0 or n > 8192, -5 A NULL, -6 lda, -11 m NULL, -12 w NULL,
 * -13 Z NULL or ldz < n, the errors of mr3_dstemr_dd, MR3_ERR_CUDA, MR3_ERR_NOMEM.
 */
int mr3_dsyevr_dd(mr3_ctx ctx, char jobz, char range, int64_t n, double *A, int64_t lda,
                  double vl, double vu, int64_t il, int64_t iu, int64_t *m, double *w, double *Z,
                  int64_t ldz, mr3_stats *stats);

/*
 * End-to-end forms with HOST buffers (same contract as mr3_dstemr_dd /
 * mr3_sstemr_d otherwise): d[n], e[n-1] are read from host memory, w[n] and Z
 * (column-major, ldz >= n, >= *m columns; may be NULL when jobz = 'N') are
 * written to host memory.  The host<->device copies run on the context's stream
 * inside the call (pinned host memory -- cudaHostAlloc / cudaHostRegister / a
 * pinned torch tensor -- gives full PCIe bandwidth; pageable memory works but is
 * staged by the driver).  Device copies of the inputs and outputs are library
 * scratch (cached in the context, released by mr3_destroy).
 */
int mr3_dstemr_dd_host(mr3_ctx ctx, char jobz, char range, int64_t n, const double *d,
                       const double *e, double vl, double vu, int64_t il, int64_t iu, int64_t *m,
                       double *w, double *Z, int64_t ldz, int64_t zcap, int64_t *zcol_begin,
                       int64_t *zcol_end, mr3_stats *stats);
int mr3_sstemr_d_host(mr3_ctx ctx, char jobz, char range, int64_t n, const float *d,
                      const float *e, float vl, float vu, int64_t il, int64_t iu, int64_t *m,
                      float *w, float *Z, int64_t ldz, int64_t zcap, int64_t *zcol_begin,
                      int64_t *zcol_end, mr3_stats *stats);

/*
 * Two-phase form for an index-set partition over `world` ranks (one GPU each).
 *
 * mr3_plan: root representation (replicated), the requested index set, and
 * bisection of this rank's static slice of it.  Returns in *brk a DEVICE buffer
 * of world * slice_cap records of MR3_BRK_REC doubles (bracket lo.hi, lo.lo, hi.hi,
 * hi.lo in root coordinates, then the binary_x Newton estimate of the eigenvalue and
 * the size of its last step, NaN / INF if none) of which this rank filled records
 * [rank*slice_cap, rank*slice_cap + slice_cnt); the caller must all-gather it in
 * place (equal-size slices, e.g. ncclAllGather / torch.distributed) before
 * mr3_execute.  The buffer stays owned by the context.
 *
 * mr3_execute: classification of the whole index set (identical on all ranks),
 * cluster-whole partition of the output columns, then child representations,
 * refinement and eigenvectors for this rank's columns [*zcol_begin, *zcol_end).
 * w receives the eigenvalues of this rank's columns at their global positions
 * (w[*zcol_begin .. *zcol_end-1]); Z receives those columns at local positions
 * 0 .. (*zcol_end - *zcol_begin - 1).  zcap: columns allocated in Z; if too
 * small MR3_ERR_ZCAP is returned with the range filled in.
 * mode: 0 = fp64 I/O (w, Z double*), 1 = fp32 I/O (w, Z float*).
 */
int mr3_plan(mr3_ctx ctx, int mode, char range, int64_t n, const void *d, const void *e, double vl,
             double vu, int64_t il, int64_t iu, int rank, int world, int64_t *m,
             double **brk, int64_t *slice_cap, int64_t *slice_cnt);
int mr3_execute(mr3_ctx ctx, char jobz, void *w, void *Z, int64_t ldz, int64_t zcap,
                int64_t *zcol_begin, int64_t *zcol_end, mr3_stats *stats);

/*
 * Host-only helper (no device work; callable without a GPU): split m output
 * columns over `world` ranks at cluster boundaries.  seg_begin[0..nseg] are the
 * column offsets where the tree's top-level nodes (singletons and clusters)
 * start (seg_begin[nseg] = m); cost[s] the work estimate of node s.  Fills
 * col_begin[0..world] (col_begin[0] = 0, col_begin[world] = m), balancing cost
 * greedily and never cutting a node.  Returns 0 or -1 on bad arguments.
 */
int mr3_partition_columns(int64_t nseg, const int64_t *seg_begin, const double *cost, int world,
                          int64_t *col_begin);

/*
 * Same-run FP64 peak microbenchmark (K7): independent DFMA chains on every SM
 * (-> *fp64_inst_per_s, FP64 instructions per second) and one dependent chain of
 * double-double Sturm steps (-> *dd_step_ns, latency of one step).
 */
int mr3_fp64_peak(mr3_ctx ctx, double *fp64_inst_per_s, double *dd_step_ns);

/* per-kernel device time of the last solve (CUDA events on the context stream):
 * names[i], total ms[i] and launches[i] for i < *count (max 16); any output may be NULL */
int mr3_last_kernel_times(mr3_ctx ctx, int *count, const char **names, double *ms, int *launches);
/* number of kernel launches issued by the last plan + execute */
int64_t mr3_last_launch_count(mr3_ctx ctx);

const char *mr3_strerror(int code);
const char *mr3_last_error_string(mr3_ctx ctx);
/* library build info: "sm_100a ..." */
const char *mr3_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MR3_H */
