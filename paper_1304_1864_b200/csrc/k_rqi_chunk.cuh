// k_rqi_chunk.cuh -- K5 for small index sets (and the stragglers of k_rqi_fb): every RQI
// iteration of ONE eigenpair as a chunk-parallel fixed-twist factorization over a CTA
// (Alg. 1 l.11-12; the parallel evaluation of reading R9d).
//
// With few eigenpairs the serial n-row chains of k_rqi_fb leave the GPU idle: 2 000
// eigenpairs of n = 20 000 (config 4) are 4 000 chains, one warp on a quarter of the SMs.
// Here the CTA of one eigenpair cuts the F rows [0, r) and the B rows (r, n) into T chunks
// (T = blockDim.x, proportional to the two lengths).  The projective transforms are linear
// in the state (p, q) (reading R8b):
//   F row k: (p, q) -> (lld_k p - lam (d_k q + p), d_k q + p)
//   B row k: (p, q) -> (d_{k-1} p - lam (lld_{k-1} q + p), lld_{k-1} q + p)
// so (1) every thread forms its chunk's 2x2 transfer matrix from two basis solutions (two
// independent chains), (2) one thread per direction chains the matrices into the chunk start
// states, (3) every thread re-runs the true recurrence from its start state: the product-form
// z components (k_zprod.cuh) written to Z, compensated sums of their squares, the inertia.
// The re-run end state of a chunk and the next chunk's start differ by the rounding of the
// chained products; that jump perturbs the recurrence at the boundary row, adding about
// delta |z_k| ||row_k|| to the residual -- summed per direction and required to stay below
// tol / 8 (and delta below 2^-50 in pair arithmetic, 2^-20 in binary64), else the eigenpair
// is handed to k_rqi (serial passes) from its current state.  Chain length ~ 3 n / T rows
// per pass instead of n / 2; about 3x the arithmetic of the serial pass.
// The iteration logic (RQ correction, Eq. (3.6) stop, stagnation, bracket guard) is k_rqi's,
// run by thread 0.  After max_rqi iterations the eigenpair goes to k_rqi's bisection
// fallback (RqiResume).  Finished columns are normalised by the CTA (k_rqi's fused epilogue).
#pragma once
#include "k_rqi_fb.cuh"

namespace mr3 {

constexpr int RC_TPB = 128;  // max threads per CTA (blockDim.x in {32, 64, 128})

template <class R>
struct ChunkIO {  // pass inputs (thread 0 writes) and outputs (reductions)
    R lam;
    R sr, pr;   // s_r = pF/qF at r (F end), p_r (B end)
    int64_t r;
    int erefF, erefB, wz, need;
    int negc, bad, eyr, exr;
    double yr, xr, sF, cF, sB, cB, jF, jB;
};

// the data one direction needs from a row: F row k: m1 = d_k, m2 = lld_k, x = ld_k (for
// l+ = ld / d+); B row k (data of row k - 1): m1 = lld, m2 = d, x = l d (for u- = l d / D-)
template <class R>
struct RowFB {
    R m1, m2;
    double x, nrm;  // (nrm: |d| + |lld| + 2 |ld|, the row's contribution to ||M||)
};
template <class R>
__device__ __forceinline__ RowFB<R> load_fb(const double *__restrict__ rep, int64_t row, bool isF) {
    const Row4<R> rw = load_row4<R>(rep, row);
    RowFB<R> o;
    o.m1 = isF ? rw.d : rw.lld;
    o.m2 = isF ? rw.lld : rw.d;
    o.x = hi(rw.ld);  // l+ = ld qF / qF' (F), u- = ld QB / QB' (B)
    o.nrm = fabs(hi(rw.d)) + fabs(hi(rw.lld)) + 2.0 * fabs(hi(rw.ld));
    return o;
}

constexpr int RC_U = 4;  // rows loaded ahead (one batch)
// phase-3 rounds (see chunk_pass): measured on glued Wilkinson children (config 3) the
// correction rounds do not shrink the jumps (the chunk products are ill-conditioned, not
// merely inexact), so one round; the eigenpairs whose jumps fail the test go to serial passes
constexpr int RC_ROUNDS = 1;

template <class R, class OutT>
__global__ void __launch_bounds__(RC_TPB) k_rqi_chunk(RqiArgs<R> A) {
    const int T = blockDim.x;
    const int tid = threadIdx.x;
    __shared__ R Mx[4 * RC_TPB];  // transfer matrices: u = M (1, 0), v = M (0, 1)
    __shared__ R Sx[2 * RC_TPB];  // chunk start states
    __shared__ int ME[RC_TPB], SE[RC_TPB];
    __shared__ R Ex[2 * RC_TPB];  // chunk end states of a phase-3 round
    __shared__ int EEx[RC_TPB];
    __shared__ double s_red[RC_TPB / 32][6];
    __shared__ int s_redi[RC_TPB / 32][2];
    __shared__ double sA[RC_TPB], sB[RC_TPB];  // per chunk: affine map W -> A W + B of the norms
    __shared__ ChunkIO<R> io;
    __shared__ ZCol s_zc;
    __shared__ double nzW, nzV;
    __shared__ int s_lrel;  // (MR3_DEBUG) worst continuity of the pass, 16 log2 + 32768

    const int pos = blockIdx.x;  // position in the list (one eigenpair per CTA)
    const int id = A.list[pos];
    const NodeInfo nd = A.nodes[A.it.node[id]];
    const int64_t n = nd.n;
    // ---- owner state (thread 0)
    int k = 0;
    R lam = mk<R>(0.0), a = lam, b = lam, gr = lam, lam_out = lam;
    double nz2 = 1.0, gap = INFINITY, tol = 0.0;
    int64_t r = 0;
    unsigned long long rows = 0;
    bool done = false, zfinal = false, zwritten = false, handoff = false;
    int erefF = 0, erefB = 0, passes = 0;
    const int64_t col0 = A.it.col[id];
    OutT *zcol = (A.jobz_v && col0 >= 0)
                     ? reinterpret_cast<OutT *>(A.Z) + nd.row0 + (col0 - A.zcol0) * A.ldz
                     : nullptr;
    ZCol zinfo;
    zinfo.row0 = nd.row0;
    zinfo.n = (int32_t)n;
    zinfo.cF = 1.0;
    zinfo.cB = 1.0;
    zinfo.ss = 1.0;
    if (tid == 0) {
        k = A.it.k[id];
        a = reinterpret_cast<const R *>(A.it.lo)[id];
        b = reinterpret_cast<const R *>(A.it.hi)[id];
        lam = half(add(a, b));
        if (A.root_widen > 0.0 && nd.depth == 0) {  // rigorous guard of a root bracket (R8d)
            const double wd = A.root_widen * (double)n * fmax(fabs(hi(a)), fabs(hi(b)));
            a = sub(a, mk<R>(wd));
            b = add(b, mk<R>(wd));
        }
        const double x0 = A.it.x0[id];
        if (!isnan(x0) && lt(a, mk<R>(x0)) && lt(mk<R>(x0), b)) lam = mk<R>(x0);
        gap = fmin(A.it.lgap[id], A.it.rgap[id]);
        if (!(gap > 0.0)) gap = fmax(hi(sub(b, a)), 1e-300);
        r = A.it.twist[id];
        if (r < 0 || r >= n) r = n - 1;
        tol = A.krs * gap * A.eps_x * sqrt((double)n);
        if (A.resume_in != nullptr) {  // a straggler of k_rqi_fb: continue from its state
            const RqiResume<R> rs = A.resume_in[id];
            lam = rs.lam;
            a = rs.a;
            b = rs.b;
            lam_out = rs.lam_out;
            erefF = rs.erefF;
            erefB = rs.erefB;
            done = (rs.flags & 1) != 0;
            zfinal = (rs.flags & 2) != 0;
            passes = rs.iters;
        }
        zinfo.r = (int32_t)r;
        if (n == 1) {  // 1x1 block: (d_1, e_1)
            lam_out = load_row4<R>(nd.rep, 0).d;
            done = true;
            if (zcol != nullptr) zcol[0] = (OutT)1.0;
            zfinal = true;
        }
    }

    // ---- one chunk-parallel fixed-twist factorization at io.lam (collective)
    auto chunk_pass = [&]() {
        const R lam_s = io.lam, mlam = neg(io.lam);
        const int64_t rs = io.r;
        OutT *zc = io.wz ? zcol : nullptr;
        const int64_t LF = rs, LB = n - 1 - rs;
        int tF = (LF + LB) > 0 ? (int)((T * LF + (LF + LB) / 2) / (LF + LB)) : 0;
        if (LF > 0 && tF < 1) tF = 1;
        if (LB > 0 && tF > T - 1) tF = T - 1;
        if (LB == 0) tF = T;
        if (LF == 0) tF = 0;
        const int tB = T - tF;
        const bool isF = tid < tF;
        const int c = isF ? tid : tid - tF, nc = isF ? tF : tB;
        // F: rows k0 .. k1-1 ascending; B: rows k0 .. k1+1 descending
        const int64_t k0 = isF ? LF * c / nc : n - 1 - LB * c / nc;
        const int64_t k1 = isF ? LF * (c + 1) / nc : n - 1 - LB * (c + 1) / nc;
        const int64_t len = isF ? k1 - k0 : k0 - k1;
        // phase 1: transfer matrix of the chunk (two basis solutions)
        {
            R up = mk<R>(1.0), uq = mk<R>(0.0), vp = mk<R>(0.0), vq = mk<R>(1.0);
            int EM = 0;
#pragma unroll 1
            for (int64_t j0 = 0; j0 < len; j0 += RC_U) {
                const int jn = (int)min((int64_t)RC_U, len - j0);
                R m1v[RC_U], m2v[RC_U];
#pragma unroll
                for (int j = 0; j < RC_U; j++)  // loads first: RC_U rows in flight
                    if (j < jn) {
                        const int64_t kk = isF ? k0 + j0 + j : k0 - j0 - j;
                        const RowFB<R> rw = load_fb<R>(nd.rep, isF ? kk : kk - 1, isF);
                        m1v[j] = rw.m1;
                        m2v[j] = rw.m2;
                    }
#pragma unroll
                for (int j = 0; j < RC_U; j++)
                    if (j < jn) {
                        const R U = fma_dd(m1v[j], uq, up), V = fma_dd(m1v[j], vq, vp);
                        up = dot2_dd(mlam, U, m2v[j], up);
                        vp = dot2_dd(mlam, V, m2v[j], vp);
                        uq = U;
                        vq = V;
                    }
                unsigned em = (unsigned)__double2hiint(hi(up)) & 0x7ff00000u, t2;
                t2 = (unsigned)__double2hiint(hi(uq)) & 0x7ff00000u;
                em = t2 > em ? t2 : em;
                t2 = (unsigned)__double2hiint(hi(vp)) & 0x7ff00000u;
                em = t2 > em ? t2 : em;
                t2 = (unsigned)__double2hiint(hi(vq)) & 0x7ff00000u;
                em = t2 > em ? t2 : em;
                if (em != 0x7ff00000u && em != 0u) {
                    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                    up = scale_pow2(up, sc);
                    uq = scale_pow2(uq, sc);
                    vp = scale_pow2(vp, sc);
                    vq = scale_pow2(vq, sc);
                    EM += (int)(em >> 20) - 1023;
                }
            }
            Mx[4 * tid] = up;
            Mx[4 * tid + 1] = uq;
            Mx[4 * tid + 2] = vp;
            Mx[4 * tid + 3] = vq;
            ME[tid] = EM;
        }
        __syncthreads();
        // phase 2: chunk start states, chained by one thread per direction
        if ((tid == 0 && tF > 0) || (tid == tF && tB > 0)) {
            R p = isF ? mlam : sub(load_row4<R>(nd.rep, n - 1).d, lam_s), q = mk<R>(1.0);
            int E = 0;
#pragma unroll 1
            for (int j = 0; j < nc; j++) {
                const int t = tid + j;
                Sx[2 * t] = p;
                Sx[2 * t + 1] = q;
                SE[t] = E;
                const R np = add(mul(p, Mx[4 * t]), mul(q, Mx[4 * t + 2]));
                const R nq = add(mul(p, Mx[4 * t + 1]), mul(q, Mx[4 * t + 3]));
                p = np;
                q = nq;
                E += ME[t];
                const unsigned ex = (unsigned)__double2hiint(hi(p)) & 0x7ff00000u;
                const unsigned ey = (unsigned)__double2hiint(hi(q)) & 0x7ff00000u;
                const unsigned em = ex > ey ? ex : ey;
                if (em != 0x7ff00000u && em != 0u) {
                    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                    p = scale_pow2(p, sc);
                    q = scale_pow2(q, sc);
                    E += (int)(em >> 20) - 1023;
                }
            }
        }
        __syncthreads();
        // phase 3 in rounds: round 0 starts every chunk from the chained start state; a round
        // whose chunk-boundary jumps are not negligible (2^-95 relative in pair arithmetic,
        // 2^-45 in binary64) is followed by one that starts each chunk from the previous
        // chunk's re-run end state (a parareal-style correction: exact after as many rounds as
        // chunks, the jumps shrink geometrically where the recurrence forgets its start state);
        // at most RC_ROUNDS rounds
        R p, q;
        int E;
        double s, cmp, Am, Bm, zlast, rnorm, jres;
        int ng, bad;
        const double rel_tight = Prec<R>::words == 2 ? 0x1p-95 : 0x1p-45;
        (void)rel_tight;
#pragma unroll 1
        for (int round = 0;; round++) {
            // phase 3: the true recurrence from the start state: z components (storing pass),
            // the prefix-norm map (W_{k+1} = l+_k^2 (1 + W_k), V likewise with u-, reading R9) of
            // the chunk as an affine map W -> Am W + Bm, the inertia
            p = Sx[2 * tid];
            q = Sx[2 * tid + 1];
            E = SE[tid];
            s = 0.0;
            cmp = 0.0;
            Am = 1.0;
            Bm = 0.0;
            ng = 0;
            zlast = 0.0;
            rnorm = 0.0;
            const int eref = isF ? io.erefF : io.erefB;
    #pragma unroll 1
            for (int64_t j0 = 0; j0 < len; j0 += RC_U) {
                const int jn = (int)min((int64_t)RC_U, len - j0);
                RowFB<R> rw[RC_U];
                double pmv[RC_U], ipmv[RC_U];
                int ev[RC_U];
    #pragma unroll
                for (int j = 0; j < RC_U; j++)
                    if (j < jn) {
                        const int64_t kk = isF ? k0 + j0 + j : k0 - j0 - j;
                        rw[j] = load_fb<R>(nd.rep, isF ? kk : kk - 1, isF);
                        pmv[j] = 1.0;
                        ipmv[j] = 1.0;
                        ev[j] = 0;
                        if (nd.pp != nullptr && zc != nullptr) {
                            const double2 *qq = reinterpret_cast<const double2 *>(nd.pp + kk * PP_STRIDE);
                            const double2 a0 = __ldg(qq), a1 = __ldg(qq + 1);
                            pmv[j] = a0.x;
                            ipmv[j] = a0.y;
                            ev[j] = __double2loint(a1.x);
                        }
                    }
    #pragma unroll
                for (int j = 0; j < RC_U; j++)
                    if (j < jn) {
                        const int64_t kk = isF ? k0 + j0 + j : k0 - j0 - j;
                        if (zc != nullptr) {
                            // F: y_kk = qF / PP_kk; B: x_kk = QB PP_kk (written scaled by 2^-eref)
                            const double zv = isF ? pow2mul_d(hi(q) * ipmv[j], E - ev[j] - eref)
                                                  : pow2mul_d(hi(q) * pmv[j], E + ev[j] - eref);
                            const OutT zo = (OutT)zv;
                            zc[kk] = zo;
                            kahan_sq((double)zo, s, cmp);
                            zlast = fabs(zv);
                            rnorm = rw[j].nrm + fabs(hi(lam_s));
                        }
                        const R m1 = rw[j].m1, m2 = rw[j].m2;
                        const R D = fma_dd(m1, q, p);
                        // l+ = ld / d+ (F), u- = l d / D- (B), in binary64 off the chain
                        const double lx = rw[j].x * hi(q) * rcp_w(hi(D));
                        const double a2 = lx * lx;
                        Am = clampbig(a2 * Am);
                        Bm = clampbig(a2 * (Bm + 1.0));
                        ng += sgn_ne_R<R>(D, q);
                        p = dot2_dd(mlam, D, m2, p);
                        q = D;
                    }
                const unsigned ex = (unsigned)__double2hiint(hi(p)) & 0x7ff00000u;
                const unsigned ey = (unsigned)__double2hiint(hi(q)) & 0x7ff00000u;
                const unsigned em = ex > ey ? ex : ey;
                if (em != 0x7ff00000u && em != 0u) {
                    const double sc = __hiloint2double((int)(0x7fe00000u - em), 0);
                    p = scale_pow2(p, sc);
                    q = scale_pow2(q, sc);
                    E += (int)(em >> 20) - 1023;
                }
            }
            sA[tid] = Am;
            sB[tid] = Bm;
            // continuity with the next chunk's start state
            bad = 0;
            jres = 0.0;
            bool loose = false;
            // gross-failure bound on the state jump; the storing pass's residual test (jr below)
            // is the accuracy criterion (non-storing passes only steer the shift)
            const double rel_max = Prec<R>::words == 2 ? 0x1p-50 : 0x1p-20;
            if (c + 1 < nc) {
                const int t = tid + 1;
                const int dE = SE[t] - E;
                if (dE > 60 || dE < -60) {
                    bad = 1;
                    loose = true;
                } else {
                    const double sc = __hiloint2double((dE + 1023) << 20, 0);
                    const R p2 = scale_pow2(Sx[2 * t], sc), q2 = scale_pow2(Sx[2 * t + 1], sc);
                    const double mag = fmax(fabs(hi(p)), fabs(hi(q)));
                    const double dif = fmax(fabs(hi(sub(p, p2))), fabs(hi(sub(q, q2))));
                    const double rel = dif / mag;
                    bad = !(rel <= rel_max) ? 1 : 0;
                loose = !(rel <= rel_tight);
                    if (A.dbg_trace) atomicMax(&s_lrel, (int)(log2(rel + 1e-300) * 16.0) + 32768);
                    const double j1 = rel * fmax(zlast, 1e-300) * rnorm;
                    jres = zc != nullptr ? j1 * j1 : 0.0;
                }
            } else if (len > 0 || nc == 1) {  // last chunk of its direction: the state at r
                if (isF) {
                    io.sr = div(p, q);
                    io.yr = hi(q);
                    io.eyr = E;
                } else {
                    io.pr = div(p, q);
                    io.xr = hi(q);
                    io.exr = E;
                }
            }
            if (round + 1 >= RC_ROUNDS || !__syncthreads_or(loose)) break;
            // next round: chunk c starts from chunk c - 1's end state
            Ex[2 * tid] = p;
            Ex[2 * tid + 1] = q;
            EEx[tid] = E;
            __syncthreads();
            if (c > 0) {
                Sx[2 * tid] = Ex[2 * (tid - 1)];
                Sx[2 * tid + 1] = Ex[2 * (tid - 1) + 1];
                SE[tid] = EEx[tid - 1];
            }
            __syncthreads();
        }
        // reductions
        const int warp = tid >> 5, lane = tid & 31;
        double v[6] = {isF ? s : 0.0, isF ? cmp : 0.0, isF ? 0.0 : s,
                       isF ? 0.0 : cmp, isF ? jres : 0.0, isF ? 0.0 : jres};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int u = 0; u < 6; u++) v[u] += __shfl_down_sync(0xffffffffu, v[u], o);
            ng += __shfl_down_sync(0xffffffffu, ng, o);
            bad += __shfl_down_sync(0xffffffffu, bad, o);
        }
        if (lane == 0) {
#pragma unroll
            for (int u = 0; u < 6; u++) s_red[warp][u] = v[u];
            s_redi[warp][0] = ng;
            s_redi[warp][1] = bad;
        }
        __syncthreads();
        if (tid == 0) {
            double acc[6] = {0, 0, 0, 0, 0, 0};
            int i1 = 0, i2 = 0;
            for (int w = 0; w < (T + 31) / 32; w++) {
                for (int u = 0; u < 6; u++) acc[u] += s_red[w][u];
                i1 += s_redi[w][0];
                i2 += s_redi[w][1];
            }
            io.sF = acc[0];
            io.cF = acc[1];
            io.sB = acc[2];
            io.cB = acc[3];
            io.jF = acc[4];
            io.jB = acc[5];
            io.negc = i1;
            io.bad = i2;
            // the norms W_r (F chunks in order from row 0) and V_r (B chunks from row n - 1)
            double Wr = 0.0, Vr = 0.0;
            for (int t = 0; t < tF; t++) Wr = clampbig(sA[t] * Wr + sB[t]);
            for (int t = tF; t < T; t++) Vr = clampbig(sA[t] * Vr + sB[t]);
            nzW = Wr;
            nzV = Vr;
            if (tF == 0) {  // r = 0: no F rows, s_0 = -lam, qF = 1
                io.sr = mlam;
                io.yr = 1.0;
                io.eyr = 0;
            }
            if (tB == 0) {  // r = n - 1: p_{n-1} = d_{n-1} - lam, QB = 1
                io.pr = sub(load_row4<R>(nd.rep, n - 1).d, lam_s);
                io.xr = 1.0;
                io.exr = 0;
            }
        }
        __syncthreads();
    };

    const int maxit = A.maxit;
    // the first iteration number must be uniform over the CTA (the loop holds barriers): the
    // owner state, `passes` included, lives in thread 0 only, so every thread reads the
    // straggler's pass count itself.  (With the owner's private value the other threads ran
    // rs.iters more rounds than thread 0: a straggler that never converged -- all maxit
    // iterations -- left them waiting at a barrier thread 0 had passed for good.)
    const int pass0 = A.resume_in != nullptr ? A.resume_in[id].iters : 0;
    __syncthreads();  // (A.resume may alias A.resume_in: read before thread 0 rewrites it)
#pragma unroll 1
    for (int iters = pass0 + 1; iters <= maxit; iters++) {
        if (tid == 0) {
            const bool store_only =
                A.jobz_v && iters >= 2 && done && !zfinal && zcol != nullptr && n > 1;
            const bool need = (!done || store_only) && !handoff;
            io.need = need ? (store_only ? 2 : 1) : 0;
            io.lam = lam;
            io.r = r;
            io.erefF = erefF;
            io.erefB = erefB;
            io.wz = (need && A.jobz_v && iters >= 2 && zcol != nullptr) ? 1 : 0;
        }
        if (tid == 0) s_lrel = 0;
        __syncthreads();
        if (io.need == 0) break;
        chunk_pass();
        if (tid == 0) {
            const bool store_only = io.need == 2;
            zwritten = false;
            // join: gamma_r, inertia, ||z||^2, references (as k_rqi_fb's pass)
            double pm = 1.0, ipm = 1.0;
            int e = 0;
            if (nd.pp != nullptr) {
                const double2 *qq = reinterpret_cast<const double2 *>(nd.pp + r * PP_STRIDE);
                pm = qq[0].x;
                ipm = qq[0].y;
                e = __double2loint(qq[1].x);
            }
            const double yr = io.yr * ipm, xr = io.xr * pm;
            const int eyr = io.eyr - e, exr = io.exr + e;
            double sF = io.sF, cF_ = io.cF;
            const OutT zo = (OutT)pow2mul_d(yr, eyr - erefF);
            kahan_sq((double)zo, sF, cF_);
            const double fF = ldexp(1.0, erefF - eyr) / yr;
            const double fB = ldexp(1.0, erefB - exr) / xr;
            const double nzz = 1.0 + nzW + nzV;  // ||z||^2 for the RQ correction (as k_rqi_fb)
            const double ssw = fF * fF * (sF - cF_) + fB * fB * (io.sB - io.cB);  // written z
            const double jr = io.wz ? sqrt(fF * fF * io.jF + fB * fB * io.jB) / sqrt(ssw) : 0.0;
            if (io.bad || !(jr <= 0.125 * tol)) {
                handoff = true;  // k_rqi continues serially from the state before this pass
                if (A.dbg_trace) {
                    double *tr = A.dbg_trace + 8 * (int64_t)id;
                    tr[0] = (s_lrel - 32768) / 16.0;
                    tr[1] = jr / tol;
                    tr[2] = iters;
                    tr[3] = (double)r;
                    tr[4] = (double)n;
                    tr[5] = io.bad;
                }
            } else {
                gr = add(add(io.sr, io.pr), lam);
                const int c = io.negc + (is_neg(gr) ? 1 : 0);
                nz2 = nzz;
                rows += n;
                passes = iters;
                if (io.wz) {
                    zcol[r] = zo;
                    zinfo.cF = fF;
                    zinfo.cB = fB;
                    zinfo.ss = ssw;
                    zwritten = true;
                }
                erefF = eyr + expo_of(yr);
                erefB = exr + expo_of(xr);
                if (store_only) {
                    zfinal = zwritten;
                } else {
                    if (c >= k) {
                        if (lt(lam, b)) b = lam;
                    } else {
                        if (lt(a, lam)) a = lam;
                    }
                    const double g = hi(gr);
                    const double corr = g / nz2;
                    R lam_new = add(lam, mk<R>(corr));
                    if (fabs(g) / sqrt(nz2) <= tol ||
                        fabs(corr) <= 8.0 * Prec<R>::eps * fabs(hi(lam)) || g == 0.0) {
                        lam_out = lam_new;
                        done = true;
                        zfinal = zwritten;
                    } else {
                        if (!(lt(a, lam_new) && lt(lam_new, b))) lam_new = half(add(a, b));
                        lam = lam_new;
                    }
                }
            }
        }
        __syncthreads();
    }
    (void)zwritten;
    // ---- results
    __shared__ int s_fin;
    if (tid == 0) {
        const bool finished = done && (zfinal || zcol == nullptr);
        s_fin = finished ? 1 : 0;
        A.left[pos] = finished ? 0 : 1;
        if (finished) {
            const R lt_ = add(lam_out, mk2<R>(nd.sig_hi, nd.sig_lo));
            if (col0 >= 0) {
                if (sizeof(OutT) == 4)
                    reinterpret_cast<float *>(A.w)[col0] = (float)(hi(lt_) * A.unscale);
                else
                    reinterpret_cast<double *>(A.w)[col0] = hi(lt_) * A.unscale;
            }
            reinterpret_cast<R *>(A.it.lo)[id] = lam_out;
            atomicMax(&A.st->rqi_iters_max, passes);
            if (A.dbg_iters) A.dbg_iters[id] = passes;
            if (zcol != nullptr) A.zc[col0 - A.zcol0] = zinfo;
        } else {
            RqiResume<R> rs;
            rs.lam = lam;
            rs.a = a;
            rs.b = b;
            rs.lam_out = lam_out;
            rs.iters = passes;
            rs.erefF = erefF;
            rs.erefB = erefB;
            rs.flags = (done ? 1 : 0) | (zfinal ? 2 : 0);
            A.resume[id] = rs;
        }
        if (rows) atomicAdd(&A.st->rqi_rows, rows);
        s_zc = zinfo;
    }
    __syncthreads();
    // K6 epilogue: normalise the finished column (collective, coalesced)
    if (!A.jobz_v || !A.fuse_scale || !s_fin || zcol == nullptr) return;
    const ZCol z = s_zc;
    const double inv = 1.0 / sqrt(z.ss);
    const double fF = z.cF * inv, fB = z.cB * inv;
    for (int64_t i = tid; i < z.n; i += T) zcol[i] = (OutT)((double)zcol[i] * (i <= z.r ? fF : fB));
}

}  // namespace mr3
