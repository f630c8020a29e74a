/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (not part of the product).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and
 * `bench.py --impl reference`) may load, link or execute anything under
 * oracle/.  The CUDA product path (paper_1304_1864_b200/) shares no code,
 * header, table or constant generator with this file, and neither side
 * imports the other.
 *
 * What it computes: the plain definition of what the mixed-precision MRRR
 * hot path computes -- the eigenpairs (lambda_i, z_i), ||z_i|| = 1, of the
 * real symmetric tridiagonal T = tridiag(e, d, e)   (§1,
 * "the real symmetric tridiagonal eigenproblem (STEP)") -- in IEEE binary128
 * (__float128, eps_q = 2^-113, Table 1), with no
 * representation tree, no LDL^T, no perturbation:
 *
 *   eigenvalues : bisection with the Sturm sequence of T itself
 *                 ("Commonly, the eigenvalues are computed by some form of
 *                 bisection", §2)
 *   eigenvectors: inverse iteration on T - lambda*I (Gaussian elimination
 *                 with partial pivoting) with classical Gram-Schmidt applied
 *                 twice against the other members of the same group
 *                 (BJ:5 "inverse iteration with full
 *                 reorthogonalization")
 *   verification: Eq. (1.1) residual R (1-norm) and a
 *                 2-norm variant, orthogonality O (L133) with compensated
 *                 (Dot2) inner products, per-column sin(angle) and group
 *                 subspace residuals vs the oracle's own vectors.
 *   brute force : cyclic Jacobi on the dense matrix, n <= 16 (pins only).
 *
 * Everything is plain loops; OpenMP only distributes independent indices or
 * groups.  Build: gcc -O2 -fopenmp -shared -fPIC oracle.c -lquadmath.
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __float128 quad;

#define EPS_Q ((quad)1.0 / ((quad)(1ULL << 56) * (quad)(1ULL << 57))) /* 2^-113 */

static quad qabs(quad x) { return x < 0 ? -x : x; }
static quad qmax(quad a, quad b) { return a > b ? a : b; }

/* widen the (hi, lo) double pairs to binary128; lo may be NULL */
static void widen(int64_t n, const double *hi, const double *lo, quad *out) {
    for (int64_t i = 0; i < n; i++) out[i] = (quad)hi[i] + (lo ? (quad)lo[i] : (quad)0);
}

static void split_out(quad x, double *hi, double *lo) {
    double h = (double)x;
    *hi = h;
    *lo = (double)(x - (quad)h);
}

/* ||T||_1 = max_j sum_i |T_ij|  (Eq. (1.1) uses ||T||_1) */
static quad norm1_q(int64_t n, const quad *d, const quad *e) {
    quad m = 0;
    for (int64_t i = 0; i < n; i++) {
        quad s = qabs(d[i]);
        if (i > 0) s += qabs(e[i - 1]);
        if (i < n - 1) s += qabs(e[i]);
        m = qmax(m, s);
    }
    return m;
}

/* Gershgorin enclosure [gl, gu] of spec[T] */
static void gershgorin_q(int64_t n, const quad *d, const quad *e, quad *gl, quad *gu) {
    quad lo = 0, hi = 0;
    for (int64_t i = 0; i < n; i++) {
        quad r = 0;
        if (i > 0) r += qabs(e[i - 1]);
        if (i < n - 1) r += qabs(e[i]);
        quad a = d[i] - r, b = d[i] + r;
        if (i == 0 || a < lo) lo = a;
        if (i == 0 || b > hi) hi = b;
    }
    *gl = lo;
    *gu = hi;
}

/*
 * Sturm count: number of eigenvalues of T strictly below x.
 * q_1 = d_1 - x ; q_i = (d_i - x) - e_{i-1}^2 / q_{i-1} ; count #{q_i < 0}.
 * A pivot with |q_i| < pivmin is replaced by -pivmin (oracle
 * reading 8(c) item 2), pivmin = eps_q * ||T||_1: a perturbation of d_i of
 * size <= 2 pivmin, far below every tolerance.
 */
static int64_t sturm_q(int64_t n, const quad *d, const quad *e, quad x, quad pivmin) {
    int64_t cnt = 0;
    quad q = d[0] - x;
    if (qabs(q) < pivmin) q = -pivmin;
    if (q < 0) cnt++;
    for (int64_t i = 1; i < n; i++) {
        q = (d[i] - x) - (e[i - 1] * e[i - 1]) / q;
        if (qabs(q) < pivmin) q = -pivmin;
        if (q < 0) cnt++;
    }
    return cnt;
}

typedef struct {
    int64_t n;
    quad *d, *e;
    quad nrm, gl, gu, pivmin, absfloor;
} tri_t;

static int tri_init(tri_t *t, int64_t n, const double *d_hi, const double *d_lo,
                    const double *e_hi, const double *e_lo) {
    t->n = n;
    t->d = (quad *)malloc(sizeof(quad) * (n > 0 ? n : 1));
    t->e = (quad *)malloc(sizeof(quad) * (n > 1 ? n - 1 : 1));
    if (!t->d || !t->e) return -1;
    widen(n, d_hi, d_lo, t->d);
    if (n > 1) widen(n - 1, e_hi, e_lo, t->e);
    t->nrm = norm1_q(n, t->d, t->e);
    quad scale = t->nrm > 0 ? t->nrm : (quad)1;
    gershgorin_q(n, t->d, t->e, &t->gl, &t->gu);
    /* widen the enclosure a hair so the endpoint counts are certainly 0 and n */
    quad pad = 4 * EPS_Q * qmax(qmax(qabs(t->gl), qabs(t->gu)), scale);
    t->gl -= pad;
    t->gu += pad;
    t->pivmin = EPS_Q * scale;
    t->absfloor = EPS_Q * EPS_Q * scale * 1024; /* bracket floor for lambda == 0 */
    return 0;
}

static void tri_free(tri_t *t) {
    free(t->d);
    free(t->e);
}

/* bisection for eigenvalue index i (1-based): count(lo) < i <= count(hi) */
static quad bisect_one(const tri_t *t, int64_t i) {
    quad lo = t->gl, hi = t->gu;
    for (int it = 0; it < 2000; it++) {
        quad w = hi - lo;
        quad tol = qmax(2 * EPS_Q * qmax(qabs(lo), qabs(hi)), t->absfloor);
        if (w <= tol) break;
        quad mid = lo + w / 2;
        if (mid <= lo || mid >= hi) break;
        if (sturm_q(t->n, t->d, t->e, mid, t->pivmin) >= i)
            hi = mid;
        else
            lo = mid;
    }
    return lo + (hi - lo) / 2;
}

/* ------------------------------------------------------------------------ */
/* exported: scalar helpers                                                  */
/* ------------------------------------------------------------------------ */

void oracle_norm1(int64_t n, const double *d_hi, const double *d_lo, const double *e_hi,
                  const double *e_lo, double *out_hi, double *out_lo) {
    tri_t t;
    if (tri_init(&t, n, d_hi, d_lo, e_hi, e_lo)) return;
    split_out(t.nrm, out_hi, out_lo);
    tri_free(&t);
}

void oracle_gershgorin(int64_t n, const double *d_hi, const double *d_lo, const double *e_hi,
                       const double *e_lo, double *out /* gl_hi, gl_lo, gu_hi, gu_lo */) {
    tri_t t;
    if (tri_init(&t, n, d_hi, d_lo, e_hi, e_lo)) return;
    split_out(t.gl, out, out + 1);
    split_out(t.gu, out + 2, out + 3);
    tri_free(&t);
}

/* Sturm counts at k shifts x = x_hi + x_lo (for invariant pins) */
void oracle_sturm_counts(int64_t n, const double *d_hi, const double *d_lo, const double *e_hi,
                         const double *e_lo, int64_t k, const double *x_hi, const double *x_lo,
                         int64_t *counts) {
    tri_t t;
    if (tri_init(&t, n, d_hi, d_lo, e_hi, e_lo)) return;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < k; j++) {
        quad x = (quad)x_hi[j] + (x_lo ? (quad)x_lo[j] : (quad)0);
        counts[j] = sturm_q(t.n, t.d, t.e, x, t.pivmin);
    }
    tri_free(&t);
}

/* ------------------------------------------------------------------------ */
/* exported: eigenvalues by bisection on T                                   */
/* ------------------------------------------------------------------------ */

/* eigenvalues with 1-based indices idx[0..m-1]; results as (hi, lo) pairs */
int oracle_eigvals(int64_t n, const double *d_hi, const double *d_lo, const double *e_hi,
                   const double *e_lo, int64_t m, const int64_t *idx, double *lam_hi,
                   double *lam_lo) {
    if (n <= 0) return 0;
    tri_t t;
    if (tri_init(&t, n, d_hi, d_lo, e_hi, e_lo)) return -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t j = 0; j < m; j++) {
        quad l = bisect_one(&t, idx[j]);
        split_out(l, &lam_hi[j], &lam_lo[j]);
    }
    tri_free(&t);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* exported: eigenvectors by inverse iteration                               */
/* ------------------------------------------------------------------------ */

static uint64_t splitmix64(uint64_t *s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct {
    int64_t n;
    quad *dl, *dd, *du, *du2;
    int64_t *ipiv;
} lu_t;

/* LU with partial pivoting of the tridiagonal A = T - lambda I (row interchanges
 * between i and i+1 only, as for any tridiagonal GEPP).  A zero pivot of U is
 * replaced by eps_q ||T||_1 (a backward perturbation far below every tolerance). */
static void lu_factor(const tri_t *t, quad lambda, lu_t *f) {
    int64_t n = t->n;
    quad tiny = EPS_Q * (t->nrm > 0 ? t->nrm : (quad)1);
    for (int64_t i = 0; i < n; i++) {
        f->dd[i] = t->d[i] - lambda;
        if (i < n - 1) {
            f->dl[i] = t->e[i];
            f->du[i] = t->e[i];
        }
        if (i < n - 2) f->du2[i] = 0;
    }
    for (int64_t i = 0; i < n - 1; i++) {
        if (qabs(f->dd[i]) >= qabs(f->dl[i])) {
            if (f->dd[i] == 0) f->dd[i] = tiny;
            quad fact = f->dl[i] / f->dd[i];
            f->dl[i] = fact;
            f->dd[i + 1] -= fact * f->du[i];
            f->ipiv[i] = i;
        } else {
            quad fact = f->dd[i] / f->dl[i];
            f->dd[i] = f->dl[i];
            f->dl[i] = fact;
            quad tmp = f->du[i];
            f->du[i] = f->dd[i + 1];
            f->dd[i + 1] = tmp - fact * f->dd[i + 1];
            if (i < n - 2) {
                f->du2[i] = f->du[i + 1];
                f->du[i + 1] = -fact * f->du[i + 1];
            }
            f->ipiv[i] = i + 1;
        }
    }
    if (f->dd[n - 1] == 0) f->dd[n - 1] = tiny;
}

static void lu_solve(const lu_t *f, quad *b) {
    int64_t n = f->n;
    for (int64_t i = 0; i < n - 1; i++) {
        if (f->ipiv[i] == i) {
            b[i + 1] -= f->dl[i] * b[i];
        } else {
            quad tmp = b[i];
            b[i] = b[i + 1];
            b[i + 1] = tmp - f->dl[i] * b[i];
        }
    }
    b[n - 1] /= f->dd[n - 1];
    if (n > 1) b[n - 2] = (b[n - 2] - f->du[n - 2] * b[n - 1]) / f->dd[n - 2];
    for (int64_t i = n - 3; i >= 0; i--)
        b[i] = (b[i] - f->du[i] * b[i + 1] - f->du2[i] * b[i + 2]) / f->dd[i];
}

static void normalize_q(int64_t n, quad *x) {
    quad mx = 0;
    for (int64_t i = 0; i < n; i++) mx = qmax(mx, qabs(x[i]));
    if (mx == 0) return;
    quad s = 0;
    for (int64_t i = 0; i < n; i++) {
        x[i] /= mx;
        s += x[i] * x[i];
    }
    s = sqrtq(s);
    for (int64_t i = 0; i < n; i++) x[i] /= s;
}

/* classical Gram-Schmidt against the k vectors in V (each length n), applied twice */
static void cgs2(int64_t n, quad *x, quad *const *V, int64_t k) {
    for (int pass = 0; pass < 2; pass++) {
        for (int64_t j = 0; j < k; j++) {
            quad c = 0;
            for (int64_t i = 0; i < n; i++) c += V[j][i] * x[i];
            for (int64_t i = 0; i < n; i++) x[i] -= c * V[j][i];
        }
    }
}

/*
 * Eigenvectors for the m eigenvalues lam (ascending, hi+lo).  Groups are
 * maximal runs with consecutive gaps < group_tol (absolute).  Within a group,
 * each iterate is reorthogonalised (CGS2) against the earlier members.
 * 3 inverse iterations from a seeded pseudo-random start.
 * Output Z (n x m, column-major) as hi + lo double pairs.
 */
int oracle_eigvecs(int64_t n, const double *d_hi, const double *d_lo, const double *e_hi,
                   const double *e_lo, int64_t m, const double *lam_hi, const double *lam_lo,
                   double group_tol, uint64_t seed, int iters, double *Z_hi, double *Z_lo) {
    if (n <= 0 || m <= 0) return 0;
    tri_t t;
    if (tri_init(&t, n, d_hi, d_lo, e_hi, e_lo)) return -1;
    quad *lam = (quad *)malloc(sizeof(quad) * m);
    widen(m, lam_hi, lam_lo, lam);
    /* group starts */
    int64_t *gstart = (int64_t *)malloc(sizeof(int64_t) * (m + 1));
    int64_t ng = 0;
    for (int64_t j = 0; j < m; j++)
        if (j == 0 || lam[j] - lam[j - 1] >= (quad)group_tol) gstart[ng++] = j;
    gstart[ng] = m;
    if (iters <= 0) iters = 3;

#pragma omp parallel
    {
        lu_t f;
        f.n = n;
        f.dl = (quad *)malloc(sizeof(quad) * (n + 2));
        f.dd = (quad *)malloc(sizeof(quad) * (n + 2));
        f.du = (quad *)malloc(sizeof(quad) * (n + 2));
        f.du2 = (quad *)malloc(sizeof(quad) * (n + 2));
        f.ipiv = (int64_t *)malloc(sizeof(int64_t) * (n + 2));
#pragma omp for schedule(dynamic, 1)
        for (int64_t g = 0; g < ng; g++) {
            int64_t j0 = gstart[g], j1 = gstart[g + 1], gs = j1 - j0;
            quad **V = (quad **)malloc(sizeof(quad *) * gs);
            for (int64_t a = 0; a < gs; a++) V[a] = (quad *)malloc(sizeof(quad) * n);
            for (int64_t a = 0; a < gs; a++) {
                int64_t j = j0 + a;
                quad *x = V[a];
                uint64_t s = seed ^ (0x51ED27F1ULL * (uint64_t)(j + 1));
                for (int64_t i = 0; i < n; i++)
                    x[i] = (quad)((double)(splitmix64(&s) >> 11) * 0x1.0p-53 * 2.0 - 1.0);
                normalize_q(n, x);
                lu_factor(&t, lam[j], &f);
                for (int it = 0; it < iters; it++) {
                    lu_solve(&f, x);
                    normalize_q(n, x);
                    if (a > 0) {
                        cgs2(n, x, V, a);
                        normalize_q(n, x);
                    }
                }
                /* sign convention (comparisons are up to sign): largest |x_i| positive */
                int64_t im = 0;
                for (int64_t i = 1; i < n; i++)
                    if (qabs(x[i]) > qabs(x[im])) im = i;
                if (x[im] < 0)
                    for (int64_t i = 0; i < n; i++) x[i] = -x[i];
                for (int64_t i = 0; i < n; i++)
                    split_out(x[i], &Z_hi[i + n * j], &Z_lo[i + n * j]);
            }
            for (int64_t a = 0; a < gs; a++) free(V[a]);
            free(V);
        }
        free(f.dl);
        free(f.dd);
        free(f.du);
        free(f.du2);
        free(f.ipiv);
    }
    free(gstart);
    free(lam);
    tri_free(&t);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* exported: verification (Eq. (1.1))                                        */
/* ------------------------------------------------------------------------ */

/*
 * Residuals of computed pairs (w_j, Z[:, j]) (fp64 or widened fp32 values):
 *   r = T z - w z evaluated in binary128;  r1[j] = ||r||_1 / ||T||_1  (Eq. 1.1),
 *   r2[j] = ||r||_2 / ||T||_1,  znorm[j] = ||z||_2 - 1.
 */
int oracle_residuals(int64_t n, const double *d, const double *e, int64_t m, const double *w,
                     const double *Z, int64_t ldz, double *r1, double *r2, double *znorm) {
    if (n <= 0) return 0;
    tri_t t;
    if (tri_init(&t, n, d, NULL, e, NULL)) return -1;
    quad nrm = t.nrm > 0 ? t.nrm : (quad)1;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < m; j++) {
        const double *z = Z + ldz * j;
        quad s1 = 0, s2 = 0, zz = 0, lam = w[j];
        for (int64_t i = 0; i < n; i++) {
            quad r = (t.d[i] - lam) * (quad)z[i];
            if (i > 0) r += t.e[i - 1] * (quad)z[i - 1];
            if (i < n - 1) r += t.e[i] * (quad)z[i + 1];
            s1 += qabs(r);
            s2 += r * r;
            zz += (quad)z[i] * (quad)z[i];
        }
        r1[j] = (double)(s1 / nrm);
        r2[j] = (double)(sqrtq(s2) / nrm);
        if (znorm) znorm[j] = (double)(sqrtq(zz) - 1);
    }
    tri_free(&t);
    return 0;
}

/* error-free product / sum for the compensated dot (Ogita-Rump-Oishi Dot2) */
static inline void two_prod_d(double a, double b, double *p, double *e) {
    *p = a * b;
    *e = fma(a, b, -*p);
}
static inline void two_sum_d(double a, double b, double *s, double *e) {
    double x = a + b, bb = x - a;
    *s = x;
    *e = (a - (x - bb)) + (b - bb);
}

/* O = max_{i != j} |z_i^T z_j| (Eq. 1.1) with Dot2 inner products; also the
 * maximum |z_i^T z_i - 1| in *diag_dev. Cost O(m^2 n): small problems only. */
double oracle_orthogonality(int64_t n, int64_t m, const double *Z, int64_t ldz,
                            double *diag_dev) {
    double omax = 0, dmax = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(max : omax, dmax)
    for (int64_t a = 0; a < m; a++) {
        const double *x = Z + ldz * a;
        for (int64_t b = a; b < m; b++) {
            const double *y = Z + ldz * b;
            double s = 0, c = 0;
            for (int64_t i = 0; i < n; i++) {
                double p, ep, es;
                two_prod_d(x[i], y[i], &p, &ep);
                two_sum_d(s, p, &s, &es);
                c += ep + es;
            }
            double v = s + c;
            if (a == b) {
                double dv = fabs(v - 1.0);
                if (dv > dmax) dmax = dv;
            } else if (fabs(v) > omax) {
                omax = fabs(v);
            }
        }
    }
    if (diag_dev) *diag_dev = dmax;
    return omax;
}

/* per-column sin(angle(zhat_j, z_j)) = ||zhat - (z^T zhat) z|| / ||zhat|| in binary128,
 * z = Zo_hi + Zo_lo (the oracle's unit vectors). */
int oracle_sin_angles(int64_t n, int64_t m, const double *Zhat, int64_t ldz, const double *Zo_hi,
                      const double *Zo_lo, double *out) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < m; j++) {
        const double *x = Zhat + ldz * j;
        const double *h = Zo_hi + n * j, *l = Zo_lo + n * j;
        quad c = 0, xx = 0;
        for (int64_t i = 0; i < n; i++) {
            quad zi = (quad)h[i] + (quad)l[i];
            c += zi * (quad)x[i];
            xx += (quad)x[i] * (quad)x[i];
        }
        quad s = 0;
        for (int64_t i = 0; i < n; i++) {
            quad zi = (quad)h[i] + (quad)l[i];
            quad r = (quad)x[i] - c * zi;
            s += r * r;
        }
        out[j] = xx > 0 ? (double)sqrtq(s / xx) : 1.0;
    }
    return 0;
}

/* group subspace residual P = Zhat_G - Z_G (Z_G^T Zhat_G) in binary128, rounded to
 * fp64 (n x g column-major); sin(Theta_G) = ||P||_2 for orthonormal Zhat_G. */
int oracle_subspace_residual(int64_t n, int64_t g, const double *Zhat, int64_t ldz,
                             const double *Zo_hi, const double *Zo_lo, double *P) {
    quad *C = (quad *)calloc((size_t)(g * g), sizeof(quad));
    for (int64_t a = 0; a < g; a++)
        for (int64_t b = 0; b < g; b++) {
            quad c = 0;
            for (int64_t i = 0; i < n; i++)
                c += ((quad)Zo_hi[i + n * a] + (quad)Zo_lo[i + n * a]) * (quad)Zhat[i + ldz * b];
            C[a + g * b] = c;
        }
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < g; b++)
        for (int64_t i = 0; i < n; i++) {
            quad r = Zhat[i + ldz * b];
            for (int64_t a = 0; a < g; a++)
                r -= ((quad)Zo_hi[i + n * a] + (quad)Zo_lo[i + n * a]) * C[a + g * b];
            P[i + n * b] = (double)r;
        }
    free(C);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* exported: brute-force cyclic Jacobi on the dense matrix (pins, n <= 16)   */
/* ------------------------------------------------------------------------ */

int oracle_jacobi(int64_t n, const double *d_hi, const double *d_lo, const double *e_hi,
                  const double *e_lo, double *lam_hi, double *lam_lo, double *V_hi,
                  double *V_lo) {
    if (n <= 0 || n > 64) return -1;
    quad A[64][64], V[64][64];
    quad *d = (quad *)malloc(sizeof(quad) * n), *e = (quad *)malloc(sizeof(quad) * n);
    widen(n, d_hi, d_lo, d);
    if (n > 1) widen(n - 1, e_hi, e_lo, e);
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < n; j++) {
            A[i][j] = 0;
            V[i][j] = (i == j) ? 1 : 0;
        }
    for (int64_t i = 0; i < n; i++) A[i][i] = d[i];
    for (int64_t i = 0; i + 1 < n; i++) A[i][i + 1] = A[i + 1][i] = e[i];
    for (int sweep = 0; sweep < 100; sweep++) {
        quad off = 0, tot = 0;
        for (int64_t i = 0; i < n; i++)
            for (int64_t j = 0; j < n; j++) {
                tot += A[i][j] * A[i][j];
                if (i != j) off += A[i][j] * A[i][j];
            }
        if (off <= EPS_Q * EPS_Q * tot * 1e-4Q) break;
        for (int64_t p = 0; p < n; p++)
            for (int64_t q = p + 1; q < n; q++) {
                if (A[p][q] == 0) continue;
                quad theta = (A[q][q] - A[p][p]) / (2 * A[p][q]);
                quad tt = (theta >= 0 ? 1 : -1) / (qabs(theta) + sqrtq(theta * theta + 1));
                quad c = 1 / sqrtq(tt * tt + 1), s = tt * c;
                for (int64_t k = 0; k < n; k++) { /* A <- A J */
                    quad akp = A[k][p], akq = A[k][q];
                    A[k][p] = c * akp - s * akq;
                    A[k][q] = s * akp + c * akq;
                }
                for (int64_t k = 0; k < n; k++) { /* A <- J^T A */
                    quad apk = A[p][k], aqk = A[q][k];
                    A[p][k] = c * apk - s * aqk;
                    A[q][k] = s * apk + c * aqk;
                }
                for (int64_t k = 0; k < n; k++) {
                    quad vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = c * vkp - s * vkq;
                    V[k][q] = s * vkp + c * vkq;
                }
            }
    }
    /* selection sort ascending */
    int64_t order[64];
    for (int64_t i = 0; i < n; i++) order[i] = i;
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = i + 1; j < n; j++)
            if (A[order[j]][order[j]] < A[order[i]][order[i]]) {
                int64_t t = order[i];
                order[i] = order[j];
                order[j] = t;
            }
    for (int64_t k = 0; k < n; k++) {
        int64_t c = order[k];
        split_out(A[c][c], &lam_hi[k], &lam_lo[k]);
        for (int64_t i = 0; i < n; i++) split_out(V[i][c], &V_hi[i + n * k], &V_lo[i + n * k]);
    }
    free(d);
    free(e);
    return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
