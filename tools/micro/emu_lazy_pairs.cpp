#include <cstdio>
#include <cstdlib>
#include <vector>
// Host emulation of the fixed-twist F / B rows (k_rqi_fb) with normalised pairs (var 0) and
// with the final renormalisation of the pair dot product (var 1) or of both row operations
// (var 2) dropped -- the "lazy pair" experiment of round 2: the
// unnormalised low parts grow relative to the high parts row after row (var 1: NaN gamma on
// config 2), so the kernels keep normalised pairs.
// usage: python gen.py <config> <index>  (writes in.bin)  &&  ./emu in.bin
#include "../../paper_1304_1864_b200/csrc/dd.cuh"
using namespace mr3;
static dd renorm(dd a) { double l; const double h = quick_two_sum(a.hi, a.lo, l); return mkdd(h, l); }
static dd dot2_n(dd a, dd x, dd b, dd y) { return dot2_dd(a, x, b, y); }
static dd dot2_lazy(dd a, dd x, dd b, dd y) {
    const double p1 = mul_rn(a.hi, x.hi), p2 = mul_rn(b.hi, y.hi);
    double e1 = fma_rn(a.hi, x.hi, -p1), e2 = fma_rn(b.hi, y.hi, -p2);
    e1 = fma_rn(a.hi, x.lo, e1); e2 = fma_rn(b.hi, y.lo, e2);
    e1 = fma_rn(a.lo, x.hi, e1); e2 = fma_rn(b.lo, y.hi, e2);
    double es; const double s = two_sum(p1, p2, es);
    return mkdd(s, add_rn(es, add_rn(e1, e2)));
}
static dd fma_dd_u(dd a, dd b, dd c, double &h) {
    double p = mul_rn(a.hi, b.hi), e = fma_rn(a.hi, b.hi, -p);
    e = fma_rn(a.hi, b.lo, e); e = fma_rn(a.lo, b.hi, e);
    double s2; double s = two_sum(p, c.hi, s2);
    s2 = add_rn(s2, add_rn(e, c.lo)); h = add_rn(s, s2);
    return mkdd(s, s2);
}
static void rescale(dd &x, dd &y, int &E) {
    int ex, ey; frexp(x.hi, &ex); frexp(y.hi, &ey);
    int em = ex > ey ? ex : ey;
    if (x.hi == 0 && y.hi == 0) return;
    double sc = ldexp(1.0, -em);
    x = mkdd(x.hi * sc, x.lo * sc); y = mkdd(y.hi * sc, y.lo * sc); E += em;
}
int main(int argc, char **argv) {
    int n; double lam_hi, lam_lo; long r;
    FILE *f = fopen(argv[1], "rb");
    fread(&n, 4, 1, f); fread(&lam_hi, 8, 1, f); fread(&lam_lo, 8, 1, f); fread(&r, 8, 1, f);
    std::vector<dd> d(n), ld(n), lld(n);
    for (int i = 0; i < n; i++) { double v[6]; fread(v, 8, 6, f); d[i] = mkdd(v[0], v[1]); ld[i] = mkdd(v[2], v[3]); lld[i] = mkdd(v[4], v[5]); }
    dd lam = mkdd(lam_hi, lam_lo), mlam = neg(lam);
    for (int var = 0; var < 3; var++) {  // 0 normalised, 1 lazy dot2 + normalised fma, 2 both lazy
        dd px = mlam, qx = mkdd(1, 0); int E = 0, negc = 0; double qh = 1;
        for (long k = 0; k < r; k++) {
            double Dh; dd D;
            if (var == 2) D = fma_dd_u(d[k], qx, px, Dh); else { D = fma_dd(d[k], qx, px); Dh = D.hi; }
            dd p2 = var == 0 ? dot2_n(mlam, D, lld[k], px) : dot2_lazy(mlam, D, lld[k], px);
            negc += ((Dh < 0) != (qh < 0));
            if (var == 1 && (std::isnan(p2.hi) || std::isnan(D.hi)) ) { printf("k %ld: px %a %a qx %a %a D %a %a p2 %a %a\n", k, px.hi, px.lo, qx.hi, qx.lo, D.hi, D.lo, p2.hi, p2.lo); break; }
            px = p2; qx = D; qh = Dh;
            if ((k & 7) == 7) { rescale(px, qx, E); qh = ldexp(qh, 0); qh = qx.hi + 0.0; if (var == 2) qh = add_rn(qx.hi, qx.lo); }
        }
        dd pF = renorm(px), qF = renorm(qx);
        dd pb = sub(d[n - 1], lam), qb = mkdd(1, 0); double qbh = 1;
        for (long k = n - 1; k > r; k--) {
            double Eh; dd Ee;
            if (var == 2) Ee = fma_dd_u(lld[k - 1], qb, pb, Eh); else { Ee = fma_dd(lld[k - 1], qb, pb); Eh = Ee.hi; }
            dd P2 = var == 0 ? dot2_n(mlam, Ee, d[k - 1], pb) : dot2_lazy(mlam, Ee, d[k - 1], pb);
            negc += ((Eh < 0) != (qbh < 0));
            if (var == 1 && (std::isnan(P2.hi) || std::isnan(Ee.hi) || std::isinf(P2.hi)|| std::isinf(Ee.hi))) { printf("B k %ld: pb %a %a qb %a %a E %a %a P2 %a %a\n", k, pb.hi, pb.lo, qb.hi, qb.lo, Ee.hi, Ee.lo, P2.hi, P2.lo); break; }
            if (var == 1 && k > n - 40) printf("B k %ld: pb %a %a qb %a %a E %a %a P2 %a %a\n", k, pb.hi, pb.lo, qb.hi, qb.lo, Ee.hi, Ee.lo, P2.hi, P2.lo);
            pb = P2; qb = Ee; qbh = Eh;
            if (((n - 1 - k) & 7) == 7) { int E2 = 0; rescale(pb, qb, E2); qbh = var == 2 ? add_rn(qb.hi, qb.lo) : qb.hi; }
        }
        dd pB = renorm(pb), qB = renorm(qb);
        if (var == 1) printf("pF %a %a qF %a %a pB %a %a qB %a %a\n", pF.hi, pF.lo, qF.hi, qF.lo, pB.hi, pB.lo, qB.hi, qB.lo);
        dd g = add(add(div(pF, qF), div(pB, qB)), lam);
        printf("var %d: gamma = %.17e + %.6e  negc %d\n", var, g.hi, g.lo, negc + (g.hi < 0));
    }
}
