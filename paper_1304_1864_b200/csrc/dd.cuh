// dd.cuh -- B0: the wide working precision binary_y of PAPER.md §3.1 (L746-L801).
//
// For fp64 I/O the paper's working format is binary128 in software (L1318-L1326);
// here it is double-double ("pair") arithmetic on the FP64 FMA pipe
// (eps_y ~ 2^-104), for fp32 I/O it is plain binary64
// (L1291-L1304).  Both present the same overload set so every kernel is written
// once as a template over R in {dd, double}:
//     add sub mul div neg half hi mk is_neg absd lt
//
// Error-free transforms must not be contracted into FMAs: all primitive ops go
// through __dadd_rn / __dsub_rn / __dmul_rn / __fma_rn on the device, and the
// host side is compiled with -ffp-contract=off (SURVEY.md §7 hard part 7).
//
// Additions are the "sloppy" pair addition (one two-sum on the high parts): its
// error is eps_y*(|a|+|b|) rather than eps_y*|a+b|.  Inside dstqds/dpqds that is
// a relative perturbation of the data and the shift of size eps_y per step,
// far below the eps_x-level the method needs (reading R7).
#pragma once
#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define MR3_HD __host__ __device__ __forceinline__
#else
#define MR3_HD inline
#endif

namespace mr3 {

#if defined(__CUDA_ARCH__)
MR3_HD double add_rn(double a, double b) { return __dadd_rn(a, b); }
MR3_HD double sub_rn(double a, double b) { return __dsub_rn(a, b); }
MR3_HD double mul_rn(double a, double b) { return __dmul_rn(a, b); }
MR3_HD double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
// MUFU.RCP64H seed (about 2^-22 relative); refined below.
MR3_HD double rcp_seed(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}
#else
MR3_HD double add_rn(double a, double b) { return a + b; }
MR3_HD double sub_rn(double a, double b) { return a - b; }
MR3_HD double mul_rn(double a, double b) { return a * b; }
MR3_HD double fma_rn(double a, double b, double c) { return fma(a, b, c); }
MR3_HD double rcp_seed(double x) { return (double)(1.0f / (float)x); }
#endif

// reciprocal to ~1 ulp: one cubic Newton step e = 1 - b r, r += r (e + e^2)
MR3_HD double rcp(double b) {
    double r = rcp_seed(b);
    double e = fma_rn(-b, r, 1.0);
    return fma_rn(fma_rn(e, e, e), r, r);
}

// reciprocal to ~2^-44 relative (one quadratic Newton step): for the prefix norms W, V of
// the twisted factorizations (reading R9), which only feed ||z||^2 of the RQ correction and
// the stopping test -- a relative error of n 2^-43 there moves the corrected shift by that
// fraction of the correction, far below the dd accuracy the next pass needs
MR3_HD double rcp_w(double b) {
    const double r = rcp_seed(b);
    return fma_rn(r, fma_rn(-b, r, 1.0), r);
}

// a / b to ~1 ulp with one residual correction (fp64-internal mode)
MR3_HD double div(double a, double b) {
    double r = rcp(b);
    double q = mul_rn(a, r);
    return fma_rn(r, fma_rn(-q, b, a), q);
}

// ------------------------------------------------------------ fp64 "R" overloads
MR3_HD double add(double a, double b) { return add_rn(a, b); }
MR3_HD double sub(double a, double b) { return sub_rn(a, b); }
MR3_HD double mul(double a, double b) { return mul_rn(a, b); }
MR3_HD double neg(double a) { return -a; }
MR3_HD double half(double a) { return 0.5 * a; }
MR3_HD double hi(double a) { return a; }
MR3_HD double lo_part(double) { return 0.0; }
MR3_HD bool is_neg(double a) { return a < 0.0; }
MR3_HD bool lt(double a, double b) { return a < b; }
MR3_HD double absd(double a) { return fabs(a); }
MR3_HD double sqrt_r(double a) { return sqrt(a); }

// ------------------------------------------------------------ double-double
struct dd {
    double hi, lo;
};

MR3_HD double two_sum(double a, double b, double &e) {
    double s = add_rn(a, b);
    double bb = sub_rn(s, a);
    e = add_rn(sub_rn(a, sub_rn(s, bb)), sub_rn(b, bb));
    return s;
}
MR3_HD double quick_two_sum(double a, double b, double &e) {  // |a| >= |b|
    double s = add_rn(a, b);
    e = sub_rn(b, sub_rn(s, a));
    return s;
}
MR3_HD dd mkdd(double h, double l) {
    dd r;
    r.hi = h;
    r.lo = l;
    return r;
}
MR3_HD dd add(dd a, dd b) {  // sloppy pair addition
    double e;
    double s = two_sum(a.hi, b.hi, e);
    e = add_rn(e, add_rn(a.lo, b.lo));
    double l;
    s = quick_two_sum(s, e, l);
    return mkdd(s, l);
}
MR3_HD dd add_ieee(dd a, dd b) {  // accurate pair addition (QD "ieee_add")
    double s2, t2;
    double s1 = two_sum(a.hi, b.hi, s2);
    double t1 = two_sum(a.lo, b.lo, t2);
    s2 = add_rn(s2, t1);
    s1 = quick_two_sum(s1, s2, s2);
    s2 = add_rn(s2, t2);
    s1 = quick_two_sum(s1, s2, s2);
    return mkdd(s1, s2);
}
MR3_HD dd neg(dd a) { return mkdd(-a.hi, -a.lo); }
MR3_HD dd sub(dd a, dd b) { return add(a, neg(b)); }
MR3_HD dd add(dd a, double b) {
    double e;
    double s = two_sum(a.hi, b, e);
    e = add_rn(e, a.lo);
    double l;
    s = quick_two_sum(s, e, l);
    return mkdd(s, l);
}
MR3_HD dd mul(dd a, dd b) {
    double p = mul_rn(a.hi, b.hi);
    double e = fma_rn(a.hi, b.hi, -p);
    e = fma_rn(a.hi, b.lo, e);
    e = fma_rn(a.lo, b.hi, e);
    double l;
    p = quick_two_sum(p, e, l);
    return mkdd(p, l);
}
MR3_HD dd mul(dd a, double b) {
    double p = mul_rn(a.hi, b);
    double e = fma_rn(a.hi, b, -p);
    e = fma_rn(a.lo, b, e);
    double l;
    p = quick_two_sum(p, e, l);
    return mkdd(p, l);
}
// a / b: q1 = a.hi / b.hi (1 ulp), exact residual a - q1 b, q2 = residual / b.hi
MR3_HD dd div(dd a, dd b) {
    double r = rcp(b.hi);
    double q1 = mul_rn(a.hi, r);
    double p = mul_rn(q1, b.hi);
    double pe = fma_rn(q1, b.hi, -p);  // q1*b.hi = p + pe exactly
    double rem = sub_rn(a.hi, p);      // exact (Sterbenz)
    rem = add_rn(sub_rn(rem, pe), a.lo);
    rem = fma_rn(-q1, b.lo, rem);
    double q2 = mul_rn(rem, r);
    double l;
    double h = quick_two_sum(q1, q2, l);
    return mkdd(h, l);
}
// a * b + c in pair arithmetic (one two-prod, one two-sum; error ~ eps_y (|a b| + |c|))
MR3_HD dd fma_dd(dd a, dd b, dd c) {
    double p = mul_rn(a.hi, b.hi);
    double e = fma_rn(a.hi, b.hi, -p);
    e = fma_rn(a.hi, b.lo, e);
    e = fma_rn(a.lo, b.hi, e);
    double s2;
    double s = two_sum(p, c.hi, s2);
    s2 = add_rn(s2, add_rn(e, c.lo));
    double l;
    s = quick_two_sum(s, s2, l);
    return mkdd(s, l);
}
MR3_HD double fma_dd(double a, double b, double c) { return fma_rn(a, b, c); }
// a x + b y in pair arithmetic: two two-prods, one two-sum (error ~ eps_y (|a x| + |b y|));
// the two products are independent, so its dependent chain is one product + one two-sum
MR3_HD dd dot2_dd(dd a, dd x, dd b, dd y) {
    const double p1 = mul_rn(a.hi, x.hi), p2 = mul_rn(b.hi, y.hi);
    double e1 = fma_rn(a.hi, x.hi, -p1), e2 = fma_rn(b.hi, y.hi, -p2);
    e1 = fma_rn(a.hi, x.lo, e1);
    e2 = fma_rn(b.hi, y.lo, e2);
    e1 = fma_rn(a.lo, x.hi, e1);
    e2 = fma_rn(b.lo, y.hi, e2);
    double es;
    const double s = two_sum(p1, p2, es);
    const double t = add_rn(es, add_rn(e1, e2));
    double l;
    const double h = quick_two_sum(s, t, l);
    return mkdd(h, l);
}
MR3_HD double dot2_dd(double a, double x, double b, double y) { return fma_rn(a, x, mul_rn(b, y)); }
// exact scaling by a power of two
MR3_HD dd scale_pow2(dd a, double sc) { return mkdd(mul_rn(a.hi, sc), mul_rn(a.lo, sc)); }
MR3_HD double scale_pow2(double a, double sc) { return mul_rn(a, sc); }
MR3_HD dd half(dd a) { return mkdd(0.5 * a.hi, 0.5 * a.lo); }
MR3_HD double hi(dd a) { return a.hi; }
MR3_HD double lo_part(dd a) { return a.lo; }
MR3_HD bool is_neg(dd a) { return a.hi < 0.0; }
MR3_HD bool lt(dd a, dd b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }
MR3_HD double absd(dd a) { return fabs(a.hi); }
MR3_HD dd sqrt_r(dd a) {  // one Newton step on the fp64 root
    if (a.hi <= 0.0) return mkdd(0.0, 0.0);
    double s = sqrt(a.hi);
    double e = fma_rn(-s, s, a.hi);
    e = add_rn(e, a.lo);
    double c = e / (2.0 * s);
    double l;
    double h = quick_two_sum(s, c, l);
    return mkdd(h, l);
}

// R construction from a double, uniformly for both types
template <class R>
MR3_HD R mk(double x);
template <>
MR3_HD double mk<double>(double x) {
    return x;
}
template <>
MR3_HD dd mk<dd>(double x) {
    return mkdd(x, 0.0);
}

template <class R>
MR3_HD R mk2(double h, double l);
template <>
MR3_HD double mk2<double>(double h, double l) {
    return h + l;
}
template <>
MR3_HD dd mk2<dd>(double h, double l) {
    return mkdd(h, l);
}

// unit roundoff of the internal precision (eps_y)
template <class R>
struct Prec;
template <>
struct Prec<double> {
    static constexpr double eps = 1.1102230246251565e-16;  // 2^-53
    static constexpr int words = 1;                         // doubles per R
};
template <>
struct Prec<dd> {
    static constexpr double eps = 4.930380657631324e-32;  // 2^-104
    static constexpr int words = 2;
};

}  // namespace mr3
