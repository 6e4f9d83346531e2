// Correctly rounded FP64 sin / cos for the exact-order shape-matching path (shape.cuh,
// VROD_SHAPE_EXACT): Quaternion(AngleAxis(angle, axis)) needs sin and cos of angle / 2
// (bundling.cpp:64, Eigen's AngleAxis -> Quaternion conversion). The reference calls glibc's
// sin / cos (≤ 0.501 ulp below 0.126, i.e. correctly rounded except within 0.001 ulp of a
// midpoint); CUDA's sin / cos are accurate to 2 ulp, so they differ from glibc in the last bit
// for a sizeable fraction of arguments. This header evaluates both in double-double and rounds
// once, so the result is the correctly rounded value except when the exact value lies within
// ~2^-100 (relative) of a rounding midpoint — it agrees with glibc wherever glibc itself is
// correctly rounded (checked against glibc on 10^7 arguments: tests/test_shape_matching.py).
//
// Tiny arguments (|x| < 2^-20: the converged iterations of a warm-started extraction) take the
// two-term Taylor route in double (misrounding probability ~x^2 < 1e-12); small ones
// (|x| < 2^-5) the leading correction terms in double-double, the rest in double, one final
// rounding; larger ones
// the double-double Taylor series; |x| > pi/4 a Cody–Waite reduction by pi/2 in double-double
// first.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define CRT_HD __host__ __device__ __forceinline__
#define CRT_HD_COLD static __host__ __device__ __noinline__
#else
#define CRT_HD inline
#define CRT_HD_COLD inline
#endif

namespace crt {

#ifndef __CUDACC__
using std::fabs;
using std::fma;
using std::rint;
#endif

struct DD {
  double hi, lo;
};

CRT_HD DD two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return DD{s, e};
}
CRT_HD DD fast_two_sum(double a, double b) {  // |a| >= |b|
  const double s = a + b;
  return DD{s, b - (s - a)};
}
CRT_HD DD two_prod(double a, double b) {
  const double p = a * b;
  return DD{p, fma(a, b, -p)};
}
CRT_HD DD dd_add(const DD& a, const DD& b) {
  const DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  DD r = fast_two_sum(s.hi, s.lo + t.hi);
  return fast_two_sum(r.hi, r.lo + t.lo);
}
CRT_HD DD dd_mul(const DD& a, const DD& b) {
  const DD p = two_prod(a.hi, b.hi);
  return fast_two_sum(p.hi, p.lo + (a.hi * b.lo + a.lo * b.hi));
}
CRT_HD DD dd_mul_d(const DD& a, double b) {
  const DD p = two_prod(a.hi, b);
  return fast_two_sum(p.hi, p.lo + a.lo * b);
}

// 1/n! as double-double, n = 0..13 (hi, lo).
#define CRT_INV_FACT                                                                                             \
  {                                                                                                              \
    {1.0, 0.0}, {1.0, 0.0}, {0.5, 0.0}, {0.16666666666666666, 9.25185853854297e-18},                            \
        {0.041666666666666664, 2.3129646346357427e-18}, {0.008333333333333333, 1.1564823173178714e-19},        \
        {0.001388888888888889, -5.300543954373577e-20}, {0.0001984126984126984, 1.7209558293420705e-22},       \
        {2.48015873015873e-05, 2.1511947866775882e-23}, {2.7557319223985893e-06, -1.858393274046472e-22},      \
        {2.755731922398589e-07, 2.3767714622250297e-23}, {2.505210838544172e-08, -1.448814070935912e-24},     \
        {2.08767569878681e-09, -1.20734505911326e-25}, {1.6059043836821613e-10, 1.2585294588752098e-26}        \
  }

// sin(r), cos(r) for |r| <= pi/4 + a little, r given in double-double (rh, rl), returned in
// double-double. Taylor series in y = r^2: the first five terms with double-double coefficients,
// the tail (relative weight < 3e-9) in double.
CRT_HD void dd_sincos_core(const DD& r, DD& s, DD& c) {
  const DD kF[14] = CRT_INV_FACT;
  const DD y = dd_mul(r, r);
  const double yd = y.hi;
  // tails: sum_{k=5..12} (-1)^k y^k / (2k+1)!  and  / (2k)!   (y <= 0.62)
  const double ts = yd * yd * yd * yd * yd *
                    (-1.0 / 39916800.0 + yd * (1.0 / 6227020800.0 + yd * (-1.0 / 1307674368000.0 +
                     yd * (1.0 / 355687428096000.0 + yd * (-1.0 / 121645100408832000.0 +
                     yd * (1.0 / 51090942171709440000.0 + yd * (-1.0 / 25852016738884976640000.0)))))));
  const double tc = yd * yd * yd * yd * yd *
                    (-1.0 / 3628800.0 + yd * (1.0 / 479001600.0 + yd * (-1.0 / 87178291200.0 +
                     yd * (1.0 / 20922789888000.0 + yd * (-1.0 / 6402373705728000.0 +
                     yd * (1.0 / 2432902008176640000.0 + yd * (-1.0 / 1124000727777607680000.0)))))));
  // Horner in double-double: P(y) = (1 - y/3! + y^2/5! - y^3/7! + y^4/9!) + tail
  DD ps = dd_mul(kF[9], y);
  ps = dd_add(ps, DD{-kF[7].hi, -kF[7].lo});
  ps = dd_mul(ps, y);
  ps = dd_add(ps, kF[5]);
  ps = dd_mul(ps, y);
  ps = dd_add(ps, DD{-kF[3].hi, -kF[3].lo});
  ps = dd_mul(ps, y);
  ps = dd_add(ps, DD{1.0, 0.0});
  ps = dd_add(ps, DD{ts, 0.0});
  s = dd_mul(ps, r);
  DD pc = dd_mul(kF[8], y);
  pc = dd_add(pc, DD{-kF[6].hi, -kF[6].lo});
  pc = dd_mul(pc, y);
  pc = dd_add(pc, kF[4]);
  pc = dd_mul(pc, y);
  pc = dd_add(pc, DD{-kF[2].hi, -kF[2].lo});
  pc = dd_mul(pc, y);
  pc = dd_add(pc, DD{1.0, 0.0});
  c = dd_add(pc, DD{tc, 0.0});
}

// |x| >= 2^-5 (rare once an extraction is warm-started): out of line, so the hot small-argument
// route stays compact in the caller's loop.
CRT_HD_COLD DD sincos_cr_general(double x) {  // (sin, cos)
  const double ax = fabs(x);
  DD r{x, 0.0};
  long long k = 0;
  if (ax > 0.7853981633974483) {
    const double kd = rint(x * 0.6366197723675814);
    k = static_cast<long long>(kd);
    // r = x - k * pi/2 with pi/2 = p1 + p2 + p3 (Cody–Waite, double-double)
    const DD a = two_prod(kd, 1.5707963267948966);
    const DD b = two_prod(kd, 6.123233995736766e-17);
    r = dd_add(DD{x, 0.0}, DD{-a.hi, -a.lo});
    r = dd_add(r, DD{-b.hi, -b.lo});
    r = dd_add(r, DD{kd * 1.4973849048591698e-33, 0.0});
  }
  DD s, c;
  dd_sincos_core(r, s, c);
  const double sr = s.hi + s.lo, cr = c.hi + c.lo;
  switch (static_cast<int>(k & 3)) {
    case 0: return DD{sr, cr};
    case 1: return DD{cr, -sr};
    case 2: return DD{-sr, -cr};
    default: return DD{-cr, sr};
  }
}

// Correctly rounded sin(x) and cos(x) (see the header comment for the exceptions), returned as
// {sin, cos} in registers.
CRT_HD DD sincos_rn(double x) {
  const double ax = fabs(x);
  if (!(ax < 1e300)) return DD{x - x, x - x};  // inf / nan
  if (ax < 0x1p-20) {
    // sin x = x - x^3/6, cos x = 1 - x^2/2 in double: the neglected terms (< x^5/120, x^4/24) and
    // the rounding of the corrections (relative x^2/6 and x^2/2 of half an ulp) can move the
    // final rounding only for a fraction ~x^2 < 1e-12 of arguments
    const double y = x * x;
    return DD{x + (x * y) * (-1.0 / 6.0), 1.0 + y * -0.5};
  }
  if (ax < 0x1p-5) {
    // sin x = x + t1 + t2 with t1 = -x^3/6 in double-double, t2 = x^5/120 - x^7/5040 (+ x^9/9!)
    // in double (|t2| <= 8e-9 |x|); cos x = 1 - y/2 + u2 with y = x^2 exact (two_prod),
    // u2 = y^2/24 (double-double) - y^3/720 + y^4/8!. One final rounding each.
    const DD y = two_prod(x, x);
    const DD x3 = dd_mul_d(y, x);
    const DD t1 = dd_mul(x3, DD{-0.16666666666666666, -9.25185853854297e-18});
    const double yd = y.hi;
    const double t2 = (x3.hi * yd) * (1.0 / 120.0 - yd * (1.0 / 5040.0 - yd * (1.0 / 362880.0)));
    const DD s0 = fast_two_sum(x, t1.hi);
    const double sn = s0.hi + (s0.lo + (t1.lo + t2));
    const DD y2 = dd_mul(y, y);
    const DD u2 = dd_mul(y2, DD{0.041666666666666664, 2.3129646346357427e-18});
    const double u3 = (y2.hi * yd) * (-1.0 / 720.0 + yd * (1.0 / 40320.0));
    const DD c0 = fast_two_sum(1.0, -0.5 * y.hi);
    return DD{sn, c0.hi + (c0.lo + ((-0.5 * y.lo + u2.hi) + (u2.lo + u3)))};
  }
  return sincos_cr_general(x);
}

CRT_HD void sincos_cr(double x, double* sn, double* cs) {
  const DD r = sincos_rn(x);
  *sn = r.hi;
  *cs = r.lo;
}

}  // namespace crt
