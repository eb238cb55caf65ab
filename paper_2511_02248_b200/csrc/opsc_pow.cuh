// x ** e for the interference factor (perfmodel.py:174-187, `excess **
// params.exponent`), rounded to nearest from a double-double evaluation.
//
// The reference's `**` is glibc's pow (<= 0.52 ulp); libdevice's pow is
// <= 2 ulp and differs from it in ~16% of random (excess, exponent) draws
// (tools/pow_probe.py). Evaluating exp(e * log(x)) in double-double arithmetic
// (relative error ~2^-97 before the final rounding) returns the correctly
// rounded value except within ~2^-44 ulp of a rounding midpoint, which
// matches glibc wherever glibc itself rounds correctly (all but ~0.1% of
// draws). The exponents 1, 2 and 0.5 keep their exact forms in k_place.cu.
//
// Plain C++ on the host (tests/test_pow.py compiles it with g++ and checks it
// against a 60-digit decimal evaluation), __host__ __device__ under nvcc.
#pragma once
#include <math.h>

#ifdef __CUDACC__
#define OPSC_HD __host__ __device__ __forceinline__
#define OPSC_HD_CALL __host__ __device__ __noinline__  // out of line: no register cost at the call sites
#else
#define OPSC_HD static inline
#define OPSC_HD_CALL static inline
#endif

namespace opsc_pow {

struct dd {
  double hi, lo;
};

OPSC_HD dd two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
OPSC_HD dd fast_two_sum(double a, double b) {  // |a| >= |b| (or a == 0)
  const double s = a + b;
  return {s, b - (s - a)};
}
OPSC_HD dd add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s = fast_two_sum(s.hi, s.lo + t.hi);
  return fast_two_sum(s.hi, s.lo + t.lo);
}
OPSC_HD dd mul(dd a, dd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return fast_two_sum(p, e);
}
OPSC_HD dd mul_d(dd a, double b) {
  const double p = a.hi * b;
  return fast_two_sum(p, fma(a.lo, b, fma(a.hi, b, -p)));
}

// e^r - 1 for |r| <= 0.35: Taylor to r'^9 at r' = r / 256 (coefficients up
// to 1/5! in double-double), then (1 + q)^256 - 1 by eight q <- q (2 + q).
OPSC_HD dd expm1_small(dd r) {
  const dd s = {r.hi * 0x1p-8, r.lo * 0x1p-8};
  dd p = {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73};  // 1/9!
  p = add(mul(p, s), dd{0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76});  // 1/8!
  p = add(mul(p, s), dd{0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73});  // 1/7!
  p = add(mul(p, s), dd{0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65});  // 1/6!
  p = add(mul(p, s), dd{0x1.1111111111111p-7, 0x1.1111111111111p-63});   // 1/5!
  p = add(mul(p, s), dd{0x1.5555555555555p-5, 0x1.5555555555555p-59});   // 1/4!
  p = add(mul(p, s), dd{0x1.5555555555555p-3, 0x1.5555555555555p-57});   // 1/3!
  p = add(mul(p, s), dd{0.5, 0.0});
  p = add(mul(p, s), dd{1.0, 0.0});
  dd q = mul(p, s);
  for (int i = 0; i < 8; ++i) q = mul(q, add(dd{2.0, 0.0}, q));
  return q;
}

constexpr double kLn2Hi = 0x1.62e42fefa39efp-1, kLn2Lo = 0x1.abc9e3b39803fp-56;

// log(x) for a positive normal finite x: x = m 2^k, m in [sqrt(1/2), sqrt(2)),
// y0 = log(m) refined by one Newton step on exp: log m = y0 + log(m e^-y0).
OPSC_HD dd log_dd(double x) {
  int k;
  double m = frexp(x, &k);  // [0.5, 1)
  if (m < 0.70710678118654752) {
    m *= 2.0;
    --k;
  }
  const double y0 = log(m);
  const dd q = expm1_small(dd{-y0, 0.0});          // e^-y0 - 1
  dd u = add(dd{m - 1.0, 0.0}, mul_d(q, m));       // m e^-y0 - 1 (m - 1 exact: Sterbenz)
  u = add(u, dd{-0.5 * u.hi * u.hi, 0.0});         // log(1 + u), |u| ~ 2^-52
  const dd lm = add(dd{y0, 0.0}, u);
  return add(mul_d(dd{kLn2Hi, kLn2Lo}, (double)k), lm);
}

// e^z for |z.hi| <= 708 (normal, finite result), rounded to nearest.
OPSC_HD double exp_dd(dd z) {
  const double n = rint(z.hi * 0x1.71547652b82fep0);
  const dd r = add(z, mul_d(dd{-kLn2Hi, -kLn2Lo}, n));
  const dd q = expm1_small(r);
  dd one = two_sum(1.0, q.hi);
  one = fast_two_sum(one.hi, one.lo + q.lo);
  return ldexp(one.hi, (int)n);
}

OPSC_HD_CALL double pow_rn(double x, double e) {
  if (e == 0.0 || x == 1.0) return 1.0;
  if (!(x >= 0x1p-1022) || !(x <= 1.7976931348623157e308) || !(fabs(e) <= 1.7976931348623157e308))
    return pow(x, e);  // zero, subnormal, inf, NaN: the library's special cases
  const dd z = mul_d(log_dd(x), e);
  if (!(fabs(z.hi) <= 708.0)) return pow(x, e);  // overflow / underflow range
  return exp_dd(z);
}

}  // namespace opsc_pow
