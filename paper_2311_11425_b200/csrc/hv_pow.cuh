// x^y for the equation of state (state.py:84-101: P = P_A (R Theta / P_A)^gamma), x > 0.
//
// CUDA's pow() costs ~380 instructions per call in the Euler column sweep (a third of the kernel's
// issue slots: special-case handling, integer-y tests, 32-bit IMAD shuffles of the halves, spills
// under the 64-register cap).  The EOS argument is a positive normal number, so this version keeps
// only the arithmetic: log(x) as a double-double (x = m 2^e, s = (m - 1)/(m + 1) with its division
// residual, log m = 2 atanh s), the product with y as a double-double, exp with the low part folded
// into the reduced argument.  ~65 FP64 operations, no branches on the fast path.  Measured against
// glibc's pow on the host (tests/test_hv_pow.py compiles this header with g++): <= 1 ulp, i.e. at
// least as close to the reference's numpy/glibc result as CUDA's pow (2 ulp bound).  Arguments
// outside [2^-500, 2^500], non-finite or non-positive, or |y log x| > 600 take the library pow().
//
// The same source compiles for the host (fma() from <cmath>), so the CPU test pins the exact
// operation sequence the device executes: every step is an explicit IEEE operation (no contraction).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define HV_POW_HD __host__ __device__ __forceinline__
#else
#define HV_POW_HD inline
#endif

namespace hv {

HV_POW_HD double pw_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
HV_POW_HD double pw_mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;   // no contraction into a neighbouring add
  return r;
#endif
}
HV_POW_HD double pw_add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
HV_POW_HD double pw_rcp(double a) {
#if defined(__CUDA_ARCH__)
  return __drcp_rn(a);
#else
  return 1.0 / a;
#endif
}
HV_POW_HD int64_t pw_bits(double a) {
#if defined(__CUDA_ARCH__)
  return __double_as_longlong(a);
#else
  int64_t b;
  std::memcpy(&b, &a, 8);
  return b;
#endif
}
HV_POW_HD double pw_double(int64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(b);
#else
  double a;
  std::memcpy(&a, &b, 8);
  return a;
#endif
}

// polynomial coefficients: on the device in constant memory, so that the FMAs take them as constant-bank
// operands (as immediates every 64-bit coefficient costs two uniform-register moves: ~45 extra issue slots
// per call)
#if defined(__CUDACC__)
#define HV_POW_TAB static __constant__ double
#else
#define HV_POW_TAB static const double
#endif
HV_POW_TAB pw_log_c[11] = {2.0 / 23.0, 2.0 / 21.0, 2.0 / 19.0, 2.0 / 17.0, 2.0 / 15.0, 2.0 / 13.0,
                           2.0 / 11.0, 2.0 / 9.0,  2.0 / 7.0,  2.0 / 5.0,  2.0 / 3.0};
HV_POW_TAB pw_exp_c[12] = {1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
                           1.0 / 362880.0,     1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,
                           1.0 / 120.0,        1.0 / 24.0,        1.0 / 6.0,        0.5};
#if defined(__CUDACC__) && !defined(__CUDA_ARCH__)
// host pass of a .cu file: the tables are device symbols; the host functions below are never called there
#define HV_POW_C(tab, i) 0.0
#else
#define HV_POW_C(tab, i) tab[i]
#endif

// a / b with rb = the correctly rounded reciprocal of b (__drcp_rn; 1.0 / b on the host): a rb, then one
// exact-residual correction (Markstein's theorem: the result is the correctly rounded quotient barring
// over/underflow, i.e. what IEEE division gives; hv_probe_div counts the differences from a / b on the
// device).  The compiler's out-of-line division routine cost ~40 instructions per quotient in the Euler
// column sweep (16 % of its instructions for five quotients per node); this is 3 per quotient after one
// reciprocal per divisor.
HV_POW_HD double div_rcp(double a, double b, double rb) {
  const double q = pw_mul(a, rb);
  const double e = pw_fma(-q, b, a);
  return pw_fma(e, rb, q);
}

// fast path: x a positive normal in [2^-500, 2^500], |y log x| <= 600 (checked by pow_pos)
HV_POW_HD double pow_pos_core(double x, double y, bool* ok) {
  const double LN2_HI = 6.93147180369123816490e-01;   // 0x3fe62e42fee00000: 21 trailing zero bits x ... exact e * LN2_HI
  const double LN2_LO = 1.90821492927058770002e-10;   // ln 2 - LN2_HI
  const double LOG2E = 1.44269504088896338700e+00;
  // x = m 2^e, m in [sqrt(1/2), sqrt(2))
  const int64_t xb = pw_bits(x);
  int e = (int)(xb >> 52) - 1023;
  double m = pw_double((xb & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  if (m > 1.4142135623730951) {
    m = pw_mul(m, 0.5);
    e += 1;
  }
  // s = (m - 1) / (m + 1) = s_hi + s_lo
  const double num = pw_add(m, -1.0);                       // exact
  const double den = pw_add(m, 1.0);
  const double den_lo = pw_add(m, -pw_add(den, -1.0));      // exact rounding error of den
  const double r = pw_rcp(den);
  const double s_hi = pw_mul(num, r);
  double res = pw_fma(-s_hi, den, num);
  res = pw_fma(-s_hi, den_lo, res);
  const double s_lo = pw_mul(res, r);
  // log m = 2 s + s^3 (2/3 + 2/5 s^2 + ... + 2/23 s^20)
  const double s2 = pw_mul(s_hi, s_hi);
  double p = HV_POW_C(pw_log_c, 0);
#pragma unroll
  for (int i = 1; i < 11; ++i) p = pw_fma(p, s2, HV_POW_C(pw_log_c, i));
  const double s3 = pw_mul(s2, s_hi);
  const double lm_hi = pw_add(s_hi, s_hi);
  // d(2 atanh s)/ds = 2 / (1 - s^2): the low part of s enters as 2 s_lo (1 + s^2)
  const double lm_lo = pw_fma(s3, p, pw_mul(pw_add(s_lo, s_lo), pw_add(1.0, s2)));
  // log x = e ln 2 + log m = L_hi + L_lo
  const double ed = (double)e;
  const double a_hi = pw_mul(ed, LN2_HI);                   // exact
  const double L_hi = pw_add(a_hi, lm_hi);
  double L_lo = pw_add(pw_add(a_hi, -L_hi), lm_hi);         // exact (|a_hi| >= |lm_hi| or a_hi == 0)
  L_lo = pw_add(L_lo, pw_fma(ed, LN2_LO, lm_lo));
  // t = y log x = t_hi + t_lo
  const double t_hi = pw_mul(y, L_hi);
  const double t_lo = pw_fma(y, L_lo, pw_fma(y, L_hi, -t_hi));
  *ok = fabs(t_hi) <= 600.0;
  // exp(t): t = k ln 2 + rr (k = 0 when the caller will discard the result)
  const double kd = *ok ? rint(pw_mul(t_hi, LOG2E)) : 0.0;
  const double rr_hi = pw_fma(-kd, LN2_HI, t_hi);            // exact
  const double rr_lo = pw_fma(-kd, LN2_LO, t_lo);
  const double rr = pw_add(rr_hi, rr_lo);
  double q = HV_POW_C(pw_exp_c, 0);                         // 1/13!, ..., 1/2
#pragma unroll
  for (int i = 1; i < 12; ++i) q = pw_fma(q, rr, HV_POW_C(pw_exp_c, i));
  // exp(rr) = (1 + rr_hi) + (rr_lo + rr^2 q), the first sum with its rounding error carried
  const double w = pw_fma(pw_mul(rr, rr), q, rr_lo);
  const double hi = pw_add(1.0, rr_hi);
  const double er = pw_add(pw_add(1.0, -hi), rr_hi);        // exact (|rr_hi| < 1)
  const double ex = pw_add(hi, pw_add(er, w));
  return pw_double(pw_bits(ex) + ((int64_t)(int)kd << 52));
}

#if defined(__CUDACC__)
static __device__ __noinline__ double pow_slow(double x, double y) { return pow(x, y); }
#endif

// x^y, x > 0 expected (the EOS argument); anything the fast path does not cover goes to pow()
HV_POW_HD double pow_pos(double x, double y) {
#if defined(__CUDACC__) && !defined(__CUDA_ARCH__)
  return std::pow(x, y);   // host pass of a .cu file: the coefficient tables are device symbols
#else
  bool ok = false;
  const int ex = (int)(pw_bits(x) >> 52);   // sign and exponent: 523 .. 1523 <=> positive, 2^-500 <= x < 2^501
  const double v = pow_pos_core(x, y, &ok);
  if (ex >= 523 && ex <= 1523 && ok) return v;
#if defined(__CUDA_ARCH__)
  return pow_slow(x, y);
#else
  return std::pow(x, y);
#endif
#endif
}

}  // namespace hv
