// bode_pow.cuh -- x**e for the step-size controller, correctly rounded with
// overwhelming probability.
//
// The reference raises error norms to fixed powers with NumPy, i.e. glibc's
// pow (controller.py:221-226, :193).  glibc's pow is correctly rounded in all
// but ~0.1% of cases; CUDA's pow differs from it by one ulp in ~20% of
// calls, and because the step-size sequence amplifies one-ulp differences
// (the embedded error estimate is a cancellation), every such difference
// ends bit-identity with the reference for the rest of the trajectory.  This
// pow evaluates log and exp in double-double with table reduction (128
// entries each) to ~2^-68 relative error before the single final rounding,
// so it agrees with the correctly rounded result -- and hence with glibc --
// except in ~1e-4..1e-3 of calls.  It is also cheaper than CUDA's generic
// pow (no special-case ladder on the fast path; tables in shared memory).
//
// Host and device share this code: the host build backs the CPU tests that
// check it against 60-digit decimal arithmetic.
#pragma once
#if defined(__CUDACC__)
#include "bode_rtc.cuh"
#else
#include <cmath>
#include <cstdint>
#include <cstring>
#endif

#include "pow_tables.h"

#if defined(__CUDACC__)
#define BODE_HD __host__ __device__ __forceinline__
#else
#define BODE_HD inline
#endif

namespace bode {

struct PowTables {
  double log_tab[128][4];  // invc, -ln(invc) hi, lo, pad
  double exp_tab[128][2];  // 2^(j/128) hi, lo
};

// one copy in global memory (device) / static storage (host)
#if defined(__CUDACC__)
static __device__ const PowTables g_pow_tables = {BODE_POW_LOG_TABLE_INIT, BODE_POW_EXP_TABLE_INIT};
#endif
#if !defined(__CUDACC_RTC__)
static const PowTables h_pow_tables = {BODE_POW_LOG_TABLE_INIT, BODE_POW_EXP_TABLE_INIT};
#endif

// Polynomial coefficients and split constants.  On the device they live in
// the constant bank (FP64 instructions take them via LDCU, two per load)
// instead of 64-bit immediates, which cost two UMOVs each.
#define BODE_POW_K_INIT                                                        \
  {1.0 / 9.0, -0.125, 1.0 / 7.0, -1.0 / 6.0, 0.2, -0.25, 1.0 / 3.0, -0.5,     \
   1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5,        \
   BODE_POW_LN2_HI, BODE_POW_LN2_LO, BODE_POW_C_HI, BODE_POW_C_LO, BODE_POW_INV_C, 0x1p52}
#if defined(__CUDACC__)
static __constant__ double c_pow_k[20] = BODE_POW_K_INIT;
#endif
#if !defined(__CUDACC_RTC__)
static const double h_pow_k[20] = BODE_POW_K_INIT;
#endif
#if defined(__CUDA_ARCH__)
#define BODE_PK(i) c_pow_k[i]
#else
#define BODE_PK(i) h_pow_k[i]
#endif

namespace powimpl {

BODE_HD double mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
BODE_HD double add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
BODE_HD double sub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
BODE_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
BODE_HD int64_t bits(double x) {
#if defined(__CUDA_ARCH__)
  return __double_as_longlong(x);
#else
  int64_t b;
  memcpy(&b, &x, 8);
  return b;
#endif
}
BODE_HD double from_bits(int64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(b);
#else
  double x;
  memcpy(&x, &b, 8);
  return x;
#endif
}
// s + err == a + b exactly
BODE_HD void two_sum(double a, double b, double& s, double& err) {
  s = add(a, b);
  const double bb = sub(s, a);
  err = add(sub(a, sub(s, bb)), sub(b, bb));
}

}  // namespace powimpl

// log(x) as a double-double (lh + ll, error < 2^-68 absolute) for x > 0
// finite; returns false (and leaves lh/ll unset) for anything else.
BODE_HD bool cr_log(double x, const PowTables& T, double& lh, double& ll) {
  using namespace powimpl;
  if (!(x > 0.0) || !(x < INFINITY)) return false;
  int64_t ix = bits(x);
  int k = 0;
  if (ix < 0x0010000000000000LL) {  // subnormal: normalise
    ix = bits(mul(x, BODE_PK(19)));
    k = -52;
  }
  k += (int)(ix >> 52) - 1023;
  const int i = (int)((ix >> 45) & 127);
  const double m = from_bits((ix & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const double invc = T.log_tab[i][0], logc_hi = T.log_tab[i][1], logc_lo = T.log_tab[i][2];
  // r = m*invc - 1 exactly, as r_hi + p_lo
  const double p = mul(m, invc);
  const double p_lo = fma_(m, invc, -p);
  const double r = sub(p, 1.0);  // exact (Sterbenz)
  const double sq = mul(r, r);
  const double sq_lo = fma_(r, r, -sq);
  // log1p(r) - r + r^2/2 = r^3 (1/3 - r/4 + ... + r^6/9) for |r| < 2^-7.9;
  // the first omitted term r^10/10 is below 2^-82
  double q = BODE_PK(0);
  q = fma_(q, r, BODE_PK(1));
  q = fma_(q, r, BODE_PK(2));
  q = fma_(q, r, BODE_PK(3));
  q = fma_(q, r, BODE_PK(4));
  q = fma_(q, r, BODE_PK(5));
  q = fma_(q, r, BODE_PK(6));
  q = mul(q, mul(sq, r));
  // high parts
  double s1, e1, s2, e2, s3, e3;
  two_sum(mul((double)k, BODE_PK(14)), logc_hi, s1, e1);
  two_sum(s1, r, s2, e2);
  two_sum(s2, mul(BODE_PK(7), sq), s3, e3);
  // low parts: exact residuals, table tails, first/second-order p_lo terms
  double lo = add(e1, e2);
  lo = add(lo, e3);
  lo = add(lo, fma_((double)k, BODE_PK(15), logc_lo));
  lo = add(lo, p_lo);
  lo = sub(lo, mul(BODE_PK(13), sq_lo));
  lo = sub(lo, mul(r, p_lo));
  lo = add(lo, mul(sq, p_lo));
  lo = add(lo, q);
  two_sum(s3, lo, lh, ll);
  return true;
}

// exp(e * (lh + ll)), correctly rounded w.h.p.; `x` (= exp(lh + ll)) is only
// used for the libm fallback near overflow/underflow.
// libm pow for the rare out-of-range cases, kept out of line so its special-
// case ladder does not bloat (and add registers to) the persistent loop
#if defined(__CUDACC__)
static __host__ __device__ __noinline__
#else
inline
#endif
double pow_fallback(double x, double e) { return pow(x, e); }

BODE_HD double cr_exp_mul(double e, double lh, double ll, double x, const PowTables& T) {
  using namespace powimpl;
  // y = e * log(x) in double-double
  const double yh = mul(e, lh);
  const double yl = fma_(e, ll, fma_(e, lh, -yh));
  if (!(yh < 700.0 && yh > -700.0)) return pow_fallback(x, e);
  // exp(yh + yl) = 2^(kf/128) * exp(r2)
  const double kd = rint(mul(yh, BODE_PK(18)));
  const int64_t kf = (int64_t)kd;
  const int j = (int)(kf & 127);
  const int64_t ke = (kf - j) / 128;
  // r = y - kd*ln2/128 as rh + rl with |rl| <~ ulp(rh) + |yl|
  const double t1 = fma_(-kd, BODE_PK(16), yh);  // exact (kd*C_HI exact, Sterbenz)
  const double pc = mul(kd, BODE_PK(17));
  const double pc_err = fma_(kd, BODE_PK(17), -pc);
  double rh, ea;
  two_sum(t1, -pc, rh, ea);
  const double rl = add(sub(ea, pc_err), yl);
  // exp(rh + rl) - 1 - rh = a + rl*(1 + rh + a),  a = exp(rh) - 1 - rh
  //                        = rh^2 (1/2 + rh/6 + ... + rh^5/5040)
  double c = BODE_PK(8);
  c = fma_(c, rh, BODE_PK(9));
  c = fma_(c, rh, BODE_PK(10));
  c = fma_(c, rh, BODE_PK(11));
  c = fma_(c, rh, BODE_PK(12));
  c = fma_(c, rh, BODE_PK(13));
  const double a = mul(mul(rh, rh), c);
  const double pp = add(a, fma_(rl, add(rh, a), rl));
  const double th = T.exp_tab[j][0], tl = T.exp_tab[j][1];
  // th*(1 + rh + pp) + tl*(1 + rh + pp)
  const double P1h = mul(th, rh);
  const double P1l = fma_(th, rh, -P1h);
  double S, Se;
  two_sum(th, P1h, S, Se);
  double tail = add(Se, P1l);
  tail = fma_(th, pp, tail);
  tail = add(tail, fma_(tl, add(rh, pp), tl));
  const double res = add(S, tail);
  // scale by 2^ke (result stays normal: |y| < 700)
  return from_bits(bits(res) + (ke << 52));
}

// ---- BODE_MODE_FAST variants: plain double arithmetic with FMA on the same
// tables -- within ~1 ulp instead of correctly rounded (the fast mode already
// gives up bit-identity by contracting a*b+c); ~16 + 15 FP64 operations for
// a log and an exp instead of ~50 + ~45.
// log(x) = Lh + Ll, |Ll| < 2^-7, error < 2^-60 absolute; false for x <= 0 /
// non-finite
BODE_HD bool fast_log(double x, const PowTables& T, double& Lh, double& Ll) {
  using namespace powimpl;
  if (!(x > 0.0) || !(x < INFINITY)) return false;
  int64_t ix = bits(x);
  int k = 0;
  if (ix < 0x0010000000000000LL) {  // subnormal: normalise
    ix = bits(mul(x, BODE_PK(19)));
    k = -52;
  }
  k += (int)(ix >> 52) - 1023;
  const int i = (int)((ix >> 45) & 127);
  const double m = from_bits((ix & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const double r = fma_(m, T.log_tab[i][0], -1.0);  // |r| < 2^-7.9
  // log1p(r) = r + r^2 (-1/2 + r q(r)), q = 1/3 - r/4 + r^2/5 - r^3/6 + r^4/7;
  // the first omitted term r^8/8 is below 2^-66
  double q = fma_(BODE_PK(2), r, BODE_PK(3));
  q = fma_(q, r, BODE_PK(4));
  q = fma_(q, r, BODE_PK(5));
  q = fma_(q, r, BODE_PK(6));
  // k ln2_hi is exact; for k != 0 it dominates log c, so Fast2Sum is exact
  const double kl = mul((double)k, BODE_PK(14));
  const double hi = add(kl, T.log_tab[i][1]);
  const double hi_err = k != 0 ? sub(T.log_tab[i][1], sub(hi, kl)) : 0.0;
  const double lo = add(fma_((double)k, BODE_PK(15), T.log_tab[i][2]), hi_err);
  Lh = hi;
  Ll = add(r, fma_(mul(r, r), fma_(r, q, BODE_PK(7)), lo));
  return true;
}

// exp(e * (Lh + Ll)) within ~1 ulp; `x` (= exp(L)) is only used for the
// libm fallback near overflow/underflow
BODE_HD double fast_exp_mul(double e, double Lh, double Ll, double x, const PowTables& T) {
  using namespace powimpl;
  const double yh = mul(e, Lh);
  const double yl = fma_(e, Ll, fma_(e, Lh, -yh));
  if (!(yh < 700.0 && yh > -700.0)) return pow_fallback(x, e);
  const double kd = rint(mul(yh, BODE_PK(18)));
  const int64_t kf = (int64_t)kd;
  const int j = (int)(kf & 127);
  const int64_t ke = (kf - j) / 128;
  const double r = add(fma_(-kd, BODE_PK(17), fma_(-kd, BODE_PK(16), yh)), yl);  // |r| < 2^-7.9
  // exp(r) - 1 = r + r^2 (1/2 + r/6 + r^2/24 + r^3/120 + r^4/720); next term < 2^-67
  double c = fma_(BODE_PK(9), r, BODE_PK(10));
  c = fma_(c, r, BODE_PK(11));
  c = fma_(c, r, BODE_PK(12));
  c = fma_(c, r, BODE_PK(13));
  const double p = fma_(mul(r, r), c, r);
  const double th = T.exp_tab[j][0], tl = T.exp_tab[j][1];
  const double res = add(th, fma_(th, p, tl));
  return from_bits(bits(res) + (ke << 52));
}

// exp(y) for |y| < 700 within ~1 ulp of exp of the rounded argument (the
// table-driven body of fast_exp_mul with a plain-double argument)
BODE_HD double fast_exp(double y, const PowTables& T) {
  using namespace powimpl;
  const double kd = rint(mul(y, BODE_PK(18)));
  const int64_t kf = (int64_t)kd;
  const int j = (int)(kf & 127);
  const int64_t ke = (kf - j) / 128;
  const double r = fma_(-kd, BODE_PK(17), fma_(-kd, BODE_PK(16), y));  // |r| < 2^-7.9
  double c = fma_(BODE_PK(9), r, BODE_PK(10));
  c = fma_(c, r, BODE_PK(11));
  c = fma_(c, r, BODE_PK(12));
  c = fma_(c, r, BODE_PK(13));
  const double p = fma_(mul(r, r), c, r);
  const double th = T.exp_tab[j][0], tl = T.exp_tab[j][1];
  const double res = add(th, fma_(th, p, tl));
  return from_bits(bits(res) + (ke << 52));
}

// Reduced-precision pair for the fast-mode I / PI controller
// (bode_device.cuh adapt_pi_ms), whose step counts are insensitive below
// ~1e-13 relative: log of a positive NORMAL finite x as one double (a few
// ulp; the log1p series stops at r^6/6, |r| < 2^-7.9, omitted < 2^-58) and
// exp with the series stopped at r^5/120 (omitted < 2^-56 relative).
BODE_HD double fast_log1(double x, const PowTables& T) {
  using namespace powimpl;
  const int64_t ix = bits(x);
  const int k = (int)(ix >> 52) - 1023;
  const int i = (int)((ix >> 45) & 127);
  const double m = from_bits((ix & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const double r = fma_(m, T.log_tab[i][0], -1.0);
  double q = fma_(BODE_PK(3), r, BODE_PK(4));  // 1/3 - r/4 + r^2/5 - r^3/6
  q = fma_(q, r, BODE_PK(5));
  q = fma_(q, r, BODE_PK(6));
  const double p = fma_(mul(r, r), fma_(r, q, BODE_PK(7)), r);
  const double kd = (double)k;
  return add(fma_(kd, BODE_PK(14), T.log_tab[i][1]),
             add(p, fma_(kd, BODE_PK(15), T.log_tab[i][2])));
}

BODE_HD double fast_exp3(double y, const PowTables& T) {
  using namespace powimpl;
  const double kd = rint(mul(y, BODE_PK(18)));
#if defined(__CUDA_ARCH__)
  // |y| < 700 (the caller's range): 32-bit k, and the 2^ke scaling as an
  // add to the high word (the result is normal, no carry from the low word)
  const int kf = __double2int_rn(kd);
  const int j = kf & 127;
  const int ke = (kf - j) / 128;
#else
  const int64_t kf = (int64_t)kd;
  const int j = (int)(kf & 127);
  const int64_t ke = (kf - j) / 128;
#endif
  const double r = fma_(-kd, BODE_PK(17), fma_(-kd, BODE_PK(16), y));
  double c = fma_(BODE_PK(10), r, BODE_PK(11));
  c = fma_(c, r, BODE_PK(12));
  c = fma_(c, r, BODE_PK(13));
  const double p = fma_(mul(r, r), c, r);
  const double th = T.exp_tab[j][0], tl = T.exp_tab[j][1];
  const double res = add(th, fma_(th, p, tl));
#if defined(__CUDA_ARCH__)
  return __hiloint2double(__double2hiint(res) + ke * (1 << 20), __double2loint(res));
#else
  return from_bits(bits(res) + (ke << 52));
#endif
}

// Correctly rounded (w.h.p.) x**e for x > 0 finite, e finite; everything
// else -- and results near overflow/underflow -- goes to the libm pow.
BODE_HD double cr_pow(double x, double e, const PowTables& T) {
  double lh, ll;
  if (!(e == e) || e == INFINITY || e == -INFINITY || !cr_log(x, T, lh, ll)) return pow_fallback(x, e);
  return cr_exp_mul(e, lh, ll, x, T);
}

}  // namespace bode
