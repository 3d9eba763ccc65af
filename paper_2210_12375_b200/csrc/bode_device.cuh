// bode_device.cuh -- device-side numerics shared by the persistent solver
// and the unit-op kernels.  Every function restates one reference function
// (paths relative to /root/reference/pkg/src/batchode/) in the reference's
// NumPy operation order; Ops selects exact (separately rounded IEEE ops,
// SURVEY.md Appendix A) or fast (FMA-contracted) arithmetic.
#pragma once
#include "bode_rtc.cuh"

#include "../../include/bode.h"
#include "bode_pow.cuh"
#include "tableau_coeffs.h"

namespace bode {

// ----------------------------------------------------------------- ops --
struct ExactOps {
  static constexpr bool kFast = false;
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  // (a*b)+c with two roundings, as NumPy evaluates it
  static __device__ __forceinline__ double mad(double a, double b, double c) {
    return __dadd_rn(__dmul_rn(a, b), c);
  }
};

// Fast mode fuses exactly where the code says so (mad, explicit fma) and
// nowhere else: mul/add/sub are round-to-nearest intrinsics, which the
// compiler may not contract.  Implicit contraction is decided per
// instantiation (it depends on register allocation), so without this the
// trajectory-recording instantiation of the solver could round differently
// from the plain one.
struct FastOps {
  static constexpr bool kFast = true;
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mad(double a, double b, double c) { return fma(a, b, c); }
};

__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// np.maximum / np.minimum: NaN-propagating (unlike fmax/fmin).  a NaN -> a;
// b NaN (a not) -> the comparison is false -> b; otherwise the ordinary max.
__device__ __forceinline__ double np_max(double a, double b) {
  return (a >= b || a != a) ? a : b;
}
__device__ __forceinline__ double np_min(double a, double b) {
  return (a <= b || a != a) ? a : b;
}

// array ** python-float the way NumPy evaluates it (fast_scalar_power
// short-cuts for 0, +-1, 2, 0.5; controller.py:221-226, :193)
__device__ __forceinline__ double np_scalar_pow(double x, double e,
                                                const PowTables& T = g_pow_tables) {
  if (e == 0.0) return 1.0;
  if (e == 1.0) return x;
  if (e == -1.0) return ddiv(1.0, x);
  if (e == 2.0) return __dmul_rn(x, x);
  if (e == 0.5) return dsqrt(x);
  return cr_pow(x, e, T);  // correctly rounded w.h.p. (bode_pow.cuh)
}

// NumPy pairwise_sum (umath loops_utils.h.src) seeded with 0.0, which is the
// reduction order of np.mean(..., axis=1) on a C-contiguous row.
template <int N, class O>
__device__ __forceinline__ double pairwise_sum(const double* a) {
  if constexpr (N < 8) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < N; i++) r = O::add(r, a[i]);
    return r;
  } else if constexpr (N <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a[j];
#pragma unroll
    for (int i = 8; i < N - (N % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; j++) r[j] = O::add(r[j], a[i + j]);
    }
    double res = O::add(O::add(O::add(r[0], r[1]), O::add(r[2], r[3])),
                        O::add(O::add(r[4], r[5]), O::add(r[6], r[7])));
#pragma unroll
    for (int i = N - (N % 8); i < N; i++) res = O::add(res, a[i]);
    return res;
  } else {
    constexpr int n2 = (N / 2) - ((N / 2) % 8);
    return O::add(pairwise_sum<n2, O>(a), pairwise_sum<N - n2, O>(a + n2));
  }
}

// runtime-length variant (MLP widths, unit ops)
template <class O>
__device__ double pairwise_sum_rt(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; i++) r = O::add(r, a[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = O::add(r[j], a[i + j]);
    double res = O::add(O::add(O::add(r[0], r[1]), O::add(r[2], r[3])),
                        O::add(O::add(r[4], r[5]), O::add(r[6], r[7])));
    for (; i < n; i++) res = O::add(res, a[i]);
    return res;
  }
  int64_t h = n / 2;
  h -= h % 8;
  return O::add(pairwise_sum_rt<O>(a, h), pairwise_sum_rt<O>(a + h, n - h));
}

// ------------------------------------------------------------ tableaus --
// Coefficients live in the constant bank and reach the FP64 instructions
// through uniform registers (LDCU; immediates would cost two UMOVs per
// 64-bit literal).  The generated flat layout a[7][7] | b[7] | b_err[7] |
// c[7] | w[7][4] is remapped at compile time so that the coefficients an
// instance reads together sit in aligned pairs (one LDCU.128 per two):
// a rows padded to 8, b_i and b_err_i interleaved, w rows on even offsets.
struct TabData {
  double v[112];
};
constexpr TabData remap_tab(const double (&f)[98]) {
  TabData t{};
  for (int i = 0; i < 7; i++) {
    for (int j = 0; j < 7; j++) t.v[8 * i + j] = f[i * 7 + j];  // a(i, j) -> 8 i + j
    t.v[56 + 2 * i] = f[49 + i];                               // b(i)
    t.v[57 + 2 * i] = f[56 + i];                               // b_err(i)
    t.v[70 + i] = f[63 + i];                                   // c(i)
    for (int j = 0; j < 4; j++) t.v[78 + 4 * i + j] = f[70 + i * 4 + j];  // w(i, j)
  }
  return t;
}
constexpr double k_dopri5_flat[98] = BODE_DOPRI5_FLAT_INIT;
constexpr double k_tsit5_flat[98] = BODE_TSIT5_FLAT_INIT;
constexpr double k_heun_flat[98] = BODE_HEUN_FLAT_INIT;
static __constant__ TabData c_tab[3] = {remap_tab(k_dopri5_flat), remap_tab(k_tsit5_flat),
                                        remap_tab(k_heun_flat)};

template <int M> struct TabShape;
// za/zb/ze/zw: the same coefficients as compile-time constants, used only to
// drop terms whose coefficient is exactly zero (they fold away when unrolled)
#define BODE_TAB_ZEROS(name)                                                        \
  static __device__ __forceinline__ constexpr double za(int i, int j) { return bode_##name##_a(i, j); } \
  static __device__ __forceinline__ constexpr double zb(int i) { return bode_##name##_b(i); }           \
  static __device__ __forceinline__ constexpr double ze(int i) { return bode_##name##_berr(i); }        \
  static __device__ __forceinline__ constexpr double zw(int i, int j) { return bode_##name##_interp(i, j); }
template <> struct TabShape<BODE_METHOD_DOPRI5> {
  static constexpr int S = BODE_DOPRI5_STAGES, ORDER = BODE_DOPRI5_ORDER,
                       ERR_ORDER = BODE_DOPRI5_ERROR_ORDER, NI = BODE_DOPRI5_NINTERP;
  static constexpr bool FSAL = BODE_DOPRI5_FSAL;
  BODE_TAB_ZEROS(dopri5)
};
template <> struct TabShape<BODE_METHOD_TSIT5> {
  static constexpr int S = BODE_TSIT5_STAGES, ORDER = BODE_TSIT5_ORDER,
                       ERR_ORDER = BODE_TSIT5_ERROR_ORDER, NI = BODE_TSIT5_NINTERP;
  static constexpr bool FSAL = BODE_TSIT5_FSAL;
  BODE_TAB_ZEROS(tsit5)
};
template <> struct TabShape<BODE_METHOD_HEUN> {
  static constexpr int S = BODE_HEUN_STAGES, ORDER = BODE_HEUN_ORDER,
                       ERR_ORDER = BODE_HEUN_ERROR_ORDER, NI = BODE_HEUN_NINTERP;
  static constexpr bool FSAL = BODE_HEUN_FSAL;
  BODE_TAB_ZEROS(heun)
};
#undef BODE_TAB_ZEROS

template <int M>
struct Tab : TabShape<M> {
  static __device__ __forceinline__ double a(int i, int j) { return c_tab[M].v[8 * i + j]; }
  static __device__ __forceinline__ double b(int i) { return c_tab[M].v[56 + 2 * i]; }
  static __device__ __forceinline__ double e(int i) { return c_tab[M].v[57 + 2 * i]; }
  static __device__ __forceinline__ double c(int i) { return c_tab[M].v[70 + i]; }
  static __device__ __forceinline__ double w(int i, int j) { return c_tab[M].v[78 + 4 * i + j]; }
};

// ------------------------------------------------------------ dynamics --
// Registered device functors replacing the reference's NumPy callables
// (stepper.py:19-20).  Each evaluates f(t, y) for ONE instance in the
// operation order of the NumPy expression it replaces.
struct DynParams {
  int32_t kind;
  uint32_t inst_mask;
  int32_t n_inst;
  const double* inst;
  double shared[8];
};

__device__ __forceinline__ void load_params(const DynParams& P, int64_t i, double* p, int np) {
  int r = 0;
  for (int k = 0; k < np; k++) {
    if ((P.inst_mask >> k) & 1u) {
      p[k] = P.inst[i * P.n_inst + r];
      r++;
    } else {
      p[k] = P.shared[k];
    }
  }
}

template <class O>
struct VdP {  // problems.py:45-48: (v, mu*(1-x*x)*v - x)
  static constexpr int D = 2;
  double mu;
  __device__ __forceinline__ void load(const DynParams& P, int64_t i) { load_params(P, i, &mu, 1); }
  __device__ __forceinline__ void operator()(double, const double* y, double* f) const {
    const double x = y[0], v = y[1];
    f[0] = v;
    if constexpr (O::kFast) {
      f[1] = fma(__dmul_rn(mu, fma(-x, x, 1.0)), v, -x);
    } else {
      f[1] = O::sub(O::mul(O::mul(mu, O::sub(1.0, O::mul(x, x))), v), x);
    }
  }
  // adjoint (bode_adjoint.cu): yb = J^T g, pb[slot] += (df/dp)^T g
  __device__ __forceinline__ void vjp(double, const double* y, const double* g, double* yb,
                                      double* pb) const {
    const double x = y[0], v = y[1], q = 1.0 - x * x;
    yb[0] = g[1] * (-2.0 * mu * x * v - 1.0);
    yb[1] = g[0] + g[1] * mu * q;
    pb[0] += g[1] * q * v;
  }
};

template <class O>
struct Lorenz {  // (s*(y-x), x*(r-z)-y, x*y - b*z)
  static constexpr int D = 3;
  double s, r, b;
  __device__ __forceinline__ void load(const DynParams& P, int64_t i) {
    double p[3];
    load_params(P, i, p, 3);
    s = p[0];
    r = p[1];
    b = p[2];
  }
  __device__ __forceinline__ void operator()(double, const double* y, double* f) const {
    const double x = y[0], yy = y[1], z = y[2];
    f[0] = O::mul(s, O::sub(yy, x));
    if constexpr (O::kFast) {
      f[1] = fma(x, __dsub_rn(r, z), -yy);
      f[2] = fma(x, yy, -__dmul_rn(b, z));
    } else {
      f[1] = O::sub(O::mul(x, O::sub(r, z)), yy);
      f[2] = O::sub(O::mul(x, yy), O::mul(b, z));
    }
  }
  __device__ __forceinline__ void vjp(double, const double* y, const double* g, double* yb,
                                      double* pb) const {
    const double x = y[0], yy = y[1], z = y[2];
    yb[0] = -s * g[0] + (r - z) * g[1] + yy * g[2];
    yb[1] = s * g[0] - g[1] + x * g[2];
    yb[2] = -x * g[1] - b * g[2];
    pb[0] += (yy - x) * g[0];
    pb[1] += x * g[1];
    pb[2] += -z * g[2];
  }
};

template <class O>
struct Harmonic {  // problems.py:169-170
  static constexpr int D = 2;
  __device__ __forceinline__ void load(const DynParams&, int64_t) {}
  __device__ __forceinline__ void operator()(double, const double* y, double* f) const {
    f[0] = y[1];
    f[1] = -y[0];
  }
  __device__ __forceinline__ void vjp(double, const double*, const double* g, double* yb,
                                      double*) const {
    yb[0] = -g[1];
    yb[1] = g[0];
  }
};

template <class O>
struct Damped {  // (y1, -y0 - 0.1*y1*|y1|)
  static constexpr int D = 2;
  __device__ __forceinline__ void load(const DynParams&, int64_t) {}
  __device__ __forceinline__ void operator()(double, const double* y, double* f) const {
    f[0] = y[1];
    if constexpr (O::kFast) {
      f[1] = fma(-__dmul_rn(0.1, y[1]), fabs(y[1]), -y[0]);
    } else {
      f[1] = O::sub(-y[0], O::mul(O::mul(0.1, y[1]), fabs(y[1])));
    }
  }
  __device__ __forceinline__ void vjp(double, const double* y, const double* g, double* yb,
                                      double*) const {
    yb[0] = -g[1];
    yb[1] = g[0] - 0.2 * fabs(y[1]) * g[1];  // d(y|y|)/dy = 2|y|
  }
};

// Component-wise family; the sub-kind is uniform across a launch.
template <class O, int DD>
struct Elementwise {
  static constexpr int D = DD;
  int32_t kind;
  double p[3];
  __device__ __forceinline__ void load(const DynParams& P, int64_t i) {
    kind = P.kind;
    load_params(P, i, p, 3);
  }
  __device__ __forceinline__ void operator()(double t, const double* y, double* f) const {
    switch (kind) {
      case BODE_DYN_ZERO:
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = 0.0;
        break;
      case BODE_DYN_CONST:
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = p[0];
        break;
      case BODE_DYN_LINEAR:
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = O::mul(p[0], y[j]);
        break;
      case BODE_DYN_LINEAR_COS: {
        const double g = O::mul(p[1], cos(O::mul(p[2], t)));
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = O::mad(p[0], y[j], g);
        break;
      }
      case BODE_DYN_LINEAR_SIN: {
        const double g = O::mul(p[1], sin(O::mul(p[2], t)));
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = O::mad(p[0], y[j], g);
        break;
      }
      case BODE_DYN_RELAX_COS: {
        const double g = cos(O::mul(p[1], t));
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = O::mul(p[0], O::sub(y[j], g));
        break;
      }
      case BODE_DYN_SQUARE:
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = (y[j] > p[0]) ? __longlong_as_double(0x7ff0000000000000LL)
                                                         : O::mul(y[j], y[j]);
        break;
      case BODE_DYN_LOGISTIC:
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = O::mul(y[j], O::sub(1.0, y[j]));
        break;
      case BODE_DYN_SIN_PLUS_T:
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = O::add(sin(y[j]), t);
        break;
      default:
#pragma unroll
        for (int j = 0; j < D; j++) f[j] = __longlong_as_double(0x7ff8000000000000LL);
    }
  }
  __device__ __forceinline__ void vjp(double t, const double* y, const double* g, double* yb,
                                      double* pb) const {
    double sg = 0.0;  // sum of g over components (shared-term gradients)
#pragma unroll
    for (int j = 0; j < D; j++) sg += g[j];
    switch (kind) {
      case BODE_DYN_ZERO:
#pragma unroll
        for (int j = 0; j < D; j++) yb[j] = 0.0;
        break;
      case BODE_DYN_CONST:
#pragma unroll
        for (int j = 0; j < D; j++) yb[j] = 0.0;
        pb[0] += sg;
        break;
      case BODE_DYN_LINEAR:
      case BODE_DYN_LINEAR_COS:
      case BODE_DYN_LINEAR_SIN:
#pragma unroll
        for (int j = 0; j < D; j++) {
          yb[j] = p[0] * g[j];
          pb[0] += y[j] * g[j];
        }
        if (kind == BODE_DYN_LINEAR_COS) {
          double sn, cs;
          sincos(p[2] * t, &sn, &cs);
          pb[1] += cs * sg;
          pb[2] -= p[1] * sn * t * sg;
        } else if (kind == BODE_DYN_LINEAR_SIN) {
          double sn, cs;
          sincos(p[2] * t, &sn, &cs);
          pb[1] += sn * sg;
          pb[2] += p[1] * cs * t * sg;
        }
        break;
      case BODE_DYN_RELAX_COS: {
        double sn, cs;
        sincos(p[1] * t, &sn, &cs);
#pragma unroll
        for (int j = 0; j < D; j++) {
          yb[j] = p[0] * g[j];
          pb[0] += (y[j] - cs) * g[j];
        }
        pb[1] += p[0] * sn * t * sg;
        break;
      }
      case BODE_DYN_SQUARE:
#pragma unroll
        for (int j = 0; j < D; j++) yb[j] = 2.0 * y[j] * g[j];
        break;
      case BODE_DYN_LOGISTIC:
#pragma unroll
        for (int j = 0; j < D; j++) yb[j] = (1.0 - 2.0 * y[j]) * g[j];
        break;
      case BODE_DYN_SIN_PLUS_T:
#pragma unroll
        for (int j = 0; j < D; j++) yb[j] = cos(y[j]) * g[j];
        break;
      default:
#pragma unroll
        for (int j = 0; j < D; j++) yb[j] = __longlong_as_double(0x7ff8000000000000LL);
    }
  }
};

// ---------------------------------------------------------- controller --
struct CtrlParams {
  double e1, e2, e3;  // (-beta_i)/k formed on the host (controller.py:221-226)
  double safety, fmin, fmax;
  int32_t hist;
  // host-derived: e1, e2 finite and not NumPy's special exponents, e3 == 0
  // (I / PI controllers): the fast-mode controller takes a branch-free path
  int32_t plain_pi;
};

// 1/x to ~1 ulp: hardware approximation + two Newton steps (fast mode only)
// 1/x to ~2^-46 relative (one Newton step): enough for the squared-norm
// controller, whose accept decisions only move when a norm lies within
// that distance of 1
__device__ __forceinline__ double fast_rcp1(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}

__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// error_norm, controller.py:120-142 (one instance)
template <int D, class O>
__device__ __forceinline__ double error_norm(const double* e, const double* y0, const double* y1,
                                             double atol, double rtol) {
  double sq[D];
#pragma unroll
  for (int j = 0; j < D; j++) {
    const double scale = O::mad(rtol, np_max(fabs(y0[j]), fabs(y1[j])), atol);
    // fast mode: e * (1/scale) within ~1 ulp of the quotient instead of the
    // IEEE division's ~19 instructions
    const double r = O::kFast ? e[j] * fast_rcp(scale) : ddiv(e[j], scale);
    sq[j] = O::mul(r, r);
  }
  const double s = pairwise_sum<D, O>(sq);
  double mean;
  if constexpr ((D & (D - 1)) == 0) {
    mean = __dmul_rn(s, 1.0 / D);  // exact: division by a power of two
  } else {
    mean = ddiv(s, (double)D);
  }
  const double norm = dsqrt(mean);
  return isfinite(norm) ? norm : __longlong_as_double(0x7ff0000000000000LL);
}

// fast mode: the squared norm mean(r*r) (what error_norm takes the square
// root of), +inf when non-finite -- the I/PI controller below never needs
// the root
template <int D, class O>
__device__ __forceinline__ double error_ms(const double* e, const double* y0, const double* y1,
                                           double atol, double rtol) {
  double sq[D], rr[D];
#pragma unroll
  for (int j = 0; j < D; j++) {
    // a plain compare-select instead of NumPy's NaN-propagating maximum: a
    // NaN |y0| or |y1| implies a NaN error estimate here, so the ratio is NaN
    // (-> +inf, rejection) whichever operand the select keeps
    const double a0 = fabs(y0[j]), a1 = fabs(y1[j]);
    const double scale = O::mad(rtol, a0 > a1 ? a0 : a1, atol);
    rr[j] = __dmul_rn(e[j], fast_rcp1(scale));
    sq[j] = O::mul(rr[j], rr[j]);
  }
  double s;
  if constexpr (D < 8) {  // NumPy's sequential order, the squares fused in
    s = sq[0];
#pragma unroll
    for (int j = 1; j < D; j++) s = fma(rr[j], rr[j], s);
  } else {
    s = pairwise_sum<D, O>(sq);
  }
  const double mean = s * (1.0 / D);  // (exact for power-of-two D, ~1 ulp otherwise)
  return mean < INFINITY ? mean : __longlong_as_double(0x7ff0000000000000LL);  // NaN -> inf
}

// adapt_step, controller.py:200-238 (one instance).  dt is dt_used on entry,
// dt_next on exit; returns accept.
__device__ __forceinline__ bool adapt(const CtrlParams& C, double norm, double& n1, double& n2,
                                      double& dt, const PowTables& T = g_pow_tables) {
  const bool accept = norm <= 1.0;
  const double a = np_max(norm, 1e-10);
  const double b = np_max(n1, 1e-10);
  const double g = np_max(n2, 1e-10);
  double factor = __dmul_rn(C.safety, np_scalar_pow(a, C.e1, T));
  if (C.e2 != 0.0) factor = __dmul_rn(factor, np_scalar_pow(b, C.e2, T));
  if (C.e3 != 0.0) factor = __dmul_rn(factor, np_scalar_pow(g, C.e3, T));
  if (!isfinite(factor)) factor = C.fmin;
  factor = np_min(np_max(factor, C.fmin), C.fmax);
  dt = __dmul_rn(dt, factor);
  if (C.hist || accept) {
    n2 = n1;
    n1 = a;
  }
  return accept;
}

__device__ __forceinline__ bool np_special_exponent(double e) {
  return e == 0.0 || e == 1.0 || e == -1.0 || e == 2.0 || e == 0.5;
}

// x**e given log(x) (when known): the same operations as np_scalar_pow
// (special exponents, then cr_pow = cr_log + cr_exp_mul), so results are
// bit-identical to the uncached path.
__device__ __forceinline__ double pow_logged(double x, double e, bool ok, double lh, double ll,
                                             const PowTables& T) {
  if (np_special_exponent(e)) return np_scalar_pow(x, e, T);
  return (ok && isfinite(e)) ? cr_exp_mul(e, lh, ll, x, T) : pow_fallback(x, e);
}

// adapt() for the persistent solver: the PID term n_prev^(-beta2/k) reuses
// log(n_prev), computed one step earlier as log of that step's norm, so a
// PI step costs one log + two exp instead of two full pows.  n1 >= 1e-10
// always holds (initialised to 1, then max(norm, NORM_FLOOR)), hence
// max(n1, NORM_FLOOR) == n1.  Bit-identical to adapt().
struct LogCache {
  double h, l;
  bool ok;  // false: log unknown (x = inf) -> libm path
};

// fast mode: x**e from a plain-double log (few ulp), special exponents as
// NumPy evaluates them
__device__ __forceinline__ double pow_logged_fast(double x, double e, bool ok, double Lh,
                                                  double Ll, const PowTables& T) {
  if (np_special_exponent(e)) return np_scalar_pow(x, e, T);
  return (ok && isfinite(e)) ? fast_exp_mul(e, Lh, Ll, x, T) : pow_fallback(x, e);
}

template <class O>
__device__ __forceinline__ bool adapt_cached(const CtrlParams& C, double norm, double& n1,
                                             double& n2, LogCache& L1, double& dt,
                                             const PowTables& T) {
  const bool accept = norm <= 1.0;
  const double a = np_max(norm, 1e-10);
  const double g = np_max(n2, 1e-10);
  LogCache La;
  La.ok = false;
  const bool need_log = !np_special_exponent(C.e1) || (C.e2 != 0.0 && !np_special_exponent(C.e2));
  double factor;
  if constexpr (O::kFast) {
    if (C.plain_pi) {
      // I / PI controller, fast mode: a = max(norm, 1e-10) is never NaN,
      // zero or subnormal and n1 >= 1e-10 always holds; only a = +inf (a
      // non-finite error estimate) leaves the log/exp path
      const double a2 = norm >= 1e-10 ? norm : 1e-10;
      if (a2 < INFINITY) {
        fast_log(a2, T, La.h, La.l);
        La.ok = true;
        factor = __dmul_rn(C.safety, fast_exp_mul(C.e1, La.h, La.l, a2, T));
      } else {
        factor = __dmul_rn(C.safety, pow_fallback(a2, C.e1));
      }
      if (C.e2 != 0.0)
        factor = __dmul_rn(factor, L1.ok ? fast_exp_mul(C.e2, L1.h, L1.l, n1, T) : pow_fallback(n1, C.e2));
      if (!(factor < INFINITY)) factor = C.fmin;  // factor >= 0: this is !isfinite
      factor = np_min(np_max(factor, C.fmin), C.fmax);
      dt = __dmul_rn(dt, factor);
      if (C.hist || accept) {
        n2 = n1;
        n1 = a2;
        L1 = La;
      }
      (void)g;
      return accept;
    }
    if (need_log) La.ok = fast_log(a, T, La.h, La.l);
    factor = __dmul_rn(C.safety, pow_logged_fast(a, C.e1, La.ok, La.h, La.l, T));
    if (C.e2 != 0.0) factor = __dmul_rn(factor, pow_logged_fast(n1, C.e2, L1.ok, L1.h, L1.l, T));
  } else {
    if (need_log) La.ok = cr_log(a, T, La.h, La.l);
    factor = __dmul_rn(C.safety, pow_logged(a, C.e1, La.ok, La.h, La.l, T));
    if (C.e2 != 0.0) factor = __dmul_rn(factor, pow_logged(n1, C.e2, L1.ok, L1.h, L1.l, T));
  }
  if (C.e3 != 0.0) factor = __dmul_rn(factor, np_scalar_pow(g, C.e3, T));
  if (!isfinite(factor)) factor = C.fmin;
  factor = np_min(np_max(factor, C.fmin), C.fmax);
  dt = __dmul_rn(dt, factor);
  if (C.hist || accept) {
    n2 = n1;
    n1 = a;
    L1 = La;
  }
  return accept;
}

// Fast-mode I / PI controller (C.plain_pi) on the squared norm ms:
//   accept  = norm <= 1          <=>  ms <= 1 + 2^-52 (sqrt correctly rounded)
//   factor  = safety * a^e1 * n1^e2 = safety * exp(e1 log a + e2 log n1)
// with log a = log(ms)/2 (a = max(norm, NORM_FLOOR), controller.py:26), the
// history term from the cached log of the previous norm, and ONE exp of the
// combined exponent (fast_log1 / fast_exp3: a few ulp, like the two ~1-ulp
// pows it replaces: the accept decisions are insensitive at that level --
// statuses and step counts stay equal to the oracle's at full scale,
// tests/test_gpu_parity.py, tools/parity_report.py --extra fast).  The
// non-finite cases resolve to what the reference computes: a = +inf or
// n1 = +inf make the product 0 or inf, i.e. factor_min; an exponent beyond
// the double range gives inf (factor_min) or a finite huge / tiny factor
// (clipped to factor_max / factor_min).
__device__ __forceinline__ bool adapt_pi_ms(const CtrlParams& C, double ms, LogCache& L1,
                                            double& dt, const PowTables& T) {
  const bool accept = ms <= 1.0000000000000002;
  LogCache La;
  La.ok = ms < INFINITY;
  La.l = 0.0;  // single-double logs on this path (fast_log1)
  double factor = C.fmin;
  if (La.ok) {
    const bool tiny = !(ms >= 1e-20);  // norm below the floor: a = 1e-10 exactly
    La.h = fast_log1(tiny ? 1e-10 : ms, T) * (tiny ? 1.0 : 0.5);
    if (C.e2 == 0.0 || L1.ok) {
      // (e2 == 0: fma(0, 0, y) == y -- no second uniform test of e2)
      const double y = fma(C.e2, L1.ok ? L1.h : 0.0, C.e1 * La.h);
      if (y < 700.0 && y > -700.0) {
        // finite and > 0: plain compare-selects (fmax/fmin would add NaN
        // handling that cannot trigger here)
        const double x = C.safety * fast_exp3(y, T);
        factor = x > C.fmin ? x : C.fmin;
        factor = factor < C.fmax ? factor : C.fmax;
      }
      else
        factor = (y > 0.0 && y < 709.78) ? C.fmax : C.fmin;
    }
  }
  dt = __dmul_rn(dt, factor);
  if (C.hist || accept) L1 = La;
  return accept;
}

// initial_step, controller.py:145-197 (one instance).  Returns dt (NaN when
// f0 is non-finite) and writes f0.
template <class F, class O>
__device__ __forceinline__ double initial_step(const F& f, double t0, const double* y0, int order,
                                               double atol, double rtol, double direction,
                                               double* f0) {
  constexpr int D = F::D;
  f(t0, y0, f0);
  bool bad = false;
  double scale[D], sq[D];
#pragma unroll
  for (int j = 0; j < D; j++) {
    bad |= !isfinite(f0[j]);
    scale[j] = O::mad(rtol, fabs(y0[j]), atol);
  }
#pragma unroll
  for (int j = 0; j < D; j++) {
    const double q = ddiv(y0[j], scale[j]);
    sq[j] = O::mul(q, q);
  }
  const double d0 = dsqrt(ddiv(pairwise_sum<D, O>(sq), (double)D));
#pragma unroll
  for (int j = 0; j < D; j++) {
    const double q = ddiv(f0[j], scale[j]);
    sq[j] = O::mul(q, q);
  }
  const double d1 = dsqrt(ddiv(pairwise_sum<D, O>(sq), (double)D));
  const bool degenerate = (d0 < 1e-5) || (d1 < 1e-5) || !isfinite(d1);
  const double h0 = degenerate ? 1e-6 : ddiv(__dmul_rn(0.01, d0), d1);
  const double hd = __dmul_rn(h0, direction);
  double y1[D], f1[D];
#pragma unroll
  for (int j = 0; j < D; j++) y1[j] = O::mad(hd, f0[j], y0[j]);
  f(__dadd_rn(t0, hd), y1, f1);
#pragma unroll
  for (int j = 0; j < D; j++) {
    const double q = ddiv(O::sub(f1[j], f0[j]), scale[j]);
    sq[j] = O::mul(q, q);
  }
  const double d2 = ddiv(dsqrt(ddiv(pairwise_sum<D, O>(sq), (double)D)), h0);
  const double dmax = np_max(d1, d2);
  const bool small = (dmax <= 1e-15) || !isfinite(dmax);
  const double h1 = small ? np_max(1e-6, __dmul_rn(h0, 1e-3))
                          : np_scalar_pow(ddiv(0.01, dmax), ddiv(1.0, (double)(order + 1)));
  const double dt = __dmul_rn(np_min(__dmul_rn(100.0, h0), h1), direction);
  return bad ? __longlong_as_double(0x7ff8000000000000LL) : dt;
}

// True when the last stage's input IS the solution: a[S-1][j] == b[j] for
// every j and b[S-1] == 0 (dopri5 and tsit5, the FSAL property).  The
// stage-(S-1) input and y_next are then the same sum of the same terms in
// the same order (zero terms skipped alike), i.e. bitwise equal, so y_next
// is taken from the stage instead of being summed a second time.
template <class T>
__device__ __forceinline__ constexpr bool last_stage_is_solution() {
  for (int j = 0; j < T::S - 1; j++)
    if (T::za(T::S - 1, j) != T::zb(j)) return false;
  return T::zb(T::S - 1) == 0.0;
}

// Stepper.step, stepper.py:54-110 (one instance).  k[0] must hold f0 for
// FSAL tableaus; on return k[0..S-1] are the stage derivatives.
template <class T, class F, class O>
__device__ __forceinline__ void rk_step(const F& f, double t, double h, const double* y,
                                        double (*k)[F::D], double* y_next, double* err) {
  // Terms with a zero coefficient (dopri5: a61, b1, b6, e1; tsit5: b6) add
  // exactly +-0 in the reference, so they are skipped -- except that 0*inf
  // and 0*NaN are NaN there: a non-finite skipped stage value is replayed by
  // making y_next / err NaN, which is what the reference's sums produce.
  // (The stage-6 input skips a61*k1; k1 non-finite already makes the a21
  // term, hence every later stage and err, non-finite.)  The only
  // representable difference left is the sign of an exactly-zero sum.
  constexpr int D = F::D, S = T::S;
  constexpr bool kLast = last_stage_is_solution<T>();
  if constexpr (!T::FSAL) f(t, y, k[0]);
#pragma unroll
  for (int i = 1; i < S; i++) {
    double ys[D];
#pragma unroll
    for (int c = 0; c < D; c++) {
      double s = O::mul(T::a(i, 0), k[0][c]);
#pragma unroll
      for (int j = 1; j < i; j++)
        if (T::za(i, j) != 0.0) s = O::mad(T::a(i, j), k[j][c], s);
      ys[c] = O::mad(h, s, y[c]);
      if (kLast && i == S - 1) y_next[c] = ys[c];
    }
    f(O::mad(T::c(i), h, t), ys, k[i]);
  }
#pragma unroll
  for (int c = 0; c < D; c++) {
    double s = O::mul(T::b(0), k[0][c]);
    double e = O::mul(T::e(0), k[0][c]);
    bool skipped_nonfinite = false;
#pragma unroll
    for (int i = 1; i < S; i++) {
      if (!kLast && T::zb(i) != 0.0) s = O::mad(T::b(i), k[i][c], s);
      if (T::ze(i) != 0.0) e = O::mad(T::e(i), k[i][c], e);
      // (exact mode only: in fast mode a non-finite stage already makes err
      // non-finite through the following stages, so the step is rejected and
      // y_next is never observed)
      if (!O::kFast && (T::zb(i) == 0.0 || T::ze(i) == 0.0))
        skipped_nonfinite |= !isfinite(k[i][c]);
    }
    if constexpr (!kLast) y_next[c] = O::mad(h, s, y[c]);
    err[c] = O::mul(h, e);
    if (skipped_nonfinite) {
      y_next[c] = __longlong_as_double(0x7ff8000000000000LL);
      err[c] = y_next[c];
    }
  }
}

// Stepper.interpolate, stepper.py:112-139: Horner weights, then y0 + dt*sum.
template <class T, int D, class O>
__device__ __forceinline__ void interpolate(const double (*k)[D], const double* y0, double h,
                                            double theta, double* out) {
  constexpr int S = T::S, M = T::NI;
  double w[S];
#pragma unroll
  for (int i = 0; i < S; i++) {
    double v = T::w(i, M - 1);
#pragma unroll
    for (int j = M - 2; j >= 0; j--) v = O::mad(v, theta, T::w(i, j));
    w[i] = O::mul(v, theta);
  }
#pragma unroll
  for (int c = 0; c < D; c++) {
    double s = O::mul(w[0], k[0][c]);
#pragma unroll
    for (int i = 1; i < S; i++) {
      bool zero_row = true;  // dopri5 row 1: w_1(theta) == 0 (k_1 finite on accepted steps)
#pragma unroll
      for (int j = 0; j < M; j++) zero_row &= T::zw(i, j) == 0.0;
      if (!zero_row) s = O::mad(w[i], k[i][c], s);
    }
    out[c] = O::mad(h, s, y0[c]);
  }
}

}  // namespace bode
