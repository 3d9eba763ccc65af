// bode_units.cu -- the reference's building blocks as standalone batched
// device ops (exact arithmetic), so the reference's unit tests
// (tests/test_stepper.py, tests/test_controller.py) can be re-expressed
// against the GPU.  One thread per instance; these are test/diagnostic
// entry points, not the hot path (that is bode_persistent_kernel).
#include "bode_units.cuh"
#include "bode_units_dev.cuh"

namespace bode {

__global__ void bode_finalize_kernel(const unsigned long long* max_n, const uint32_t* refresh,
                                     int stages, int fsal, int64_t* n_f_evals,
                                     int64_t* max_out, uint8_t* map_out, int64_t map_len) {
  if (map_out) {
    for (int64_t j = threadIdx.x; j < map_len; j += blockDim.x)
      map_out[j] = (uint8_t)((refresh[j >> 5] >> (j & 31)) & 1u);
    if (threadIdx.x == 0 && max_out) *max_out = (int64_t)*max_n;
  } else if (threadIdx.x == 0 && max_out) {
    *max_out = (int64_t)*max_n;
  }
  __shared__ unsigned long long s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const unsigned long long mx = *max_n;
  unsigned long long cnt = 0;
  if (fsal) {
    const unsigned long long words = (mx + 31) / 32;
    for (unsigned long long w = threadIdx.x; w < words; w += blockDim.x) {
      uint32_t v = refresh[w];
      // keep bits j with 1 <= j < max_n
      const unsigned long long lo = w * 32;
      for (int b = 0; b < 32; b++) {
        const unsigned long long j = lo + b;
        if (((v >> b) & 1u) && j >= 1 && j < mx) cnt++;
      }
    }
    atomicAdd(&s_cnt, cnt);
  }
  __syncthreads();
  if (threadIdx.x == 0)
    *n_f_evals = fsal ? (int64_t)(1 + (unsigned long long)(stages - 1) * mx + s_cnt)
                      : (int64_t)(1 + (unsigned long long)stages * mx);
}

__global__ void error_norm_kernel(int64_t n, int64_t d, const double* err, const double* y0,
                                  const double* y1, const double* atol_v, const double* rtol_v,
                                  double atol, double rtol, double* norm, double* scratch) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = atol_v ? atol_v[i] : atol, r = rtol_v ? rtol_v[i] : rtol;
  double* sq = scratch + i * d;
  for (int64_t j = 0; j < d; j++) {
    const double scale = ExactOps::mad(r, np_max(fabs(y0[i * d + j]), fabs(y1[i * d + j])), a);
    const double q = ddiv(err[i * d + j], scale);
    sq[j] = ExactOps::mul(q, q);
  }
  const double v = dsqrt(ddiv(pairwise_sum_rt<ExactOps>(sq, d), (double)d));
  norm[i] = isfinite(v) ? v : __longlong_as_double(0x7ff0000000000000LL);
}

__global__ void adapt_step_kernel(int64_t n, const double* norm, CtrlParams C, double* n1,
                                  double* n2, double* dt, uint8_t* accept, double* dt_next) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = n1[i], b = n2[i], h = dt[i];
  accept[i] = adapt(C, norm[i], a, b, h);
  n1[i] = a;
  n2[i] = b;
  dt[i] = h;
  dt_next[i] = h;
}

static inline unsigned grid_for(int64_t n) { return (unsigned)((n + 127) / 128); }

// Stepper.interpolate (stepper.py:112-139) for any tableau: Horner weights
// with separate roundings, every stage term included, y0 + dt * sum
__global__ void interpolate_tab_kernel(const bode_tableau* __restrict__ T, int64_t n, int64_t d,
                                       const double* k, const double* y0, const double* dt,
                                       const double* theta, double* out) {
  using O = ExactOps;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int S = T->stages, M = T->n_interp;
  const double th = theta[i], h = dt[i];
  double w[BODE_TABLEAU_MAX_STAGES];
  for (int s = 0; s < S; s++) {
    double v = T->interp[s * BODE_TABLEAU_MAX_INTERP + M - 1];
    for (int j = M - 2; j >= 0; j--) v = O::add(O::mul(v, th), T->interp[s * BODE_TABLEAU_MAX_INTERP + j]);
    w[s] = O::mul(v, th);
  }
  for (int64_t c = 0; c < d; c++) {
    double acc = O::mul(w[0], k[i * d + c]);
    for (int s = 1; s < S; s++) acc = O::add(acc, O::mul(w[s], k[(s * n + i) * d + c]));
    out[i * d + c] = O::add(y0[i * d + c], O::mul(h, acc));
  }
}

cudaError_t unit_interpolate_tab(const bode_tableau* tab, int64_t n, int64_t d, const double* k,
                                 const double* y0, const double* dt, const double* theta,
                                 double* out, cudaStream_t st) {
  interpolate_tab_kernel<<<grid_for(n), 128, 0, st>>>(tab, n, d, k, y0, dt, theta, out);
  return cudaGetLastError();
}

template <int M, class F>
static cudaError_t launch_rk(const DynParams& dp, int64_t n, const double* t, const double* dt,
                             const double* y, const double* f0, double* yn, double* err,
                             double* k, cudaStream_t st) {
  rk_step_kernel<M, F><<<grid_for(n), 128, 0, st>>>(dp, n, t, dt, y, f0, yn, err, k);
  return cudaGetLastError();
}

template <int M>
static cudaError_t rk_for_method(const DynParams& dp, int64_t d, int64_t n, const double* t,
                                 const double* dt, const double* y, const double* f0, double* yn,
                                 double* err, double* k, cudaStream_t st) {
  using O = ExactOps;
  switch (dp.kind) {
    case BODE_DYN_VDP:
      return d == 2 ? launch_rk<M, VdP<O>>(dp, n, t, dt, y, f0, yn, err, k, st) : cudaErrorInvalidValue;
    case BODE_DYN_LORENZ:
      return d == 3 ? launch_rk<M, Lorenz<O>>(dp, n, t, dt, y, f0, yn, err, k, st) : cudaErrorInvalidValue;
    case BODE_DYN_HARMONIC:
      return d == 2 ? launch_rk<M, Harmonic<O>>(dp, n, t, dt, y, f0, yn, err, k, st) : cudaErrorInvalidValue;
    case BODE_DYN_DAMPED:
      return d == 2 ? launch_rk<M, Damped<O>>(dp, n, t, dt, y, f0, yn, err, k, st) : cudaErrorInvalidValue;
    default:
      switch (d) {
        case 1: return launch_rk<M, Elementwise<O, 1>>(dp, n, t, dt, y, f0, yn, err, k, st);
        case 2: return launch_rk<M, Elementwise<O, 2>>(dp, n, t, dt, y, f0, yn, err, k, st);
        case 3: return launch_rk<M, Elementwise<O, 3>>(dp, n, t, dt, y, f0, yn, err, k, st);
        case 4: return launch_rk<M, Elementwise<O, 4>>(dp, n, t, dt, y, f0, yn, err, k, st);
        default: return cudaErrorNotSupported;
      }
  }
}

cudaError_t unit_rk_step(int method, const DynParams& dp, int64_t n, int64_t d, const double* t,
                         const double* dt, const double* y, const double* f0, double* yn,
                         double* err, double* k, cudaStream_t st) {
  switch (method) {
    case BODE_METHOD_DOPRI5: return rk_for_method<BODE_METHOD_DOPRI5>(dp, d, n, t, dt, y, f0, yn, err, k, st);
    case BODE_METHOD_TSIT5: return rk_for_method<BODE_METHOD_TSIT5>(dp, d, n, t, dt, y, f0, yn, err, k, st);
    case BODE_METHOD_HEUN: return rk_for_method<BODE_METHOD_HEUN>(dp, d, n, t, dt, y, f0, yn, err, k, st);
  }
  return cudaErrorInvalidValue;
}

template <int M>
static cudaError_t interp_for_method(int64_t n, int64_t d, const double* k, const double* y0,
                                     const double* dt, const double* theta, double* out,
                                     cudaStream_t st) {
  switch (d) {
    case 1: interpolate_kernel<M, 1><<<grid_for(n), 128, 0, st>>>(n, k, y0, dt, theta, out); break;
    case 2: interpolate_kernel<M, 2><<<grid_for(n), 128, 0, st>>>(n, k, y0, dt, theta, out); break;
    case 3: interpolate_kernel<M, 3><<<grid_for(n), 128, 0, st>>>(n, k, y0, dt, theta, out); break;
    case 4: interpolate_kernel<M, 4><<<grid_for(n), 128, 0, st>>>(n, k, y0, dt, theta, out); break;
    default: return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

cudaError_t unit_interpolate(int method, int64_t n, int64_t d, const double* k, const double* y0,
                             const double* dt, const double* theta, double* out, cudaStream_t st) {
  switch (method) {
    case BODE_METHOD_DOPRI5: return interp_for_method<BODE_METHOD_DOPRI5>(n, d, k, y0, dt, theta, out, st);
    case BODE_METHOD_TSIT5: return interp_for_method<BODE_METHOD_TSIT5>(n, d, k, y0, dt, theta, out, st);
    case BODE_METHOD_HEUN: return interp_for_method<BODE_METHOD_HEUN>(n, d, k, y0, dt, theta, out, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t unit_error_norm(int64_t n, int64_t d, const double* err, const double* y0,
                            const double* y1, const double* atol_v, const double* rtol_v,
                            double atol, double rtol, double* norm, double* scratch,
                            cudaStream_t st) {
  error_norm_kernel<<<grid_for(n), 128, 0, st>>>(n, d, err, y0, y1, atol_v, rtol_v, atol, rtol,
                                                  norm, scratch);
  return cudaGetLastError();
}

cudaError_t unit_adapt_step(int64_t n, const double* norm, const CtrlParams& C, double* n1,
                            double* n2, double* dt, uint8_t* accept, double* dt_next,
                            cudaStream_t st) {
  adapt_step_kernel<<<grid_for(n), 128, 0, st>>>(n, norm, C, n1, n2, dt, accept, dt_next);
  return cudaGetLastError();
}

template <class F>
static cudaError_t launch_init(const DynParams& dp, int64_t n, const double* t0, const double* y0,
                               int order, const double* av, const double* rv, double a, double r,
                               const double* dir, double* dt, double* f0, cudaStream_t st) {
  initial_step_kernel<F><<<grid_for(n), 128, 0, st>>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0);
  return cudaGetLastError();
}

cudaError_t unit_initial_step(const DynParams& dp, int64_t n, int64_t d, const double* t0,
                              const double* y0, int order, const double* av, const double* rv,
                              double a, double r, const double* dir, double* dt, double* f0,
                              cudaStream_t st) {
  using O = ExactOps;
  switch (dp.kind) {
    case BODE_DYN_VDP:
      return d == 2 ? launch_init<VdP<O>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0, st) : cudaErrorInvalidValue;
    case BODE_DYN_LORENZ:
      return d == 3 ? launch_init<Lorenz<O>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0, st) : cudaErrorInvalidValue;
    case BODE_DYN_HARMONIC:
      return d == 2 ? launch_init<Harmonic<O>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0, st) : cudaErrorInvalidValue;
    case BODE_DYN_DAMPED:
      return d == 2 ? launch_init<Damped<O>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0, st) : cudaErrorInvalidValue;
    default:
      switch (d) {
        case 1: return launch_init<Elementwise<O, 1>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0, st);
        case 2: return launch_init<Elementwise<O, 2>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0, st);
        case 3: return launch_init<Elementwise<O, 3>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0, st);
        case 4: return launch_init<Elementwise<O, 4>>(dp, n, t0, y0, order, av, rv, a, r, dir, dt, f0, st);
        default: return cudaErrorNotSupported;
      }
  }
}

template <class F>
static cudaError_t launch_eval(const DynParams& dp, int64_t n, const double* t, const double* y,
                               double* out, cudaStream_t st) {
  eval_dynamics_kernel<F><<<grid_for(n), 128, 0, st>>>(dp, n, t, y, out);
  return cudaGetLastError();
}

cudaError_t unit_eval_dynamics(const DynParams& dp, int64_t n, int64_t d, const double* t,
                               const double* y, double* out, cudaStream_t st) {
  using O = ExactOps;
  switch (dp.kind) {
    case BODE_DYN_VDP:
      return d == 2 ? launch_eval<VdP<O>>(dp, n, t, y, out, st) : cudaErrorInvalidValue;
    case BODE_DYN_LORENZ:
      return d == 3 ? launch_eval<Lorenz<O>>(dp, n, t, y, out, st) : cudaErrorInvalidValue;
    case BODE_DYN_HARMONIC:
      return d == 2 ? launch_eval<Harmonic<O>>(dp, n, t, y, out, st) : cudaErrorInvalidValue;
    case BODE_DYN_DAMPED:
      return d == 2 ? launch_eval<Damped<O>>(dp, n, t, y, out, st) : cudaErrorInvalidValue;
    default:
      switch (d) {
        case 1: return launch_eval<Elementwise<O, 1>>(dp, n, t, y, out, st);
        case 2: return launch_eval<Elementwise<O, 2>>(dp, n, t, y, out, st);
        case 3: return launch_eval<Elementwise<O, 3>>(dp, n, t, y, out, st);
        case 4: return launch_eval<Elementwise<O, 4>>(dp, n, t, y, out, st);
        default: return cudaErrorNotSupported;
      }
  }
}

}  // namespace bode
