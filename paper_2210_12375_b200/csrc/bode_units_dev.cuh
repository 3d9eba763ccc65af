// bode_units_dev.cuh -- device kernels of the unit ops (Stepper.step /
// interpolate / initial_step as batched one-thread-per-instance kernels).
// Templates only: instantiated by bode_units.cu for the registered
// functors and by run-time-compiled programs (bode_program.cu) for
// user-supplied dynamics / tableaus.
#pragma once
#include "bode_solver.cuh"

namespace bode {

template <int M, class F>
__global__ void rk_step_kernel(DynParams dp, int64_t n, const double* t, const double* dt,
                               const double* y, const double* f0, double* y_next, double* err,
                               double* k) {
  constexpr int D = F::D, S = Tab<M>::S;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  F f;
  f.load(dp, i);
  double kk[S][D], yy[D], yn[D], e[D];
#pragma unroll
  for (int c = 0; c < D; c++) {
    yy[c] = y[i * D + c];
    kk[0][c] = Tab<M>::FSAL ? f0[i * D + c] : 0.0;
  }
  rk_step<Tab<M>, F, ExactOps>(f, t[i], dt[i], yy, kk, yn, e);
#pragma unroll
  for (int c = 0; c < D; c++) {
    y_next[i * D + c] = yn[c];
    err[i * D + c] = e[c];
  }
#pragma unroll
  for (int s = 0; s < S; s++)
#pragma unroll
    for (int c = 0; c < D; c++) k[(s * n + i) * D + c] = kk[s][c];
}

template <int M, int D>
__global__ void interpolate_kernel(int64_t n, const double* k, const double* y0, const double* dt,
                                   const double* theta, double* out) {
  constexpr int S = Tab<M>::S;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double kk[S][D], yy[D], o[D];
#pragma unroll
  for (int c = 0; c < D; c++) yy[c] = y0[i * D + c];
#pragma unroll
  for (int s = 0; s < S; s++)
#pragma unroll
    for (int c = 0; c < D; c++) kk[s][c] = k[(s * n + i) * D + c];
  interpolate<Tab<M>, D, ExactOps>(kk, yy, dt[i], theta[i], o);
#pragma unroll
  for (int c = 0; c < D; c++) out[i * D + c] = o[c];
}

template <class F>
__global__ void initial_step_kernel(DynParams dp, int64_t n, const double* t0, const double* y0,
                                    int order, const double* atol_v, const double* rtol_v,
                                    double atol, double rtol, const double* direction, double* dt,
                                    double* f0) {
  constexpr int D = F::D;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  F f;
  f.load(dp, i);
  double yy[D], ff[D];
#pragma unroll
  for (int c = 0; c < D; c++) yy[c] = y0[i * D + c];
  dt[i] = initial_step<F, ExactOps>(f, t0[i], yy, order, atol_v ? atol_v[i] : atol,
                                    rtol_v ? rtol_v[i] : rtol, direction[i], ff);
#pragma unroll
  for (int c = 0; c < D; c++) f0[i * D + c] = ff[c];
}

// f(t, y) on the batch: a registered functor evaluated for callers that
// call the dynamics object itself (problems.py:41-50 returns a callable)
template <class F>
__global__ void eval_dynamics_kernel(DynParams dp, int64_t n, const double* t, const double* y,
                                     double* out) {
  constexpr int D = F::D;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  F f;
  f.load(dp, i);
  double yy[D], ff[D];
#pragma unroll
  for (int c = 0; c < D; c++) yy[c] = y[i * D + c];
  f(t[i], yy, ff);
#pragma unroll
  for (int c = 0; c < D; c++) out[i * D + c] = ff[c];
}

// ---- runtime-coefficient tableau (any ButcherTableau, tableau.py:17-83) --
// The unit ops of the stepping API take the tableau by value from device
// memory, so Stepper.step / interpolate with a user tableau need no
// recompilation per coefficient set.  Every term is included, zeros too,
// in the reference's order (stepper.py:75-101, :128-139).
constexpr int kRtMaxStages = BODE_TABLEAU_MAX_STAGES, kRtMaxInterp = BODE_TABLEAU_MAX_INTERP;

template <class F>
__global__ void rk_step_rt_kernel(DynParams dp, const bode_tableau* __restrict__ T, int64_t n,
                                  const double* t, const double* dt, const double* y,
                                  const double* f0, double* y_next, double* err, double* k) {
  constexpr int D = F::D;
  using O = ExactOps;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int S = T->stages;
  F f;
  f.load(dp, i);
  double kk[kRtMaxStages][D], yy[D], ys[D];
  const double ti = t[i], h = dt[i];
#pragma unroll
  for (int c = 0; c < D; c++) yy[c] = y[i * D + c];
  if (T->fsal) {
#pragma unroll
    for (int c = 0; c < D; c++) kk[0][c] = f0[i * D + c];
  } else {
    f(ti, yy, kk[0]);
  }
  for (int s = 1; s < S; s++) {
#pragma unroll
    for (int c = 0; c < D; c++) {
      double acc = O::mul(T->a[s * kRtMaxStages], kk[0][c]);
      for (int j = 1; j < s; j++) acc = O::add(acc, O::mul(T->a[s * kRtMaxStages + j], kk[j][c]));
      ys[c] = O::add(O::mul(h, acc), yy[c]);
    }
    f(O::add(ti, O::mul(T->c[s], h)), ys, kk[s]);
  }
#pragma unroll
  for (int c = 0; c < D; c++) {
    double acc = O::mul(T->b[0], kk[0][c]);
    double e = O::mul(T->b_err[0], kk[0][c]);
    for (int s = 1; s < S; s++) {
      acc = O::add(acc, O::mul(T->b[s], kk[s][c]));
      e = O::add(e, O::mul(T->b_err[s], kk[s][c]));
    }
    y_next[i * D + c] = O::add(yy[c], O::mul(h, acc));
    err[i * D + c] = O::mul(h, e);
  }
  for (int s = 0; s < S; s++)
#pragma unroll
    for (int c = 0; c < D; c++) k[(s * n + i) * D + c] = kk[s][c];
}

}  // namespace bode
