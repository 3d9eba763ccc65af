// bode_units.cuh -- declarations of the unit-op launchers (bode_units.cu).
#pragma once
#include "bode_solver.cuh"

namespace bode {
cudaError_t unit_rk_step(int method, const DynParams& dp, int64_t n, int64_t d, const double* t,
                         const double* dt, const double* y, const double* f0, double* yn,
                         double* err, double* k, cudaStream_t st);
cudaError_t unit_interpolate(int method, int64_t n, int64_t d, const double* k, const double* y0,
                             const double* dt, const double* theta, double* out, cudaStream_t st);
cudaError_t unit_error_norm(int64_t n, int64_t d, const double* err, const double* y0,
                            const double* y1, const double* atol_v, const double* rtol_v,
                            double atol, double rtol, double* norm, double* scratch,
                            cudaStream_t st);
cudaError_t unit_adapt_step(int64_t n, const double* norm, const CtrlParams& C, double* n1,
                            double* n2, double* dt, uint8_t* accept, double* dt_next,
                            cudaStream_t st);
cudaError_t unit_initial_step(const DynParams& dp, int64_t n, int64_t d, const double* t0,
                              const double* y0, int order, const double* av, const double* rv,
                              double a, double r, const double* dir, double* dt, double* f0,
                              cudaStream_t st);
cudaError_t unit_interpolate_tab(const bode_tableau* tab, int64_t n, int64_t d, const double* k,
                                 const double* y0, const double* dt, const double* theta,
                                 double* out, cudaStream_t st);
cudaError_t unit_eval_dynamics(const DynParams& dp, int64_t n, int64_t d, const double* t,
                               const double* y, double* out, cudaStream_t st);
}  // namespace bode
