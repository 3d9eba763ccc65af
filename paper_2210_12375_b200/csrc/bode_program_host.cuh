// bode_program_host.cuh -- libbode-internal interface of the run-time
// programs (bode_program.cu) used by the solve / stepping entry points.
#pragma once
#include <string>

#include "bode_joint_dev.cuh"
#include "bode_stepper.cuh"

namespace bode {
int set_error(int code, const std::string& msg);  // bode_abi.cu
const bode_program_desc& program_desc(const bode_program* p);
// launches of the program's kernels; cudaErrorNotSupported when the program
// was not compiled with the kernel group the call needs
cudaError_t program_solve(const bode_program* p, int mode, const SolveParams& P, int threads,
                          int blocks, cudaStream_t st);
cudaError_t program_joint(const bode_program* p, int mode, const SolveParams& P, const JointWs& W,
                          cudaStream_t st);
cudaError_t program_init(const bode_program* p, int mode, const SolveParams& P, cudaStream_t st);
cudaError_t program_step(const bode_program* p, int mode, const SolveParams& P,
                         const StepState& S, cudaStream_t st);
cudaError_t program_rk_step(const bode_program* p, const bode_tableau* tab, const DynParams& dp,
                            int64_t n, const double* t, const double* dt, const double* y,
                            const double* f0, double* yn, double* err, double* k,
                            cudaStream_t st);
cudaError_t program_initial_step(const bode_program* p, const DynParams& dp, int64_t n,
                                 const double* t0, const double* y0, int order, const double* av,
                                 const double* rv, double a, double r, const double* dir,
                                 double* dt, double* f0, cudaStream_t st);
}  // namespace bode
