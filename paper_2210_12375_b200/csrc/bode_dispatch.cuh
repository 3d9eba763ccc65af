// bode_dispatch.cuh -- (method, dynamics, width, arithmetic mode) -> kernel.
// Instantiated once per method in bode_solve_<method>.cu so the three
// translation units compile in parallel.
#pragma once
#include "bode_solver.cuh"

namespace bode {

template <int M, class O>
cudaError_t dispatch_solve_ops(int kind, int64_t d, const SolveParams& P, int threads, int blocks,
                               cudaStream_t st) {
  switch (kind) {
    case BODE_DYN_VDP:
      if (d != 2) return cudaErrorInvalidValue;
      return launch_persistent<M, VdP<O>, O>(P, threads, blocks, st);
    case BODE_DYN_LORENZ:
      if (d != 3) return cudaErrorInvalidValue;
      return launch_persistent<M, Lorenz<O>, O>(P, threads, blocks, st);
    case BODE_DYN_HARMONIC:
      if (d != 2) return cudaErrorInvalidValue;
      return launch_persistent<M, Harmonic<O>, O>(P, threads, blocks, st);
    case BODE_DYN_DAMPED:
      if (d != 2) return cudaErrorInvalidValue;
      return launch_persistent<M, Damped<O>, O>(P, threads, blocks, st);
    default:
      switch (d) {
        case 1: return launch_persistent<M, Elementwise<O, 1>, O>(P, threads, blocks, st);
        case 2: return launch_persistent<M, Elementwise<O, 2>, O>(P, threads, blocks, st);
        case 3: return launch_persistent<M, Elementwise<O, 3>, O>(P, threads, blocks, st);
        case 4: return launch_persistent<M, Elementwise<O, 4>, O>(P, threads, blocks, st);
        default: return cudaErrorNotSupported;
      }
  }
}

template <int M>
cudaError_t dispatch_solve(int mode, int kind, int64_t d, const SolveParams& P, int threads,
                           int blocks, cudaStream_t st) {
  return mode == BODE_MODE_FAST ? dispatch_solve_ops<M, FastOps>(kind, d, P, threads, blocks, st)
                                : dispatch_solve_ops<M, ExactOps>(kind, d, P, threads, blocks, st);
}

cudaError_t solve_dopri5(int mode, int kind, int64_t d, const SolveParams& P, int threads,
                         int blocks, cudaStream_t st);
cudaError_t solve_tsit5(int mode, int kind, int64_t d, const SolveParams& P, int threads,
                        int blocks, cudaStream_t st);
cudaError_t solve_heun(int mode, int kind, int64_t d, const SolveParams& P, int threads,
                       int blocks, cudaStream_t st);

}  // namespace bode
