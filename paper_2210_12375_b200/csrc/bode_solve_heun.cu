// Persistent-solver instantiations for the heun tableau (see bode_dispatch.cuh).
#include "bode_dispatch.cuh"

namespace bode {
cudaError_t solve_heun(int mode, int kind, int64_t d, const SolveParams& P, int threads,
                     int blocks, cudaStream_t st) {
  return dispatch_solve<BODE_METHOD_HEUN>(mode, kind, d, P, threads, blocks, st);
}
}  // namespace bode
