// Persistent-solver instantiations for the tsit5 tableau (see bode_dispatch.cuh).
#include "bode_dispatch.cuh"

namespace bode {
cudaError_t solve_tsit5(int mode, int kind, int64_t d, const SolveParams& P, int threads,
                     int blocks, cudaStream_t st) {
  return dispatch_solve<BODE_METHOD_TSIT5>(mode, kind, d, P, threads, blocks, st);
}
}  // namespace bode
