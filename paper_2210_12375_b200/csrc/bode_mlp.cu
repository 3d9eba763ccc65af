// bode_mlp.cu -- placeholder until the tcgen05 stage kernels land.
#include "bode_mlp.cuh"

namespace bode {
size_t mlp_workspace_bytes(const bode_solve_args*) { return 0; }
cudaError_t mlp_solve(const bode_solve_args*, const SolveParams&, char*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace bode
