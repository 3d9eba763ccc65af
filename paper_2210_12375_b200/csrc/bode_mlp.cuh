// bode_mlp.cuh -- neural-ODE (MLP dynamics) solve path (kernels K3/K4).
#pragma once
#include "bode_solver.cuh"

namespace bode {
size_t mlp_workspace_bytes(const bode_solve_args* a);
cudaError_t mlp_solve(const bode_solve_args* a, const SolveParams& P, char* ws, cudaStream_t st);
}  // namespace bode
