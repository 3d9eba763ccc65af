// bode_mlp.cuh -- neural-ODE (MLP dynamics) solve path (kernels K3/K4).
#pragma once
#include "bode_solver.cuh"

namespace bode {
size_t mlp_workspace_bytes(const bode_solve_args* a);
cudaError_t mlp_solve(const bode_solve_args* a, const SolveParams& P, char* ws, cudaStream_t st,
                      int64_t* launches);

// tcgen05 3xTF32 stage evaluation (bode_mlp_tc.cu)
struct MlpTcArgs {
  int64_t n;            // rows of y / k
  int H;                // hidden width (multiple of 64)
  int stage;            // RK stage whose input is formed in the prologue
  const double* y;      // (n, 64) state
  const float* k;       // (S, n, 64) stage derivatives
  const double* h;      // (n) dt_used
  const int32_t* act;   // compacted running list (NULL: identity)
  const int32_t* count; // live rows
  const float* Yin;     // optional (count, 64) fp32 inputs instead of the prologue
  const float* wprep;   // weights pre-split by mlp_tc_prep
  const float* b1;
  const float* b2;
  float* out;           // (n, 64) rows scattered through act
};
bool mlp_tc_supported(int64_t D, int64_t H);
size_t mlp_tc_prep_bytes(int64_t H);
cudaError_t mlp_tc_prep(const float* W1, const float* W2, int64_t H, float* out, cudaStream_t st);
template <int M>
cudaError_t mlp_tc_launch(const MlpTcArgs& A, int max_tiles, cudaStream_t st);
}  // namespace bode
