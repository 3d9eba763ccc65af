// bode_adjoint.cuh -- reverse-mode gradients of a batched solve (bode_adjoint.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "bode_device.cuh"

namespace bode {

struct AdjParams {
  int64_t n;
  DynParams dyn;
  const double* t_eval;
  const int64_t* t_eval_offsets;  // CSR rows, or NULL: one shared array of t_eval_len
  int64_t t_eval_len;
  const double* traj;             // (rows, kTrajExtra + D), see SolveParams::traj
  const int64_t* traj_offsets;    // (n+1,)
  const int64_t* n_emitted;
  const double* grad_ys;          // ys layout
  double* grad_y0;                // (n, D)
  double* grad_params;            // (n, 8) or NULL
  const int64_t* order;           // queue order (longest first) or NULL
  unsigned long long* queue;
  // MLP dynamics (bode_mlp_adjoint.cu): weights, batch-summed weight
  // gradients (fp32, NULL = not wanted) and per-CTA partials (workspace)
  int64_t H;
  const float *W1, *b1, *W2, *b2;
  float *gW1, *gb1, *gW2, *gb2;
  const float* traj_stages;  // (rows, S, 64) recorded stage inputs (MLP, d = 64)
};

// workspace: [queue | LPT cost | LPT scratch | MLP partials (MLP only)]
size_t adjoint_workspace_bytes(int64_t n, int64_t d, int kind, int64_t H);
// tensor-core backward for D = 64 (bode_mlp_adjoint_tc.cu); the workspace
// of adjoint_workspace_bytes is sized for 7 stages (the widest tableau)
bool mlp_adjoint_tc_supported(int64_t d, int64_t H);
size_t mlp_adjoint_tc_bytes(int64_t n, int64_t H, int method);
cudaError_t mlp_adjoint_tc_run(int method, AdjParams A, void* ws, cudaStream_t st, int64_t* launches);
// Builds the longest-first queue from the trajectory lengths, then launches
// the persistent backward kernel; returns the number of kernels launched
// through *launches.
cudaError_t adjoint_launch(int method, int64_t d, AdjParams A, void* ws, cudaStream_t st,
                           int64_t* launches);

}  // namespace bode
