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
  float* Yout;          // optional (n, 64): the fp32 stage inputs formed (adjoint)
};
bool mlp_tc_supported(int64_t D, int64_t H);
size_t mlp_tc_prep_bytes(int64_t H);
cudaError_t mlp_tc_prep(const float* W1, const float* W2, int64_t H, float* out, cudaStream_t st);
template <int M>
cudaError_t mlp_tc_launch(const MlpTcArgs& A, int max_tiles, cudaStream_t st);

// fused persistent integrator (bode_mlp_fused.cu): after the init pass, one
// launch runs every running instance to termination
struct MlpFusedArgs {
  int H;
  int fast;                      // BODE_MODE_FAST: fused arithmetic, squared-norm I / PI control
  int64_t max_steps;
  const int32_t* act;            // running instances after the init pass
  const int32_t* count;          // their number (device)
  unsigned long long* queue;     // position counter, zeroed
  const double* y;               // (n, 64) initial state
  const float* f0;               // (n, 64) f(t0, y0) from the init pass
  const double* t;               // (n) t_start
  const double* dt;              // (n) first dt
  const float* wprep;            // weights pre-split by mlp_tc_prep
  const float* b1;
  const float* b2;
  CtrlParams ctrl;
  const double* t_end;
  const double* atol_v;
  const double* rtol_v;
  double atol, rtol;
  const double* t_eval;
  const int64_t* t_eval_offsets;
  int64_t t_eval_len;
  double* ys;
  int64_t* n_emitted;
  int64_t* n_steps;
  int64_t* n_accepted;
  double* final_dt;
  int64_t* status;
  unsigned long long* max_n;
  uint32_t* refresh;
  unsigned long long* prof;      // debug builds (-DBODE_FUSED_PROF): (grid*3, 32) cycles
  double* traj;                  // optional accepted-step trajectory (gradients),
  const int64_t* traj_offsets;   // SolveParams::traj layout
  float* traj_y;                 // optional (rows, S, 64): fp32 stage inputs of each record
};
bool mlp_fused_supported(int64_t D, int64_t H, int method);
template <int M>
cudaError_t mlp_fused_launch(const MlpFusedArgs& A, cudaStream_t st);
}  // namespace bode
