// bode_stepper.cuh -- BatchSolver.step_once (solver.py:208-282) on the
// device: ONE loop iteration of every running instance per launch, the
// reference's lockstep stepping API (tests and custom loops drive it one
// iteration at a time; solve() runs the persistent kernel instead).
//
// The per-instance state lives in device arrays between launches: the
// solve outputs double as state (final_dt = ControllerState.dt, n_emitted
// = the t_eval cursor, n_steps / n_accepted / status), plus t, y, f0, the
// PID history (norm_prev, norm_prev2) and the FSAL-valid flag.  Each
// launch rebuilds a Lane from that state, runs the same Lane::step as the
// persistent kernel (so a step_once loop and solve() take identical
// decisions), and writes the state back.
#pragma once
#include "bode_solver.cuh"

namespace bode {

struct StepState {
  double* t;            // (n) current time
  double* y;            // (n, D) current state
  double* n1;           // (n) norm_prev
  double* n2;           // (n) norm_prev2
  uint8_t* fsal_valid;  // (n) the cached f0 is f(t, y) (solver.py:217-226)
  int32_t* flags;       // [0] some instance still running after the iteration,
                        // [1] some running instance needed an FSAL refresh evaluation
};

template <int M, class F, class O>
__global__ void __launch_bounds__(128) bode_step_kernel(const SolveParams P, const StepState S) {
  constexpr int D = F::D;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P.n || P.status[i] != BODE_RUNNING) return;
  Lane<M, F, O> L;
  L.load_problem(P, i);
  L.t = S.t[i];
#pragma unroll
  for (int c = 0; c < D; c++) {
    L.y[c] = S.y[i * D + c];
    L.k[0][c] = P.f0[i * D + c];
  }
  L.dt = P.final_dt[i];
  L.n1 = S.n1[i];
  L.n2 = S.n2[i];
  L.nsteps = (int32_t)P.n_steps[i];
  L.nacc = (int32_t)P.n_accepted[i];
  L.cursor = (int32_t)P.n_emitted[i];
  L.status = BODE_RUNNING;
  const double* te = L.te_of(P);
  L.te_next = L.cursor < L.m ? te[L.cursor] : 0.0;
  // the controller's cached history log, exactly as the persistent loop
  // holds it (log of norm_prev, adapt_cached)
  if constexpr (O::kFast) {
    L.L1.ok = fast_log(L.n1, g_pow_tables, L.L1.h, L.L1.l);
  } else {
    L.L1.ok = cr_log(L.n1, g_pow_tables, L.L1.h, L.L1.l);
  }
  bool refreshed = false;
  if constexpr (Tab<M>::FSAL) {
    if (!S.fsal_valid[i]) {  // solver.py:220-226
      L.f(L.t, L.y, L.k[0]);
      S.fsal_valid[i] = 1;
      refreshed = true;
    }
  }
  const EmitBase eb{L.te_of(P), L.ys_of(P)};
  if (L.template step<false>(P, g_pow_tables, P.trace_cap > 0, nullptr, eb)) S.fsal_valid[i] = 0;
  S.t[i] = L.t;
#pragma unroll
  for (int c = 0; c < D; c++) {
    S.y[i * D + c] = L.y[c];
    P.f0[i * D + c] = L.k[0][c];
  }
  S.n1[i] = L.n1;
  S.n2[i] = L.n2;
  L.finish(P);
  if (L.status == BODE_RUNNING) atomicOr(&S.flags[0], 1);
  if (refreshed) atomicOr(&S.flags[1], 1);
}

}  // namespace bode
