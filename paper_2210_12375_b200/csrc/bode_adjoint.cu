// bode_adjoint.cu -- reverse-mode gradients through a batched solve
// (torchode's AutoDiffAdjoint backward; the
// reference itself has no gradients).
//
// Discretise-then-optimise.  The forward persistent solve records every
// accepted step (t_old, h, t_eval cursor, y_old) into a CSR trajectory
// (bode_solver.cuh, Lane::step).  This kernel walks each instance's steps
// backwards, one lane per instance, with the same persistent queue as the
// forward solve (longest trajectory first):
//
//   forward recompute of the step from y_old (stages k_s and stage inputs
//   Y_s, in registers), then the adjoint sweep
//     kbar_s  = h b_s abar + sum_p h w_s(theta_p) gbar_p   (solution update
//                                                           + dense output)
//     ybar    = abar + sum_p gbar_p
//     s = S-1..0: (Ybar, pbar) += f_vjp(t + c_s h, Y_s, kbar_s);
//                 ybar += Ybar;  kbar_j += h a_sj Ybar (j < s)
//     abar    = ybar
//
// k_0 is differentiated as f(t_old, y_old): the FSAL cache holds exactly
// that value (the refresh evaluation is a value no-op, solver.py:220-226,
// SURVEY finding 3), and stage 6 of dopri5/tsit5 evaluates f at y_next.
// Step sizes, accept decisions and dense-output positions theta are
// constants of the backward pass (no gradient through the controller).
#include "bode_adjoint.cuh"
#include "bode_sched.cuh"
#include "bode_solver.cuh"

namespace bode {

namespace {

template <int M, class F>
__device__ __forceinline__ void adjoint_instance(const AdjParams& A, int64_t i) {
  using T = Tab<M>;
  constexpr int D = F::D, S = T::S, NI = T::NI, W = kTrajStride<D>;
  F f;
  f.load(A.dyn, i);
  const double* te = A.t_eval_offsets ? A.t_eval + A.t_eval_offsets[i] : A.t_eval;
  const double* gy = A.t_eval_offsets ? A.grad_ys + A.t_eval_offsets[i] * D
                                      : A.grad_ys + i * A.t_eval_len * D;
  const int64_t r0 = A.traj_offsets[i];
  const int64_t nrec = A.traj_offsets[i + 1] - r0;
  int64_t hi = A.n_emitted[i];  // points [c_lo, hi) belong to the step being reversed
  double ab[D], pb[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int c = 0; c < D; c++) ab[c] = 0.0;

  for (int64_t r = nrec - 1; r >= 0; r--) {
    double rec[W];
#pragma unroll
    for (int q = 0; q < W; q += 4)  // whole sectors, one 256-bit load each
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(rec[q]), "=d"(rec[q + 1]), "=d"(rec[q + 2]), "=d"(rec[q + 3])
                   : "l"(A.traj + (r0 + r) * W + q));
    const double t = rec[0], h = rec[1];
    const int64_t lo = (int64_t)rec[2];
    double y[D];
#pragma unroll
    for (int c = 0; c < D; c++) y[c] = rec[kTrajExtra + c];

    // forward recompute: stage derivatives k and stage inputs Y
    double k[S][D], Y[S][D];
    f(t, y, k[0]);
#pragma unroll
    for (int c = 0; c < D; c++) Y[0][c] = y[c];
#pragma unroll
    for (int s = 1; s < S; s++) {
#pragma unroll
      for (int c = 0; c < D; c++) {
        double acc = T::a(s, 0) * k[0][c];
#pragma unroll
        for (int j = 1; j < s; j++)
          if (T::za(s, j) != 0.0) acc = fma(T::a(s, j), k[j][c], acc);
        Y[s][c] = fma(h, acc, y[c]);
      }
      f(fma(T::c(s), h, t), Y[s], k[s]);
    }

    // seeds: y_next = y + h sum b_s k_s, and the points emitted in this step
    double kb[S][D], yb[D];
#pragma unroll
    for (int c = 0; c < D; c++) yb[c] = ab[c];
#pragma unroll
    for (int s = 0; s < S; s++) {
      const double hb = h * T::b(s);
#pragma unroll
      for (int c = 0; c < D; c++) kb[s][c] = hb * ab[c];
    }
    for (int64_t p = lo; p < hi; p++) {
      double theta = ddiv(te[p] - t, h);  // as the forward's Lane::emit
      theta = np_max(theta, 0.0);
      const double* g = gy + p * D;
      double gv[D];
#pragma unroll
      for (int c = 0; c < D; c++) {
        gv[c] = g[c];
        yb[c] += gv[c];
      }
#pragma unroll
      for (int s = 0; s < S; s++) {
        double v = T::w(s, NI - 1);
#pragma unroll
        for (int j = NI - 2; j >= 0; j--) v = fma(v, theta, T::w(s, j));
        const double hw = h * (v * theta);
#pragma unroll
        for (int c = 0; c < D; c++) kb[s][c] = fma(hw, gv[c], kb[s][c]);
      }
    }
    hi = lo;

    // reverse sweep through the stages
#pragma unroll
    for (int s = S - 1; s >= 1; s--) {
      double Yb[D];
      f.vjp(fma(T::c(s), h, t), Y[s], kb[s], Yb, pb);
#pragma unroll
      for (int c = 0; c < D; c++) {
        yb[c] += Yb[c];
#pragma unroll
        for (int j = 0; j < s; j++)
          if (T::za(s, j) != 0.0) kb[j][c] = fma(h * T::a(s, j), Yb[c], kb[j][c]);
      }
    }
    {
      double Yb[D];
      f.vjp(t, y, kb[0], Yb, pb);
#pragma unroll
      for (int c = 0; c < D; c++) ab[c] = yb[c] + Yb[c];
    }
  }
  // points at t_start are copies of y0 (solver.py:200-206)
  for (int64_t p = 0; p < hi; p++) {
#pragma unroll
    for (int c = 0; c < D; c++) ab[c] += gy[p * D + c];
  }
#pragma unroll
  for (int c = 0; c < D; c++) A.grad_y0[i * D + c] = ab[c];
  if (A.grad_params) {
#pragma unroll
    for (int q = 0; q < 8; q++) A.grad_params[i * 8 + q] = q < 3 ? pb[q] : 0.0;
  }
}

template <int M, class F>
__global__ void __launch_bounds__(128) bode_adjoint_kernel(const AdjParams A) {
  const int lane = threadIdx.x & 31;
  // one queue claim per warp and round: instances are independent, the
  // longest trajectories go first, a lane that finishes takes the next one
  while (true) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(A.queue, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= (unsigned long long)A.n) break;
    const unsigned long long pos = base + lane;
    if (pos < (unsigned long long)A.n) {
      const int64_t i = A.order ? A.order[pos] : (int64_t)pos;
      adjoint_instance<M, F>(A, i);
    }
  }
}

__global__ void traj_cost_kernel(const int64_t* off, int64_t n, double* cost) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cost[i] = (double)(off[i + 1] - off[i]) + 1.0;
}

template <int M, class F>
cudaError_t launch_adjoint(const AdjParams& A, cudaStream_t st) {
  auto kern = bode_adjoint_kernel<M, F>;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (A.n + 127) / 128;
  const int64_t blocks = (int64_t)sms * per_sm < need ? (int64_t)sms * per_sm : need;
  kern<<<(unsigned)(blocks < 1 ? 1 : blocks), 128, 0, st>>>(A);
  return cudaGetLastError();
}

template <int M>
cudaError_t dispatch_adjoint(int kind, int64_t d, const AdjParams& A, cudaStream_t st) {
  using O = FastOps;
  switch (kind) {
    case BODE_DYN_VDP:
      if (d != 2) return cudaErrorInvalidValue;
      return launch_adjoint<M, VdP<O>>(A, st);
    case BODE_DYN_LORENZ:
      if (d != 3) return cudaErrorInvalidValue;
      return launch_adjoint<M, Lorenz<O>>(A, st);
    case BODE_DYN_HARMONIC:
      if (d != 2) return cudaErrorInvalidValue;
      return launch_adjoint<M, Harmonic<O>>(A, st);
    case BODE_DYN_DAMPED:
      if (d != 2) return cudaErrorInvalidValue;
      return launch_adjoint<M, Damped<O>>(A, st);
    case BODE_DYN_MLP:
      return cudaErrorNotSupported;
    default:
      switch (d) {
        case 1: return launch_adjoint<M, Elementwise<O, 1>>(A, st);
        case 2: return launch_adjoint<M, Elementwise<O, 2>>(A, st);
        case 3: return launch_adjoint<M, Elementwise<O, 3>>(A, st);
        case 4: return launch_adjoint<M, Elementwise<O, 4>>(A, st);
        default: return cudaErrorNotSupported;
      }
  }
}

}  // namespace

static size_t adjoint_lpt_end(int64_t n) {
  return 256 + ((8 * (size_t)n + 255) & ~(size_t)255) + ((lpt_workspace_bytes(n) + 255) & ~(size_t)255);
}

// workspace: [queue counter | cost (n doubles) | LPT scratch | MLP partials]
size_t adjoint_workspace_bytes(int64_t n, int64_t d, int kind, int64_t H) {
  (void)d;
  if (kind == BODE_DYN_MLP) return mlp_adjoint_tc_bytes(n, H, BODE_METHOD_DOPRI5);  // (7 stages: the widest)
  return adjoint_lpt_end(n);
}

cudaError_t adjoint_launch(int method, int64_t d, AdjParams A, void* ws, cudaStream_t st,
                           int64_t* launches) {
  if (A.dyn.kind == BODE_DYN_MLP) return mlp_adjoint_tc_run(method, A, ws, st, launches);
  char* w = (char*)ws;
  cudaError_t e = cudaMemsetAsync(w, 0, 8, st);
  if (e != cudaSuccess) return e;
  A.queue = (unsigned long long*)w;
  double* cost = (double*)(w + 256);
  const int64_t nb = (A.n + 255) / 256;
  traj_cost_kernel<<<(unsigned)(nb < 148 * 16 ? nb : 148 * 16), 256, 0, st>>>(A.traj_offsets,
                                                                              A.n, cost);
  int64_t* order = nullptr;
  e = lpt_order(cost, A.n, w + 256 + ((8 * (size_t)A.n + 255) & ~(size_t)255), &order, st);
  if (e != cudaSuccess) return e;
  A.order = order;
  *launches += 4;  // cost + 3 LPT passes
  *launches += 1;
  switch (method) {
    case BODE_METHOD_DOPRI5: return dispatch_adjoint<BODE_METHOD_DOPRI5>(A.dyn.kind, d, A, st);
    case BODE_METHOD_TSIT5: return dispatch_adjoint<BODE_METHOD_TSIT5>(A.dyn.kind, d, A, st);
    default: return dispatch_adjoint<BODE_METHOD_HEUN>(A.dyn.kind, d, A, st);
  }
}

}  // namespace bode
