// bode_mlp.cu -- neural-ODE solve path: f(y) = W2 tanh(W1 y + b1) + b2 in
// fp32 on an fp64 state (the C4 oracle is the reference
// solve with a NumPy fp32 MLP callable).
//
// Unlike the analytic path, the dynamics here is a dense contraction over
// the whole batch, so the loop runs in lockstep like the reference's
// step_once (solver.py:208-282): every iteration evaluates the six FSAL
// stages for all *running* instances as batched MLPs, then one control
// kernel (a warp per instance) forms y_next / err, the NumPy-order RMS
// norm, the PID update, accept/reject, dense output and statuses, and
// compacts the running set for the next iteration.  Finished instances drop
// out of the GEMMs (the reference keeps them in as "overhanging" rows,
// Appendix B; results are identical, the work is not).  Stage values are
// stored as fp32 -- exactly the values the reference's float64 cast of the
// fp32 MLP output holds -- and combined in fp64 in the reference order.
//
// Stage evaluation kernel: see mlp_eval_* below (CUDA-core fp32 here; the
// tcgen05 path lives in bode_mlp_tc.cu).
#include <cstdio>

#include "bode_mlp.cuh"

namespace bode {
namespace {

constexpr int kMaxD = 128;
constexpr int kTrajRowExtra = BODE_TRAJ_EXTRA;
constexpr int kTile = 32;  // instances per block in the CUDA-core MLP

struct MlpWs {
  double* y;       // (n, D)
  float* k;        // (S, n, D)
  float* Y;        // (n, D) compacted stage input, fp32
  double* t;       // (n)
  double* dt;      // (n) controller dt
  double* h;       // (n) dt_used of the pending attempt
  double* n1;      // (n)
  double* n2;      // (n)
  double* scr;     // (3n) init scratch: d1, h0, direction
  uint8_t* trunc;  // (n)
  int32_t* act[2]; // compacted running lists
  int32_t* cnt;    // [0], [1]: list sizes; [2]: iteration
  float* wprep;    // tcgen05 path: weights pre-split into TF32 hi/lo tiles
};

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t carve(const bode_solve_args* a, char* base, MlpWs* w) {
  const size_t n = (size_t)a->n, D = (size_t)a->d;
  const size_t S = a->method == BODE_METHOD_HEUN ? 2 : 7;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += align256(bytes);
    return p;
  };
  MlpWs tmp;
  MlpWs* W = w ? w : &tmp;
  W->y = (double*)take(8 * n * D);
  W->k = (float*)take(4 * S * n * D);
  W->Y = (float*)take(4 * n * D);
  W->t = (double*)take(8 * n);
  W->dt = (double*)take(8 * n);
  W->h = (double*)take(8 * n);
  W->n1 = (double*)take(8 * n);
  W->n2 = (double*)take(8 * n);
  W->scr = (double*)take(24 * n);
  W->trunc = (uint8_t*)take(n);
  W->act[0] = (int32_t*)take(4 * n);
  W->act[1] = (int32_t*)take(4 * n);
  W->cnt = (int32_t*)take(64);
  W->wprep = (float*)take(mlp_tc_supported(a->d, a->dyn.hidden) ? mlp_tc_prep_bytes(a->dyn.hidden) : 0);
  return off;
}

// ---------------------------------------------------------------- MLP ----
// out[row of active[p]] = W2 tanh(W1 Y[p] + b1) + b2, p < count.  Y rows are
// compacted (position p), outputs scattered to the instance row.
// CUDA-core fp32 version: persistent blocks (one per SM) keep both weight
// matrices transposed in shared memory and stream tiles of kTile rows.
__global__ void __launch_bounds__(256) mlp_eval_cc_kernel(const float* __restrict__ Y,
                                                          const int32_t* __restrict__ act,
                                                          const int32_t* __restrict__ count,
                                                          const float* __restrict__ W1,
                                                          const float* __restrict__ b1,
                                                          const float* __restrict__ W2,
                                                          const float* __restrict__ b2,
                                                          int D, int H, float* __restrict__ out) {
  extern __shared__ float sm[];
  float* W1t = sm;               // D x H  (W1t[c*H + j] = W1[j][c])
  float* W2t = W1t + D * H;      // H x D  (W2t[j*D + o] = W2[o][j])
  float* Ys = W2t + H * D;       // kTile x D
  float* Hs = Ys + kTile * D;    // kTile x H
  const int cnt = *count;
  if ((int)blockIdx.x * kTile >= cnt) return;
  for (int e = threadIdx.x; e < D * H; e += blockDim.x) {
    const int j = e / D, c = e % D;  // coalesced read of W1[j][c] and W2[c][j]
    W1t[c * H + j] = W1[e];
    const int o = e / H, jj = e % H;
    W2t[jj * D + o] = W2[e];
  }
  for (int tile = blockIdx.x; tile * kTile < cnt; tile += gridDim.x) {
    const int p0 = tile * kTile;
    const int rows = cnt - p0 < kTile ? cnt - p0 : kTile;
    __syncthreads();
    for (int e = threadIdx.x; e < kTile * D; e += blockDim.x) {
      const int r = e / D;
      Ys[e] = r < rows ? Y[(size_t)(p0 + r) * D + e % D] : 0.0f;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
      float acc[kTile];
#pragma unroll
      for (int r = 0; r < kTile; r++) acc[r] = 0.0f;
      for (int c = 0; c < D; c++) {
        const float w = W1t[c * H + j];
#pragma unroll
        for (int r = 0; r < kTile; r++) acc[r] = fmaf(Ys[r * D + c], w, acc[r]);
      }
      const float bj = b1[j];
#pragma unroll
      for (int r = 0; r < kTile; r++) Hs[r * H + j] = tanhf(acc[r] + bj);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * D; e += blockDim.x) {
      const int r = e / D, o = e % D;
      const float* hr = Hs + r * H;
      float acc = 0.0f;
      for (int j = 0; j < H; j++) acc = fmaf(hr[j], W2t[j * D + o], acc);
      out[(size_t)act[p0 + r] * D + o] = acc + b2[o];
    }
  }
}

// ------------------------------------------------------ stage inputs ----
// Y[p] = fp32( y + h * sum_{j<i} a_ij k_j )  in the reference order
// (stepper.py:81-89), for p < count.
template <int M>
__global__ void mlp_stage_input_kernel(MlpWs W, int64_t n, int D, int stage) {
  using T = Tab<M>;
  const int cnt = W.cnt[0];
  const int64_t total = (int64_t)cnt * D;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(e / D), c = (int)(e % D);
    const int64_t i = W.act[0][p];
    double y = W.y[i * D + c];
    if (stage > 0) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < T::S; j++) {
        if (j >= stage) break;
        const double kj = (double)W.k[((int64_t)j * n + i) * D + c];
        s = j == 0 ? ExactOps::mul(T::a(stage, 0), kj) : ExactOps::mad(T::a(stage, j), kj, s);
      }
      y = ExactOps::mad(W.h[i], s, y);
    }
    W.Y[(int64_t)p * D + c] = (float)y;
  }
}

// ---------------------------------------------------------- control ----
struct CtrlArgs {
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
  int64_t max_steps;
  unsigned long long* max_n;
  uint32_t* refresh;
  // optional accepted-step trajectory (gradients; SolveParams::traj layout)
  double* traj;
  const int64_t* traj_offsets;
};

__device__ __forceinline__ void te_of(const CtrlArgs& A, int64_t i, int D, const double*& te,
                                      int64_t& m, double*& ys) {
  if (A.t_eval_offsets) {
    const int64_t o = A.t_eval_offsets[i];
    te = A.t_eval + o;
    m = A.t_eval_offsets[i + 1] - o;
    ys = A.ys ? A.ys + o * D : nullptr;
  } else {
    te = A.t_eval;
    m = A.t_eval_len;
    ys = A.ys ? A.ys + i * A.t_eval_len * D : nullptr;
  }
}

// one warp per running instance: the rest of step_once after the stages
template <int M>
__global__ void __launch_bounds__(128) mlp_control_kernel(MlpWs W, CtrlArgs A, int64_t n, int D) {
  using T = Tab<M>;
  __shared__ double sq[4][kMaxD];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int cnt = W.cnt[0];
  const int p = blockIdx.x * 4 + wib;
  if (p >= cnt) return;
  const int64_t i = W.act[0][p];
  const double h = W.h[i], y_t = W.t[i], t_end = A.t_end[i];
  const double atol = A.atol_v ? A.atol_v[i] : A.atol, rtol = A.rtol_v ? A.rtol_v[i] : A.rtol;
  const int nslot = (D + 31) / 32;
  const int64_t nacc_before = A.n_accepted[i];  // (read before lane 0 updates it)
  double yv[4], yn[4];
  for (int s = 0; s < nslot; s++) {
    const int c = lane + 32 * s;
    if (c >= D) break;
    const double y = W.y[i * D + c];
    double sb = 0.0, se = 0.0;
#pragma unroll
    for (int j = 0; j < T::S; j++) {
      const double kj = (double)W.k[((int64_t)j * n + i) * D + c];
      sb = j == 0 ? ExactOps::mul(T::b(0), kj) : ExactOps::mad(T::b(j), kj, sb);
      se = j == 0 ? ExactOps::mul(T::e(0), kj) : ExactOps::mad(T::e(j), kj, se);
    }
    yv[s] = y;
    yn[s] = ExactOps::mad(h, sb, y);
    const double err = ExactOps::mul(h, se);
    const double scale = ExactOps::mad(rtol, np_max(fabs(y), fabs(yn[s])), atol);
    const double r = ddiv(err, scale);
    sq[wib][c] = ExactOps::mul(r, r);
  }
  __syncwarp();
  int acc_i = 0;
  double dtn = 0.0;
  if (lane == 0) {
    double nrm = dsqrt(ddiv(pairwise_sum_rt<ExactOps>(sq[wib], D), (double)D));
    if (!isfinite(nrm)) nrm = __longlong_as_double(0x7ff0000000000000LL);
    double a1 = W.n1[i], a2 = W.n2[i];
    dtn = h;
    acc_i = adapt(A.ctrl, nrm, a1, a2, dtn);
    W.n1[i] = a1;
    W.n2[i] = a2;
  }
  acc_i = __shfl_sync(0xffffffffu, acc_i, 0);
  dtn = __shfl_sync(0xffffffffu, dtn, 0);
  const bool trunc = W.trunc[i] != 0;
  const int64_t j_iter = A.n_steps[i];
  int64_t cursor = A.n_emitted[i];
  int status = BODE_RUNNING;
  double t_new = y_t;
  if (acc_i && A.traj && nacc_before < A.traj_offsets[i + 1] - A.traj_offsets[i]) {
    // record (t_old, h, cursor, y_old) for the adjoint (rows bounded: they
    // were sized by an identical solve)
    const int W = BODE_TRAJ_STRIDE(D);
    double* rec = A.traj + (A.traj_offsets[i] + nacc_before) * W;
    if (lane == 0) {
      rec[0] = y_t;
      rec[1] = h;
      rec[2] = (double)cursor;
    }
    for (int s = 0; s < nslot; s++) {
      const int c = lane + 32 * s;
      if (c < D) rec[kTrajRowExtra + c] = yv[s];
    }
  }
  if (acc_i) {
    // dense output (solver.py:284-322) from the pre-commit state
    const double* te;
    int64_t m;
    double* ys;
    te_of(A, i, D, te, m, ys);
    if (cursor < m && h != 0.0) {
      while (cursor < m) {
        double th = ddiv(ExactOps::sub(te[cursor], y_t), h);
        if (!(th <= 1.0)) break;
        th = np_max(th, 0.0);
        double w[7];
#pragma unroll
        for (int q = 0; q < T::S; q++) {
          double v = T::w(q, T::NI - 1);
          for (int r = T::NI - 2; r >= 0; r--) v = ExactOps::mad(v, th, T::w(q, r));
          w[q] = ExactOps::mul(v, th);
        }
        for (int s = 0; s < nslot; s++) {
          const int c = lane + 32 * s;
          if (c >= D) break;
          double sacc = 0.0;
#pragma unroll
          for (int q = 0; q < T::S; q++) {
            const double kq = (double)W.k[((int64_t)q * n + i) * D + c];
            sacc = q == 0 ? ExactOps::mul(w[0], kq) : ExactOps::mad(w[q], kq, sacc);
          }
          if (ys) ys[cursor * D + c] = ExactOps::mad(h, sacc, yv[s]);
        }
        cursor++;
      }
    }
    for (int s = 0; s < nslot; s++) {
      const int c = lane + 32 * s;
      if (c >= D) break;
      W.y[i * D + c] = yn[s];
      if (T::FSAL) W.k[i * D + c] = W.k[((int64_t)(T::S - 1) * n + i) * D + c];
    }
    t_new = trunc ? t_end : ExactOps::add(y_t, h);
    if (trunc) status = BODE_SUCCESS;
  }
  if (lane == 0) {
    const int64_t ns = j_iter + 1;
    if (status == BODE_RUNNING && ExactOps::add(t_new, dtn) == t_new) status = BODE_STEP_UNDERFLOW;
    if (status == BODE_RUNNING && ns >= A.max_steps) status = BODE_MAX_STEPS_EXCEEDED;
    A.n_steps[i] = ns;
    if (acc_i) A.n_accepted[i] += 1;
    A.n_emitted[i] = cursor;
    W.t[i] = t_new;
    W.dt[i] = dtn;
    A.final_dt[i] = dtn;
    A.status[i] = status;
    if (!acc_i && status == BODE_RUNNING) {
      const uint64_t bit = (uint64_t)j_iter + 1;
      atomicOr(&A.refresh[bit >> 5], 1u << (bit & 31));
    }
    if (status == BODE_RUNNING) {
      const double rem = ExactOps::sub(t_end, t_new);
      const bool tr = fabs(dtn) >= fabs(rem);
      W.h[i] = tr ? rem : dtn;
      W.trunc[i] = tr;
      W.act[1][atomicAdd(&W.cnt[1], 1)] = (int32_t)i;
    } else {
      atomicMax(A.max_n, (unsigned long long)ns);
    }
  }
}

// swap running lists: act[0] <- act[1]; also bump the iteration counter
__global__ void mlp_swap_kernel(MlpWs W) {
  if (threadIdx.x == 0) {
    W.cnt[0] = W.cnt[1];
    W.cnt[1] = 0;
    W.cnt[2] += 1;
  }
}

// pointer swap is done by copying the list (cheap relative to the stages)
__global__ void mlp_copy_list_kernel(MlpWs W) {
  const int cnt = W.cnt[1];
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < cnt; p += gridDim.x * blockDim.x)
    W.act[0][p] = W.act[1][p];
}

// ------------------------------------------------------------- init -----
struct InitArgs {
  const double* y0;
  const double* t_start;
  const double* t_end;
  const double* atol_v;
  const double* rtol_v;
  double atol, rtol;
  int32_t dt0_mode;
  double dt0;
  const double* dt0_v;
  int order;
};

__global__ void mlp_init_a_kernel(MlpWs W, InitArgs I, int64_t n, int D) {
  const int64_t total = n * D;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    W.y[e] = I.y0[e];
    W.Y[e] = (float)I.y0[e];
    if (e % D == 0) {
      const int64_t i = e / D;
      W.act[0][i] = (int32_t)i;
      W.t[i] = I.t_start[i];
      W.n1[i] = 1.0;
      W.n2[i] = 1.0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    W.cnt[0] = (int32_t)n;
    W.cnt[1] = 0;
    W.cnt[2] = 0;
  }
}

// after f0 = MLP(y0) (in k[0]): d0, d1, h0 and the Euler probe input
// (controller.py:167-185), one warp per instance
__global__ void __launch_bounds__(128) mlp_init_b_kernel(MlpWs W, InitArgs I, int64_t n, int D) {
  __shared__ double sq[4][kMaxD];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * 4 + wib;
  if (i >= n) return;
  const double atol = I.atol_v ? I.atol_v[i] : I.atol, rtol = I.rtol_v ? I.rtol_v[i] : I.rtol;
  const double dir = (I.t_end[i] - I.t_start[i]) > 0.0 ? 1.0 : -1.0;
  const int nslot = (D + 31) / 32;
  double d0 = 0.0, d1 = 0.0, h0 = 0.0;
  for (int pass = 0; pass < 2; pass++) {
    for (int s = 0; s < nslot; s++) {
      const int c = lane + 32 * s;
      if (c >= D) break;
      const double y = W.y[i * D + c];
      const double v = pass == 0 ? y : (double)W.k[i * D + c];
      const double q = ddiv(v, ExactOps::mad(rtol, fabs(y), atol));
      sq[wib][c] = ExactOps::mul(q, q);
    }
    __syncwarp();
    if (lane == 0) {
      const double dd = dsqrt(ddiv(pairwise_sum_rt<ExactOps>(sq[wib], D), (double)D));
      if (pass == 0) d0 = dd; else d1 = dd;
    }
    __syncwarp();
  }
  if (lane == 0) {
    const bool degenerate = (d0 < 1e-5) || (d1 < 1e-5) || !isfinite(d1);
    h0 = degenerate ? 1e-6 : ddiv(__dmul_rn(0.01, d0), d1);
    W.scr[i] = d1;
    W.scr[n + i] = h0;
    W.scr[2 * n + i] = dir;
  }
  h0 = __shfl_sync(0xffffffffu, h0, 0);
  const double hd = __dmul_rn(h0, dir);
  for (int s = 0; s < nslot; s++) {
    const int c = lane + 32 * s;
    if (c >= D) break;
    W.Y[i * D + c] = (float)ExactOps::mad(hd, (double)W.k[i * D + c], W.y[i * D + c]);
  }
}

// after f1 = MLP(y1) (in k[1]): d2, h1, dt (controller.py:185-197), the
// INFINITE_DYNAMICS check, points at t_start, first dt_used; warp/instance
__global__ void __launch_bounds__(128) mlp_init_c_kernel(MlpWs W, InitArgs I, CtrlArgs A,
                                                         int64_t n, int D, int have_f1) {
  __shared__ double sq[4][kMaxD];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * 4 + wib;
  if (i >= n) return;
  const double atol = I.atol_v ? I.atol_v[i] : I.atol, rtol = I.rtol_v ? I.rtol_v[i] : I.rtol;
  const int nslot = (D + 31) / 32;
  int bad = 0;
  for (int s = 0; s < nslot; s++) {
    const int c = lane + 32 * s;
    if (c >= D) break;
    const double f0 = (double)W.k[i * D + c];
    bad |= !isfinite(f0);
    if (have_f1) {
      const double y = W.y[i * D + c];
      const double q = ddiv(ExactOps::sub((double)W.k[(n + i) * D + c], f0),
                            ExactOps::mad(rtol, fabs(y), atol));
      sq[wib][c] = ExactOps::mul(q, q);
    }
  }
  bad = __any_sync(0xffffffffu, bad);
  __syncwarp();
  if (lane != 0) return;
  double dt;
  if (have_f1) {
    const double d1 = W.scr[i], h0 = W.scr[n + i], dir = W.scr[2 * n + i];
    const double d2 = ddiv(dsqrt(ddiv(pairwise_sum_rt<ExactOps>(sq[wib], D), (double)D)), h0);
    const double dmax = np_max(d1, d2);
    const bool small = (dmax <= 1e-15) || !isfinite(dmax);
    const double h1 = small ? np_max(1e-6, __dmul_rn(h0, 1e-3))
                            : np_scalar_pow(ddiv(0.01, dmax), ddiv(1.0, (double)(I.order + 1)));
    dt = __dmul_rn(np_min(__dmul_rn(100.0, h0), h1), dir);
  } else {
    dt = I.dt0_mode == BODE_DT0_SCALAR ? I.dt0 : I.dt0_v[i];
  }
  if (bad) dt = __longlong_as_double(0x7ff8000000000000LL);
  int status = BODE_RUNNING;
  if (!isfinite(dt)) {
    status = BODE_INFINITE_DYNAMICS;
    dt = 0.0;
  }
  const double t0 = W.t[i];
  const double* te;
  int64_t m;
  double* ys;
  te_of(A, i, D, te, m, ys);
  int64_t cursor = 0;
  while (cursor < m && te[cursor] == t0) {
    if (ys)
      for (int c = 0; c < D; c++) ys[cursor * D + c] = W.y[i * D + c];
    cursor++;
  }
  A.n_emitted[i] = cursor;
  A.n_steps[i] = 0;
  A.n_accepted[i] = 0;
  A.final_dt[i] = dt;
  A.status[i] = status;
  W.dt[i] = dt;
  if (status == BODE_RUNNING) {
    const double rem = ExactOps::sub(A.t_end[i], t0);
    const bool tr = fabs(dt) >= fabs(rem);
    W.h[i] = tr ? rem : dt;
    W.trunc[i] = tr;
    W.act[1][atomicAdd(&W.cnt[1], 1)] = (int32_t)i;
  }
}

// the first stage of every attempt for non-FSAL tableaus: Y = y
__global__ void mlp_state_input_kernel(MlpWs W, int D) {
  const int cnt = W.cnt[0];
  const int64_t total = (int64_t)cnt * D;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    W.Y[e] = (float)W.y[(int64_t)W.act[0][e / D] * D + e % D];
}

inline unsigned grid_for(int64_t work, int per = 256, unsigned cap = 148 * 16) {
  const int64_t g = (work + per - 1) / per;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

size_t mlp_workspace_bytes(const bode_solve_args* a) { return carve(a, nullptr, nullptr); }

template <int M>
static cudaError_t mlp_solve_m(const bode_solve_args* a, const SolveParams& P, char* wsb,
                               cudaStream_t st, int64_t* launches) {
  using T = Tab<M>;
  const int64_t n = a->n;
  const int D = (int)a->d, H = (int)a->dyn.hidden;
  if (D > kMaxD || H > 1024) return cudaErrorNotSupported;
  MlpWs W;
  carve(a, wsb, &W);
  const float *W1 = a->dyn.W1, *b1 = a->dyn.b1, *W2 = a->dyn.W2, *b2 = a->dyn.b2;
  const size_t smem = sizeof(float) * ((size_t)2 * D * H + (size_t)kTile * (D + H));
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(mlp_eval_cc_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one path per shape (no backend switch): the 64-wide tensor-core tile
  // (fused persistent integrator when it fits TMEM, per-stage tcgen05
  // kernels for a wider hidden layer), fp32 FMA kernels for other widths
  const bool use_tc = mlp_tc_supported(D, H);
  const bool use_fused = use_tc && mlp_fused_supported(D, H, a->method);
  // the recorded stage inputs (tensor-core backward) come from the fused kernel
  if (a->traj && a->traj_stages && !use_fused) return cudaErrorNotSupported;
  if (use_tc && (e = mlp_tc_prep(W1, W2, H, W.wprep, st)) != cudaSuccess) return e;
  int64_t nl = use_tc ? 1 : 0;  // kernels launched
  const int max_tiles = (int)((n + 127) / 128);
  // f(Y) for the compacted fp32 rows in W.Y (init evaluations)
  auto eval = [&](float* out) {
    if (use_tc) {
      MlpTcArgs t{n, H, 0, W.y, W.k, W.h, W.act[0], W.cnt, W.Y, W.wprep, b1, b2, out};
      mlp_tc_launch<M>(t, max_tiles, st);
      nl += 1;
      return;
    }
    nl += 1;
    // one persistent block per SM; blocks past the live tile count exit
    const unsigned g = grid_for(n, kTile, (unsigned)sms);
    mlp_eval_cc_kernel<<<g, 256, smem, st>>>(W.Y, W.act[0], W.cnt, W1, b1, W2, b2, D, H, out);
  };
  // stage s of the current attempt: input formed from y, h and k_0..k_{s-1}
  auto stage = [&](int s) {
    if (use_tc) {  // prologue fused into the tensor-core kernel
      MlpTcArgs t{n, H, s, W.y, W.k, W.h, W.act[0], W.cnt, nullptr, W.wprep, b1, b2,
                  W.k + (size_t)s * n * D};
      mlp_tc_launch<M>(t, max_tiles, st);
      nl += 1;
      return;
    }
    nl += 1;
    if (s == 0)
      mlp_state_input_kernel<<<grid_for(n * D), 256, 0, st>>>(W, D);
    else
      mlp_stage_input_kernel<M><<<grid_for(n * D), 256, 0, st>>>(W, n, D, s);
    eval(W.k + (size_t)s * n * D);
  };
  InitArgs I{a->y0, a->t_start, a->t_end, a->atol_v, a->rtol_v, a->atol, a->rtol,
             a->dt0_mode, a->dt0, a->dt0_v, T::ORDER};
  CtrlArgs A{P.ctrl, a->t_end, a->atol_v, a->rtol_v, a->atol, a->rtol, a->t_eval,
             a->t_eval_offsets, a->t_eval_offsets ? 0 : a->t_eval_len, a->ys, a->n_emitted,
             a->n_steps, a->n_accepted, a->final_dt, a->status, a->max_steps, P.max_n,
             P.refresh, a->traj, a->traj_offsets};
  mlp_init_a_kernel<<<grid_for(n * D), 256, 0, st>>>(W, I, n, D);
  eval(W.k);  // f0 = f(t0, y0)
  const bool heur = a->dt0_mode == BODE_DT0_HEURISTIC;
  if (heur) {
    mlp_init_b_kernel<<<(unsigned)((n + 3) / 4), 128, 0, st>>>(W, I, n, D);
    eval(W.k + (size_t)n * D);  // f1 = f(t0 + h0 dir, y1) into the k[1] slot
  }
  mlp_init_c_kernel<<<(unsigned)((n + 3) / 4), 128, 0, st>>>(W, I, A, n, D, heur ? 1 : 0);
  mlp_copy_list_kernel<<<grid_for(n), 256, 0, st>>>(W);
  mlp_swap_kernel<<<1, 32, 0, st>>>(W);
  nl += heur ? 5 : 4;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;

  if (use_fused) {  // one persistent launch runs every running instance to the end
    MlpFusedArgs F;
    F.H = H;
    F.max_steps = a->max_steps;
    F.act = W.act[0];  // running list after the init pass's copy + swap
    F.count = W.cnt;
    F.queue = P.queue;
    F.y = W.y;
    F.f0 = W.k;
    F.t = W.t;
    F.dt = W.dt;
    F.wprep = W.wprep;
    F.b1 = b1;
    F.b2 = b2;
    F.ctrl = P.ctrl;
    F.t_end = a->t_end;
    F.atol_v = a->atol_v;
    F.rtol_v = a->rtol_v;
    F.atol = a->atol;
    F.rtol = a->rtol;
    F.t_eval = a->t_eval;
    F.t_eval_offsets = a->t_eval_offsets;
    F.t_eval_len = a->t_eval_offsets ? 0 : a->t_eval_len;
    F.ys = a->ys;
    F.n_emitted = a->n_emitted;
    F.n_steps = a->n_steps;
    F.n_accepted = a->n_accepted;
    F.final_dt = a->final_dt;
    F.status = a->status;
    F.max_n = P.max_n;
    F.refresh = P.refresh;
    F.prof = nullptr;
    F.traj = a->traj;
    F.traj_y = a->traj ? a->traj_stages : nullptr;
    F.fast = a->mode == BODE_MODE_FAST;
    F.traj_offsets = a->traj_offsets;
#ifdef BODE_FUSED_PROF
    static unsigned long long* prof_buf = nullptr;
    if (!prof_buf) cudaMalloc(&prof_buf, 148 * 3 * 32 * 8);
    cudaMemsetAsync(prof_buf, 0, 148 * 3 * 32 * 8, st);
    F.prof = prof_buf;
#endif
    if (P.ev_start) cudaEventRecord((cudaEvent_t)P.ev_start, st);
    e = mlp_fused_launch<M>(F, st);
#ifdef BODE_FUSED_PROF
    {
      unsigned long long h[148 * 3 * 32];
      cudaMemcpyAsync(h, prof_buf, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      for (int v = 0; v < 3; v++) {
        double acc[32] = {0};
        for (int b = 0; b < 148; b++)
          for (int k = 0; k < 32; k++) acc[k] += h[(b * 3 + v) * 32 + k] / 148.0;
        fprintf(stderr, "fused prof view %d:", v);
        for (int k = 0; k < 32; k++)
          if (acc[k] != 0) fprintf(stderr, " [%d]=%.0f", k, acc[k]);
        fprintf(stderr, "\n");
      }
    }
#endif
    if (P.ev_stop) cudaEventRecord((cudaEvent_t)P.ev_stop, st);
    if (launches) *launches += nl + 1;
    return e;
  }

  // lockstep iterations in bursts; each burst ends with one host read of the
  // running count (kernels of a drained batch exit immediately)
  int32_t* h_cnt = nullptr;
  if ((e = cudaMallocHost((void**)&h_cnt, sizeof(int32_t))) != cudaSuccess) return e;
  int64_t iters = 0;
  int burst = 4;
  while (true) {
    for (int b = 0; b < burst; b++) {
      for (int s = T::FSAL ? 1 : 0; s < T::S; s++) stage(s);
      mlp_control_kernel<M><<<(unsigned)((n + 3) / 4), 128, 0, st>>>(W, A, n, D);
      mlp_copy_list_kernel<<<grid_for(n), 256, 0, st>>>(W);
      mlp_swap_kernel<<<1, 32, 0, st>>>(W);
      nl += 3;
    }
    iters += burst;
    if ((e = cudaMemcpyAsync(h_cnt, W.cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
    if (*h_cnt == 0 || iters >= a->max_steps + 1) break;
    burst = burst < 32 ? burst * 2 : 32;
  }
  cudaFreeHost(h_cnt);
  if (launches) *launches += nl;
  return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t mlp_solve(const bode_solve_args* a, const SolveParams& P, char* ws, cudaStream_t st,
                      int64_t* launches) {
  switch (a->method) {
    case BODE_METHOD_DOPRI5: return mlp_solve_m<BODE_METHOD_DOPRI5>(a, P, ws, st, launches);
    case BODE_METHOD_TSIT5: return mlp_solve_m<BODE_METHOD_TSIT5>(a, P, ws, st, launches);
    default: return mlp_solve_m<BODE_METHOD_HEUN>(a, P, ws, st, launches);
  }
}

}  // namespace bode
