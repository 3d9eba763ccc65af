// bode_mlp.cu -- neural-ODE solve path: f(y) = W2 tanh(W1 y + b1) + b2 in
// fp32 on an fp64 state (the C4 oracle is the reference
// solve with a NumPy fp32 MLP callable).
//
// One path: BatchSolver.__init__ for every row as a batched init pass (f0,
// the Hairer probe evaluation, dt0, INFINITE_DYNAMICS, points at t_start;
// the two MLP evaluations on the tensor cores, bode_mlp_tc.cu), then ONE
// launch of the fused persistent tcgen05 integrator (bode_mlp_fused.cu) that
// runs every running row to termination.  The network must fill the 64-wide
// tensor-core tile (d == 64, hidden a multiple of 32 up to 256; bode_abi.cu
// validates it): narrower networks are zero-padded by the caller (the
// Python facade does it, dynamics.mlp_pad).
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

// NumPy's pairwise sum (pairwise_sum_rt) of sq[0..D) across a warp: for
// 8 <= D <= 128, D % 8 == 0 (the MLP tile, D = 64) lanes 0-7 run the eight
// strided accumulators and three shuffle levels form the fixed tree
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) -- bitwise the serial result, in
// lane 0; other widths sum serially in lane 0
__device__ __forceinline__ double warp_pairwise_sum(const double* sq, int D, int lane) {
  if (D < 8 || D > 128 || D % 8 != 0)
    return lane == 0 ? pairwise_sum_rt<ExactOps>(sq, D) : 0.0;
  double r = 0.0;
  if (lane < 8) {
    r = sq[lane];
    for (int i = 8; i < D; i += 8) r = ExactOps::add(r, sq[i + lane]);
  }
  r = ExactOps::add(r, __shfl_down_sync(0xffffffffu, r, 1));
  r = ExactOps::add(r, __shfl_down_sync(0xffffffffu, r, 2));
  return ExactOps::add(r, __shfl_down_sync(0xffffffffu, r, 4));
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
    const double ssum = warp_pairwise_sum(sq[wib], D, lane);
    if (lane == 0) {
      const double dd = dsqrt(ddiv(ssum, (double)D));
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
  const double ssum = have_f1 ? warp_pairwise_sum(sq[wib], D, lane) : 0.0;
  if (lane != 0) return;
  double dt;
  if (have_f1) {
    const double d1 = W.scr[i], h0 = W.scr[n + i], dir = W.scr[2 * n + i];
    const double d2 = ddiv(dsqrt(ddiv(ssum, (double)D)), h0);
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
  if (!mlp_fused_supported(D, H, a->method)) return cudaErrorNotSupported;  // (validated)
  MlpWs W;
  carve(a, wsb, &W);
  const float *W1 = a->dyn.W1, *b1 = a->dyn.b1, *W2 = a->dyn.W2, *b2 = a->dyn.b2;
  cudaError_t e = mlp_tc_prep(W1, W2, H, W.wprep, st);
  if (e != cudaSuccess) return e;
  int64_t nl = 1;  // kernels launched
  const int max_tiles = (int)((n + 127) / 128);
  // f(Y) for the compacted fp32 rows in W.Y (init evaluations)
  auto eval = [&](float* out) {
    MlpTcArgs t{n, H, 0, W.y, W.k, W.h, W.act[0], W.cnt, W.Y, W.wprep, b1, b2, out};
    mlp_tc_launch<M>(t, max_tiles, st);
    nl += 1;
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

  {  // one persistent launch runs every running instance to the end
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
