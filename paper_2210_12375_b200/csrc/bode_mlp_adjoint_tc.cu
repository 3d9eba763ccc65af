// bode_mlp_adjoint_tc.cu -- the neural-ODE backward (SURVEY.md §8(f) row 1,
// torchode's AutoDiffAdjoint for f(y) = W2 tanh(W1 y + b1) + b2) with every
// contraction on the 5th-generation tensor cores.
//
// Same definition as the analytic adjoint (bode_adjoint.cu): reverse mode
// through the recorded accepted steps -- stages, solution update, dense
// output -- with step sizes and accept decisions held fixed; outputs dL/dy0
// per instance and dL/dW1, db1, dW2, db2 summed over the batch.  The network
// fills the 64-wide tile (narrower ones are zero-padded by the caller).
//
// The rows are ordered by trajectory length, longest first (a stable radix
// sort, so the order -- and every sum below -- is deterministic), and the
// trajectories are reversed in lockstep: reverse iteration `it` undoes step
// nrec-1-it of every row with nrec > it, i.e. of a prefix of the order.  Per
// iteration:
//   load     the step records of the live rows (t_old, h, cursor, y_old);
//            the fp32 stage inputs Y_s come from the recording solve
//            (bode_solve_args.traj_stages, written by the fused forward
//            kernel), so no forward stage is recomputed
//   seeds    dL/dk_s from dL/dy_next and the dense-output points of the step
//   reverse  per stage s = S-1 .. 0, one tcgen05 kernel per 128-row tile:
//              Z  = Y_s W1^T          (recomputed pre-activation, M=128 N=32 K=64)
//              V  = g_s W2            (W2^T pre-split chunks, M=128 N=32 K=64)
//              u  = V (1 - tanh(Z + b1)^2)         (epilogue, CUDA cores)
//              Yb = sum_c u_c W1_c    (W1^T pre-split chunks, M=128 N=64 K=32)
//            Y_s, g_s and u_c are the MMAs' A operands in TMEM; each stage's
//            Yb is stored, and the later launches' producers form
//            dL/dk_j = seed + sum h a_sj Yb (j < s); a fold pass adds the
//            Yb to dL/dy_old; u^T, tanh^T, Y_s^T, g_s^T are written to global
//            memory transposed (slice-contiguous blocks, 128 contiguous
//            bytes per warp store)
//   weights  one split-K tcgen05 GEMM over the iteration's (stage, row)
//            columns: dW1 | db1 = u^T [Y | 1] (M=128 per half of H, N=80),
//            dW2 | db2 = g^T [tanh | 1] (M=64, both halves interleaved in
//            TMEM lanes 0-15 / 16-31 of each quadrant, N=144 / 128).
// Every operand is K-major (tf32 MN-major descriptors read as zeros on this
// part, tools/umma_probe.cu), so contractions over the rows read the
// transposed copies.  3xTF32 throughout (hi*hi + hi*lo + lo*hi, fp32
// accumulation), like the forward.
#include <cub/cub.cuh>

#include "bode_adjoint.cuh"
#include "bode_mlp.cuh"
#include "bode_solver.cuh"
#include "bode_tc.cuh"

namespace bode {
namespace adjtc {
using namespace tc;

constexpr int kW = BODE_TRAJ_STRIDE(kD);  // trajectory row (doubles)
constexpr int kN1 = 80;                   // dW1 | db1 accumulator width
constexpr int kN2 = 144;                  // dW2 | db2 (half 0) width
constexpr int kPartFloats = 2 * 128 * kN1 + 2 * 64 * kN2;  // one CTA's partial sums

// The transposed weight-gradient operands (u^T, tanh^T: H rows; Y^T, g^T: 64
// rows) are stored in 32-column blocks, [col / 32][row][col % 32], so one
// K-slice of the GEMM is a contiguous block and a warp of row threads (32
// consecutive columns) still writes 128 contiguous bytes per row.
__host__ __device__ __forceinline__ int64_t blk(int64_t row, int64_t col, int64_t rows) {
  return ((col >> 5) * rows + row) * 32 + (col & 31);
}

__host__ __device__ constexpr uint32_t idesc_mn(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// ---------------------------------------------------------------- glue ----

__global__ void keys_kernel(const int64_t* off, int64_t n, int32_t* keys, int32_t* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (int32_t)(off[i + 1] - off[i]);
    idx[i] = (int32_t)i;
  }
}

__global__ void transpose_kernel(const float* in, int rows, int cols, float* out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x)
    out[(e % cols) * rows + e / cols] = in[e];
}

struct RowState {
  int64_t n, pmax;
  const int32_t* order;  // LPT position -> instance
  const int32_t* nrec;   // LPT position -> trajectory length (descending)
  int32_t* count;        // rows live in this iteration
  int64_t* hi;           // first point of the later step (the previous lo)
  int64_t* lo;           // cursor of the step being reversed
  int64_t* rec;          // trajectory row of the step being reversed
  double* t_old;
  double* h;
  double* y;             // (n, 64) y_old
  double* kb;            // (S, n, 64) dL/dk_s
  double* yb;            // (n, 64) dL/dy (carried as dL/dy_next to the next iteration)
};

__global__ void init_kernel(RowState R, const int64_t* n_emitted) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < R.n * kD;
       e += (int64_t)gridDim.x * blockDim.x) {
    R.yb[e] = 0.0;
    if (e % kD == 0) R.lo[e / kD] = n_emitted[R.order[e / kD]];
  }
}

// rows live at iteration it: nrec is sorted descending
__global__ void count_kernel(RowState R, int64_t it) {
  int64_t lo = 0, hi = R.n;  // first position with nrec <= it
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (R.nrec[mid] > it) lo = mid + 1; else hi = mid;
  }
  *R.count = (int32_t)lo;
}

__global__ void load_kernel(RowState R, const double* traj, const int64_t* traj_off, int64_t it) {
  const int64_t cnt = *R.count;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt * kD;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / kD;
    const int c = (int)(e % kD);
    const int64_t i = R.order[p];
    const double* rec = traj + (traj_off[i] + R.nrec[p] - 1 - it) * kW;
    R.y[e] = rec[kTrajExtra + c];
    if (c == 0) {  // (only this thread touches the row's hi / lo)
      R.rec[p] = traj_off[i] + R.nrec[p] - 1 - it;
      R.t_old[p] = rec[0];
      R.h[p] = rec[1];
      R.hi[p] = R.lo[p];
      R.lo[p] = (int64_t)rec[2];
    }
  }
}

// dL/dk_s seeds of the step: y_next = y + h sum b_s k_s and the Horner dense
// output of the points in [lo, hi) (bode_mlp_adjoint.cu, same operations)
template <int M>
__global__ void seeds_kernel(RowState R, const double* t_eval, const int64_t* t_eval_offsets,
                             int64_t t_eval_len, const double* grad_ys) {
  using T = Tab<M>;
  constexpr int S = T::S, NI = T::NI;
  const int64_t cnt = *R.count;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt * kD;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / kD;
    const int c = (int)(e % kD);
    const int64_t i = R.order[p];
    const double h = R.h[p], a0 = R.yb[e];
    double kb[S];
#pragma unroll
    for (int s = 0; s < S; s++) kb[s] = (h * T::b(s)) * a0;
    double y_b = a0;
    const double* te = t_eval_offsets ? t_eval + t_eval_offsets[i] : t_eval;
    const double* gy = t_eval_offsets ? grad_ys + t_eval_offsets[i] * kD : grad_ys + i * t_eval_len * kD;
    const double t_old = R.t_old[p];
    const int64_t hi = R.hi[p];
    for (int64_t q = R.lo[p]; q < hi; q++) {
      double theta = ddiv(te[q] - t_old, h);
      theta = np_max(theta, 0.0);
      const double g = gy[q * kD + c];
      y_b += g;
#pragma unroll
      for (int s = 0; s < S; s++) {
        double v = T::w(s, NI - 1);
#pragma unroll
        for (int j = NI - 2; j >= 0; j--) v = fma(v, theta, T::w(s, j));
        kb[s] = fma(h * (v * theta), g, kb[s]);
      }
    }
#pragma unroll
    for (int s = 0; s < S; s++) R.kb[(s * R.n + p) * kD + c] = kb[s];
    R.yb[e] = y_b;
  }
}

// dL/dy_old = dL/dy_next + points + sum over the stages (reversed order)
template <int M>
__global__ void fold_kernel(RowState R, const float* Ybar) {
  constexpr int S = Tab<M>::S;
  const int64_t cnt = *R.count;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt * kD;
       e += (int64_t)gridDim.x * blockDim.x) {
    double v = R.yb[e];
#pragma unroll
    for (int s = S - 1; s >= 0; s--) v += (double)Ybar[(int64_t)s * R.n * kD + e];
    R.yb[e] = v;
  }
}

__global__ void finish_kernel(RowState R, const double* grad_ys, const int64_t* t_eval_offsets,
                              int64_t t_eval_len, double* grad_y0) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < R.n * kD;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / kD;
    const int c = (int)(e % kD);
    const int64_t i = R.order[p];
    const double* gy = t_eval_offsets ? grad_ys + t_eval_offsets[i] * kD : grad_ys + i * t_eval_len * kD;
    double a0 = R.yb[e];
    const int64_t first = R.lo[p];  // cursor of the row's first step
    for (int64_t q = 0; q < first; q++) a0 += gy[q * kD + c];  // points at t_start
    grad_y0[i * kD + c] = a0;
  }
}

// -DBODE_ADJ_PROF (debug builds): per-phase clock64 stamps of CTA 0 in the
// stage-3 launch, lane 0 of warp 0 (a row owner) and of warp 8 (MMA issue),
// read by bode_debug_adj_prof
#ifdef BODE_ADJ_PROF
__device__ long long g_adj_prof[2][512];
__device__ int g_adj_prof_n[2];
#define ADJ_STAMP(w, tag)                                                             \
  if (blockIdx.x == 0 && A.stage == 3) {                                              \
    const int k_ = g_adj_prof_n[w]++;                                                 \
    if (k_ < 256) {                                                                   \
      g_adj_prof[w][2 * k_] = tag;                                                    \
      g_adj_prof[w][2 * k_ + 1] = clock64();                                          \
    }                                                                                 \
  }
#else
#define ADJ_STAMP(w, tag)
#endif

// ------------------------------------------------- reverse stage (VJP) ----

struct VjpArgs {
  int64_t n, pmax;
  int H, stage;
  const int32_t* count;
  const double* y;          // (n, 64) y_old of the step (Y_0 = (float) y_old)
  const float* Ystages;     // (rows, S, 64) recorded fp32 stage inputs
  const int64_t* rec;       // (n) trajectory row of the step
  const double* h;
  const double* kb;   // (S, n, 64) dL/dk_s seeds (dense output, y_next)
  float* Ybar;        // (S, n, 64) dL/dY_s of every stage reversed so far
  const float* wfwd;  // forward chunks [W1_c | W2_c] (hi | lo each)
  const float* wadj;  // adjoint chunks [(W2^T)_c | (W1^T)_c]
  const float* b1;
  float *uT, *AT, *YT, *gT;  // blocked (rows, S * pmax), column = stage * pmax + row
};

// Every A operand lives in tensor memory (tcgen05.mma's A-from-TMEM form:
// one row per lane, K along the columns), so the MMAs read only the weights
// from shared memory -- N = 32 MMAs with both operands in shared memory are
// bound by its operand bandwidth.  TMEM columns (512):
//   0 / 64      Y_s hi / lo          128 / 192   g_s hi / lo
//   256 + 64 b  chunk buffer b: Z | V accumulators (32 + 32), overwritten
//               by the epilogue with u_c hi | lo (the A of the Yb GEMM)
//   384         Yb accumulator (64)
// Shared memory holds the weights of two hidden chunks in flight (buffer =
// chunk sequence number & 1).
struct VjpSmem {
  uint8_t w1[2][2][kW1];     // [buf] W1_c hi, lo
  uint8_t wv[2][2][kW1];     // [buf] (W2^T)_c hi, lo
  uint8_t wy[2][2][kW2];     // [buf] (W1^T)_c hi, lo
  float b1[256];
  uint64_t full, wa[2], wy_full[2], g1[2], g2[2], epi[2];
  uint32_t tmem_base;
};

constexpr int kVjpThreads = 288;  // 2 row-owner warpgroups + the MMA warp
__device__ __forceinline__ void rows_sync() {  // the 256 row-owner threads
  asm volatile("bar.sync 1, 256;" ::: "memory");
}

// Production of one tile row's half (columns [32 h, 32 h + 32)) of the
// stage input Y_s and of g_s = dL/dk_s, into the TMEM TF32 hi/lo operand
// columns of the row's lane (trow) and the transposed global copies.  Y_s is the recorded stage input
// (Y_0 = y_old); g_s is the seed plus, in the order the stages were
// reversed (S-1 down to s+1), h a_s's dL/dY_s'.
template <int M>
__device__ __forceinline__ void vjp_produce(const VjpArgs& A, int64_t p, bool lv, int h,
                                            uint32_t trow) {
  using T = Tab<M>;
  const int stage = A.stage;
  const int64_t col = (int64_t)stage * A.pmax + p;
  const int c0 = 32 * h;
  float x[32], g[32];
  if (!lv) {
#pragma unroll
    for (int e = 0; e < 32; e++) x[e] = g[e] = 0.0f;
  } else {
    if (stage == 0) {  // y_old itself, rounded as the forward rounded it
      const double2* yp = reinterpret_cast<const double2*>(A.y + p * kD + c0);
#pragma unroll
      for (int e = 0; e < 16; e++) {
        const double2 d = __ldg(yp + e);
        x[2 * e] = (float)d.x, x[2 * e + 1] = (float)d.y;
      }
    } else {  // the recording solve's stage input
      const float4* yp =
          reinterpret_cast<const float4*>(A.Ystages + (A.rec[p] * T::S + stage) * kD + c0);
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const float4 v = __ldg(yp + e);
        x[4 * e] = v.x, x[4 * e + 1] = v.y, x[4 * e + 2] = v.z, x[4 * e + 3] = v.w;
      }
    }
    const double hp = A.h[p];
    const double* kp = A.kb + ((int64_t)stage * A.n + p) * kD + c0;
#pragma unroll
    for (int g8 = 0; g8 < 4; g8++) {
      double acc[8];
      float yv[T::S][8];
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const double2 d = __ldg(reinterpret_cast<const double2*>(kp + 8 * g8) + e);
        acc[2 * e] = d.x, acc[2 * e + 1] = d.y;
      }
#pragma unroll
      for (int s2 = T::S - 1; s2 > 0; s2--) {
        if (s2 <= stage || T::za(s2, stage) == 0.0) continue;
        const float4* yp = reinterpret_cast<const float4*>(A.Ybar + ((int64_t)s2 * A.n + p) * kD + c0 + 8 * g8);
        const float4 a = __ldg(yp), b = __ldg(yp + 1);
        yv[s2][0] = a.x, yv[s2][1] = a.y, yv[s2][2] = a.z, yv[s2][3] = a.w;
        yv[s2][4] = b.x, yv[s2][5] = b.y, yv[s2][6] = b.z, yv[s2][7] = b.w;
      }
#pragma unroll
      for (int s2 = T::S - 1; s2 > 0; s2--) {
        if (s2 <= stage || T::za(s2, stage) == 0.0) continue;
        const double w = hp * T::a(s2, stage);
#pragma unroll
        for (int e = 0; e < 8; e++) acc[e] = fma(w, (double)yv[s2][e], acc[e]);
      }
#pragma unroll
      for (int e = 0; e < 8; e++) g[8 * g8 + e] = (float)acc[e];
    }
#pragma unroll
    for (int e = 0; e < 32; e++) {
      A.YT[blk(c0 + e, col, kD)] = x[e];
      A.gT[blk(c0 + e, col, kD)] = g[e];
    }
  }
  // TF32 hi / lo of this half into the A-operand columns (lane = row)
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const float* v = q < 2 ? x + 16 * q : g + 16 * (q - 2);
    float hi[16], lo[16];
#pragma unroll
    for (int e = 0; e < 16; e++) {
      hi[e] = tf32_hi(v[e]);
      lo[e] = v[e] - hi[e];
    }
    const uint32_t col = (q < 2 ? 0 : 128) + c0 + 16 * (q & 1);
    tmem_st16(trow + col, hi);
    tmem_st16(trow + col + 64, lo);
  }
  tmem_wait_st();
}

// L2 prefetch of what vjp_produce will read for row p (this thread's column
// half) one tile ahead, issued while the current tile's chunks run on the
// tensor cores: production then waits on L2 instead of HBM latency
template <int M>
__device__ __forceinline__ void vjp_prefetch(const VjpArgs& A, int64_t p, int cnt, int h) {
  using T = Tab<M>;
  if (p >= cnt) return;
  auto pf = [](const void* q) { asm volatile("prefetch.global.L2 [%0];" ::"l"(q)); };
  const int stage = A.stage, c0 = 32 * h;
  if (stage == 0) {
    pf(A.y + p * kD + c0);
    pf(A.y + p * kD + c0 + 16);
  } else {
    pf(A.Ystages + (A.rec[p] * T::S + stage) * kD + c0);
  }
  const double* kp = A.kb + ((int64_t)stage * A.n + p) * kD + c0;
  pf(kp);
  pf(kp + 16);
#pragma unroll
  for (int s2 = T::S - 1; s2 > 0; s2--) {
    if (s2 <= stage || T::za(s2, stage) == 0.0) continue;
    pf(A.Ybar + ((int64_t)s2 * A.n + p) * kD + c0);
  }
}

// One CTA per SM, tiles of 128 rows; warps 0-3 and 4-7 own the rows (thread
// = row = TMEM lane) and split the columns of every production and
// epilogue; warp 8 issues every MMA and weight copy.  Per hidden chunk c:
// Z/V of chunk c+1 run on the tensor cores while the row owners do the
// epilogue of chunk c, and Yb of chunk c after it.
template <int M>
__global__ void __launch_bounds__(kVjpThreads, 1) vjp_kernel(const VjpArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  VjpSmem& S = *reinterpret_cast<VjpSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cnt = *A.count;
  const int ntiles = (cnt + kRows - 1) / kRows;
  if ((int)blockIdx.x >= ntiles) return;
  const int nchunk = A.H / kHc;
  const int my_tiles = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int total = my_tiles * nchunk;  // chunk sequence numbers q of this CTA

  if (tid == 0) {
    mbar_init(&S.full, 1);
    for (int b = 0; b < 2; b++) {
      mbar_init(&S.wa[b], 1);
      mbar_init(&S.wy_full[b], 1);
      mbar_init(&S.g1[b], 1);
      mbar_init(&S.g2[b], 1);
      mbar_init(&S.epi[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = tid; j < A.H; j += blockDim.x) S.b1[j] = A.b1[j];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&S.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  // TMEM columns: Z / V accumulators of chunk buffer b at 64 b / 64 b + 32,
  // Yb at 128, u_c hi / lo of buffer b at 192 + 64 b / 192 + 64 b + 32
  const uint32_t tmem = S.tmem_base;
  const uint32_t accY = tmem + 384;
  auto phase = [](int q) { return (uint32_t)((q >> 1) & 1); };

  if (warp == 8) {
    // ======================= MMA issue =======================
    // The whole warp runs the control flow, so the descriptors and TMEM
    // addresses are warp-uniform values in uniform registers; one elected
    // lane issues each batch of MMAs / copies.  (Issuing from a single-lane
    // branch makes the compiler move every operand into uniform registers
    // through a per-MMA R2UR.BROADCAST loop: ~60 cycles per MMA against
    // 16 / 33 for an N = 32 / 64 TS MMA, tools/mma_cost.cu.)
    const char* wf = (const char*)A.wfwd;
    const char* wa = (const char*)A.wadj;
    auto load_wa = [&](int q) {  // W1_c and (W2^T)_c of chunk q into buffer q & 1
      const int b = q & 1, c = q % nchunk;
      if (elect_one()) {
        mbar_expect_tx(&S.wa[b], 4 * kW1);
        bulk_g2s(S.w1[b][0], wf + (size_t)c * kWChunk, kW1, &S.wa[b]);
        bulk_g2s(S.w1[b][1], wf + (size_t)c * kWChunk + kW1, kW1, &S.wa[b]);
        bulk_g2s(S.wv[b][0], wa + (size_t)c * kWChunk, kW1, &S.wa[b]);
        bulk_g2s(S.wv[b][1], wa + (size_t)c * kWChunk + kW1, kW1, &S.wa[b]);
      }
      __syncwarp();
    };
    auto load_wy = [&](int q) {  // (W1^T)_c
      const int b = q & 1, c = q % nchunk;
      if (elect_one()) {
        mbar_expect_tx(&S.wy_full[b], 2 * kW2);
        bulk_g2s(S.wy[b][0], wa + (size_t)c * kWChunk + 2 * kW1, kW2, &S.wy_full[b]);
        bulk_g2s(S.wy[b][1], wa + (size_t)c * kWChunk + 2 * kW1 + kW2, kW2, &S.wy_full[b]);
      }
      __syncwarp();
    };
    auto issue_zv = [&](int q) {  // Z = Y_s W1_c^T, V = g_s (W2^T)_c^T into buffer q & 1
      const int b = q & 1;
      mbar_wait(&S.wa[b], phase(q));
      if (q >= 2) mbar_wait(&S.g2[b], phase(q - 2));  // Yb(q-2) read u from this buffer
      const uint32_t az = tmem + 256 + 64 * b, av = az + 32;
      const uint64_t w1[2] = {smem_desc(smem_u32(S.w1[b][0]), 2048), smem_desc(smem_u32(S.w1[b][1]), 2048)};
      const uint64_t wv[2] = {smem_desc(smem_u32(S.wv[b][0]), 2048), smem_desc(smem_u32(S.wv[b][1]), 2048)};
      if (elect_one()) {
        fence_after();
        const int tb[3] = {0, 1, 0};
        const uint32_t ya[3] = {tmem, tmem, tmem + 64}, ga[3] = {tmem + 128, tmem + 128, tmem + 192};
#pragma unroll
        for (int s = 0; s < kD / 8; s++)
#pragma unroll
          for (int term = 0; term < 3; term++) {
            mma_tf32_ts(az, ya[term] + 8 * s, w1[tb[term]] + 16 * s, idesc(kHc), (term | s) ? 1u : 0u);
            mma_tf32_ts(av, ga[term] + 8 * s, wv[tb[term]] + 16 * s, idesc(kHc), (term | s) ? 1u : 0u);
          }
        mma_commit(&S.g1[b]);
      }
      __syncwarp();
    };
    auto issue_yb = [&](int q, int c) {  // Yb += u_c (W1^T)_c^T (A from TMEM)
      const int b = q & 1;
      mbar_wait(&S.epi[b], phase(q));
      mbar_wait(&S.wy_full[b], phase(q));
      const uint32_t uhi = tmem + 256 + 64 * b, ulo = uhi + 32;
      const uint64_t wh = smem_desc(smem_u32(S.wy[b][0]), 1024);
      const uint64_t wl = smem_desc(smem_u32(S.wy[b][1]), 1024);
      if (elect_one()) {
        fence_after();
#pragma unroll
        for (int s = 0; s < kHc / 8; s++) {
          mma_tf32_ts(accY, uhi + 8 * s, wh + 16 * s, idesc(kD), (c | s) ? 1u : 0u);
          mma_tf32_ts(accY, uhi + 8 * s, wl + 16 * s, idesc(kD), 1u);
          mma_tf32_ts(accY, ulo + 8 * s, wh + 16 * s, idesc(kD), 1u);
        }
        mma_commit(&S.g2[b]);
      }
      __syncwarp();
    };
    load_wa(0);
    load_wy(0);
    if (total > 1) {
      load_wa(1);
      load_wy(1);
    }
    for (int kl = 0; kl < my_tiles; kl++) {
      mbar_wait(&S.full, kl & 1);  // tiles produced; the previous tile's Yb read out
      if (lane == 0) { ADJ_STAMP(1, 10) }
      const int q0 = kl * nchunk;
      issue_zv(q0);
      for (int c = 0; c < nchunk; c++) {
        const int q = q0 + c;
        if (c + 1 < nchunk) issue_zv(q + 1);
        if (lane == 0) { ADJ_STAMP(1, 20) }
        // weights of chunk q+2 into buffer q & 1 once ZV(q) has read it
        mbar_wait(&S.g1[q & 1], phase(q));
        if (q + 2 < total) load_wa(q + 2);
        issue_yb(q, c);
        if (lane == 0) { ADJ_STAMP(1, 21) }
        if (q >= 1) {  // Yb(q-1) done: its (W1^T) buffer takes chunk q+1
          mbar_wait(&S.g2[(q - 1) & 1], phase(q - 1));
          if (q + 1 < total) load_wy(q + 1);
        }
      }
    }
  } else {
    // ============ row owners: production + epilogues (column half h) ============
    const int h = warp >> 2, r = tid & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    int kl = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, kl++) {
      const int64_t p = (int64_t)tile * kRows + r;
      const bool live = p < cnt;
      const int64_t col = (int64_t)A.stage * A.pmax + p;
      // (Y_s / g_s tiles free: every ZV of the previous tile was waited for
      // by its last epilogue; the previous Yb was read out below)
      if (tid == 0) { ADJ_STAMP(0, 1) }
      vjp_produce<M>(A, p, live, h, tmem + lane_off);
      fence_before();
      rows_sync();
      if (tid == 0) mbar_arrive(&S.full);
      if (tid == 0) { ADJ_STAMP(0, 2) }
      vjp_prefetch<M>(A, (int64_t)(tile + (int)gridDim.x) * kRows + r, cnt, h);
      const int q0 = kl * nchunk;
      for (int c = 0; c < nchunk; c++) {
        const int q = q0 + c, b = q & 1;
        mbar_wait(&S.g1[b], phase(q));  // Z / V of this chunk (Yb(q-2) had left the buffer)
        fence_after();
        if (tid == 0) { ADJ_STAMP(0, 3) }
        // ---- tanh, u = V (1 - tanh^2) -> TMEM (hi, lo); u^T, tanh^T
        {
          float z[16], v[16], uh[16], ul[16];
          tmem_ld16(tmem + 256 + 64 * b + 16 * h + lane_off, z);
          tmem_ld16(tmem + 256 + 64 * b + 32 + 16 * h + lane_off, v);
          const int c16 = (q % nchunk) * kHc + 16 * h;
#pragma unroll
          for (int j = 0; j < 16; j++) {
            const float a = tanhf(z[j] + S.b1[c16 + j]);
            const float uu = v[j] * (1.0f - a * a);
            uh[j] = tf32_hi(uu);
            ul[j] = uu - uh[j];
            if (live) {
              A.uT[blk(c16 + j, col, A.H)] = uu;
              A.AT[blk(c16 + j, col, A.H)] = a;
            }
          }
          // u hi / lo over this thread's own Z / V columns (read above)
          const uint32_t ub = tmem + 256 + 64 * b + 16 * h + lane_off;
          tmem_st16(ub, uh);
          tmem_st16(ub + 32, ul);
          tmem_wait_st();
        }
        fence_before();
        rows_sync();
        if (tid == 0) mbar_arrive(&S.epi[b]);
        if (tid == 0) { ADJ_STAMP(0, 4) }
      }
      // ---- this row's dL/dY_s (columns 32 h .. 32 h + 31)
      mbar_wait(&S.g2[(q0 + nchunk - 1) & 1], phase(q0 + nchunk - 1));
      fence_after();
      {
        float yb[32];
        tmem_ld32(accY + lane_off + 32 * h, yb);
        if (live) {
          float4* dst = reinterpret_cast<float4*>(A.Ybar + ((int64_t)A.stage * A.n + p) * kD + 32 * h);
#pragma unroll
          for (int e = 0; e < 8; e++)
            dst[e] = make_float4(yb[4 * e], yb[4 * e + 1], yb[4 * e + 2], yb[4 * e + 3]);
        }
      }
      fence_before();
      if (tid == 0) { ADJ_STAMP(0, 5) }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(S.tmem_base));
}

// --------------------------------------------- weight gradients (GEMM) ----

struct WgArgs {
  int H, S;
  int64_t pmax, ldt;
  const int32_t* count;
  const float *uT, *AT, *YT, *gT;
  float* part;  // (grid, kPartFloats)
};

// K-slices of 16 columns in two shared-memory stages: the operands of slice
// i+1 are converted into one stage while the MMAs of slice i read the other,
// and the global loads of slice i+2 are in flight in registers meanwhile.
constexpr int kWgK = 16;
struct WgStage {
  uint8_t au[2][2][128 * kWgK * 4];  // u^T halves [h][hi, lo]
  uint8_t ag[2][64 * kWgK * 4];      // g^T [hi, lo]
  uint8_t by[2][kN1 * kWgK * 4];     // [Y^T | 1] [hi, lo]
  uint8_t ba[2][2][kN2 * kWgK * 4];  // [tanh^T half | 1 (half 0)] [h][hi, lo]
};
struct WgSmem {
  WgStage st[2];
  uint64_t done[2];
  uint32_t tmem_base;
};

struct WgTile {
  const float* src;   // the matrix (blocked layout); set to the slice's block per fetch
  int nrows, ones;
  int64_t rows;       // the matrix's row count (block stride)
  int64_t row0;       // first row of this tile
  int off, lo_off;    // byte offsets of the hi and lo tiles inside a stage
};
template <int TROWS>
constexpr int wg_vec() { return (TROWS * (kWgK / 4) + 255) / 256; }

template <int TROWS>
__device__ __forceinline__ void wg_fetch(WgTile T, int64_t c0, int64_t cmax,
                                         float4 (&v)[wg_vec<TROWS>()]) {
  T.src += ((c0 >> 5) * T.rows + T.row0) * 32 + (c0 & 31);
#pragma unroll
  for (int q = 0; q < wg_vec<TROWS>(); q++) {
    const int e = threadIdx.x + 256 * q;
    const int r = e / (kWgK / 4), k4 = e % (kWgK / 4);
    float4 x = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (e < TROWS * (kWgK / 4)) {
      if (r < T.nrows)  // (src: this slice's half of a 32-column block, row-major)
        // (.L2::128B: the whole 128-byte block row comes into L2 -- this
        // CTA reads its other half in the next slice)
        asm volatile("ld.global.nc.L2::128B.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                     : "l"(T.src + (int64_t)r * 32 + 4 * k4));
      else if (r == T.ones)
        x = make_float4(1.0f, 1.0f, 1.0f, 1.0f);
    }
    v[q] = x;  // (columns >= cmax are zeroed at the store: nothing here waits on the load)
  }
}

// hi tile at st + off, lo tile one tile later
template <int TROWS>
__device__ __forceinline__ void wg_store(const WgTile& T, uint8_t* st, int64_t c0, int64_t cmax,
                                         const float4 (&v)[wg_vec<TROWS>()]) {
#pragma unroll
  for (int q = 0; q < wg_vec<TROWS>(); q++) {
    const int e = threadIdx.x + 256 * q;
    if (e < TROWS * (kWgK / 4)) {
      const int r = e / (kWgK / 4), k4 = e % (kWgK / 4);
      float4 x = v[q];
      const int64_t c = c0 + 4 * k4;
      if (c >= cmax) x.x = 0.0f;
      if (c + 1 >= cmax) x.y = 0.0f;
      if (c + 2 >= cmax) x.z = 0.0f;
      if (c + 3 >= cmax) x.w = 0.0f;
      float4 hi, lo;
      hi.x = tf32_hi(x.x), hi.y = tf32_hi(x.y), hi.z = tf32_hi(x.z), hi.w = tf32_hi(x.w);
      lo.x = x.x - hi.x, lo.y = x.y - hi.y, lo.z = x.z - hi.z, lo.w = x.w - hi.w;
      const uint32_t o = cm_off(r, 4 * k4, kWgK);
      *reinterpret_cast<float4*>(st + T.off + o) = hi;
      *reinterpret_cast<float4*>(st + T.lo_off + o) = lo;
    }
  }
}

// the operand tiles of one slice: u^T and [tanh^T | 1] per half of H,
// g^T, [Y^T | 1]; the second half is loaded only when H > 128
struct WgRegs {
  float4 u0[wg_vec<128>()], a0[wg_vec<kN2>()], u1[wg_vec<128>()], a1[wg_vec<128>()];
  float4 g[wg_vec<64>()], y[wg_vec<kN1>()];
};
struct WgTiles {
  WgTile u0, a0, u1, a1, g, y;
};
__device__ __forceinline__ void wg_fetch_all(const WgTiles& T, bool two, int64_t c0, int64_t cmax,
                                             WgRegs& R) {
  wg_fetch<128>(T.u0, c0, cmax, R.u0);
  wg_fetch<kN2>(T.a0, c0, cmax, R.a0);
  if (two) {
    wg_fetch<128>(T.u1, c0, cmax, R.u1);
    wg_fetch<128>(T.a1, c0, cmax, R.a1);
  }
  wg_fetch<64>(T.g, c0, cmax, R.g);
  wg_fetch<kN1>(T.y, c0, cmax, R.y);
}
__device__ __forceinline__ void wg_store_all(const WgTiles& T, bool two, uint8_t* st, int64_t c0,
                                             int64_t cmax, const WgRegs& R) {
  wg_store<128>(T.u0, st, c0, cmax, R.u0);
  wg_store<kN2>(T.a0, st, c0, cmax, R.a0);
  if (two) {
    wg_store<128>(T.u1, st, c0, cmax, R.u1);
    wg_store<128>(T.a1, st, c0, cmax, R.a1);
  }
  wg_store<64>(T.g, st, c0, cmax, R.g);
  wg_store<kN1>(T.y, st, c0, cmax, R.y);
}

__global__ void __launch_bounds__(256, 1) wg_kernel(const WgArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  WgSmem& S = *reinterpret_cast<WgSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int cnt = *A.count;
  const int per_stage = (cnt + kWgK - 1) / kWgK;
  const int nslices = A.S * per_stage;
  // this CTA's slices: a contiguous range (consecutive slices are the two
  // halves of one 32-column block)
  const int per_cta = (nslices + (int)gridDim.x - 1) / (int)gridDim.x;
  const int first = (int)blockIdx.x * per_cta;
  const int last = first + per_cta < nslices ? first + per_cta : nslices;
  if (first >= nslices) return;
  const int halves = A.H > 128 ? 2 : 1;
  if (tid == 0) {
    mbar_init(&S.done[0], 1);
    mbar_init(&S.done[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&S.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = S.tmem_base;
  const int rows0 = A.H < 128 ? A.H : 128, rows1 = A.H - rows0;
  const bool two = halves == 2;
  const WgStage& s0 = S.st[0];
  auto off = [&](const void* p) { return (int)((const uint8_t*)p - (const uint8_t*)&s0); };
  const WgTiles T{WgTile{A.uT, rows0, -1, A.H, 0, off(s0.au[0][0]), off(s0.au[0][1])},
                  WgTile{A.AT, rows0, 128, A.H, 0, off(s0.ba[0][0]), off(s0.ba[0][1])},
                  WgTile{A.uT, rows1, -1, A.H, 128, off(s0.au[1][0]), off(s0.au[1][1])},
                  WgTile{A.AT, rows1, -1, A.H, 128, off(s0.ba[1][0]), off(s0.ba[1][1])},
                  WgTile{A.gT, kD, -1, kD, 0, off(s0.ag[0]), off(s0.ag[1])},
                  WgTile{A.YT, kD, kD, kD, 0, off(s0.by[0]), off(s0.by[1])}};
  auto slice_cols = [&](int sl, int64_t& c0, int64_t& cmax) {
    const int s = sl / per_stage;
    c0 = (int64_t)s * A.pmax + (int64_t)(sl % per_stage) * kWgK;
    cmax = (int64_t)s * A.pmax + cnt;
  };
  // TMEM: dW1|db1 half h at columns 80 h (M = 128: row = hidden unit);
  // dW2|db2 at columns 160 (M = 64: row = output; half 0 in lanes 0-15,
  // half 1 in lanes 16-31 of each quadrant)
  // slice i of this CTA = blockIdx.x + i * gridDim.x; the loads of slices
  // i+1 and i+2 are in flight (two register sets) while slice i is stored
  auto fetch = [&](int i, WgRegs& R) {
    const int sl = first + i;
    if (sl >= last) return;
    int64_t c0, cmax;
    slice_cols(sl, c0, cmax);
    wg_fetch_all(T, two, c0, cmax, R);
  };
  auto step = [&](int i, WgRegs& R) {
    const int b = i & 1;
    if (i >= 2) mbar_wait(&S.done[b], ((i - 2) >> 1) & 1);  // MMAs of slice i-2 read stage b
    uint8_t* st = reinterpret_cast<uint8_t*>(&S.st[b]);
    int64_t c0, cmax;
    slice_cols(first + i, c0, cmax);
    wg_store_all(T, two, st, c0, cmax, R);
    fence_async_smem();
    fence_before();
    __syncthreads();
    if (warp == 0) {  // warp-uniform operands, one elected lane issues
      const WgStage& g = S.st[b];
      uint64_t au[2][2], ba[2][2], ag[2], by[2];
#pragma unroll
      for (int t = 0; t < 2; t++) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          au[h][t] = smem_desc(smem_u32(g.au[h][t]), 512);
          ba[h][t] = smem_desc(smem_u32(g.ba[h][t]), 512);
        }
        ag[t] = smem_desc(smem_u32(g.ag[t]), 512);
        by[t] = smem_desc(smem_u32(g.by[t]), 512);
      }
      if (elect_one()) {
        fence_after();
        const int ta[3] = {0, 0, 1}, tb[3] = {0, 1, 0};
#pragma unroll
        for (int ks = 0; ks < kWgK / 8; ks++)
#pragma unroll
          for (int term = 0; term < 3; term++) {
            const uint32_t acc = (i | ks | term) ? 1u : 0u;
#pragma unroll
            for (int h = 0; h < 2; h++) {
              if (h >= halves) break;
              mma_tf32(tmem + kN1 * h, au[h][ta[term]] + 16 * ks, by[tb[term]] + 16 * ks,
                       idesc_mn(128, kN1), acc);
              mma_tf32(tmem + 2 * kN1 + (h ? (16u << 16) : 0u), ag[ta[term]] + 16 * ks,
                       ba[h][tb[term]] + 16 * ks, idesc_mn(64, h ? 128 : kN2), acc);
            }
          }
        mma_commit(&S.done[b]);
      }
      __syncwarp();
    }
    fetch(i + 2, R);  // (the register set just stored)
  };
  const int mine = last - first;
  WgRegs R0, R1;
  fetch(0, R0);
  fetch(1, R1);
  int i = 0;
  while (i < mine) {
    step(i++, R0);
    if (i >= mine) break;
    step(i++, R1);
  }
  if (i >= 1) mbar_wait(&S.done[(i - 1) & 1], ((i - 1) >> 1) & 1);  // the last slice's MMAs
  fence_after();
  // add this CTA's sums to its partial (the same CTA index every iteration:
  // a fixed summation order), 16 columns per batch of loads
  if (warp < 4) {
    float* part = A.part + (size_t)blockIdx.x * kPartFloats;
    const uint32_t lo = (uint32_t)(warp * 32) << 16;
    const int l = tid & 31;
    auto add16 = [&](float* dst, uint32_t taddr, int width) {
      float v[16];
      tmem_ld16(taddr, v);
      float4* d4 = reinterpret_cast<float4*>(dst);
      float4 cur[4];
#pragma unroll
      for (int e = 0; e < 4; e++) cur[e] = d4[e];
#pragma unroll
      for (int e = 0; e < 4; e++) {
        if (4 * e < width) {
          cur[e].x += v[4 * e], cur[e].y += v[4 * e + 1], cur[e].z += v[4 * e + 2], cur[e].w += v[4 * e + 3];
          d4[e] = cur[e];
        }
      }
    };
    for (int h = 0; h < halves; h++) {
      float* dst = part + (size_t)h * 128 * kN1 + (size_t)tid * kN1;  // row = hidden 128 h + tid
      for (int c = 0; c < kN1; c += 16) add16(dst + c, tmem + kN1 * h + lo + c, 16);
    }
    // M = 64 accumulators: lane l < 16 of quadrant w holds output 16 w + l
    // of half 0, lane 16 + l the same output of half 1
    const int hh = l >> 4, o = 16 * warp + (l & 15);
    const int width = hh ? 128 : kN2;
    float* dst = part + (size_t)2 * 128 * kN1 + ((size_t)hh * 64 + o) * kN2;
    for (int c = 0; c < kN2; c += 16) {
      const int w = hh < halves ? (width - c < 16 ? width - c : 16) : 0;
      add16(dst + c, tmem + 2 * kN1 + lo + c, w);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// partials -> gW1 (H, 64), gb1 (H), gW2 (64, H), gb2 (64); fixed order
__global__ void wg_reduce_kernel(const float* part, int parts, int H, float* gW1, float* gb1,
                                 float* gW2, float* gb2) {
  const int total = H * kD + H + kD * H + kD;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    size_t off;
    if (e < H * kD) {
      const int j = e / kD, c = e % kD;
      off = (size_t)(j >> 7) * 128 * kN1 + (size_t)(j & 127) * kN1 + c;
    } else if (e < H * kD + H) {
      const int j = e - H * kD;
      off = (size_t)(j >> 7) * 128 * kN1 + (size_t)(j & 127) * kN1 + kD;
    } else if (e < 2 * H * kD + H) {
      const int r = e - H * kD - H, o = r / H, j = r % H;
      off = (size_t)2 * 128 * kN1 + ((size_t)(j >> 7) * 64 + o) * kN2 + (j & 127);
    } else {
      const int o = e - 2 * H * kD - H;
      off = (size_t)2 * 128 * kN1 + (size_t)o * kN2 + 128;
    }
    double s = 0.0;
    for (int b = 0; b < parts; b++) s += (double)part[(size_t)b * kPartFloats + off];
    const float v = (float)s;
    if (e < H * kD) {
      if (gW1) gW1[e] = v;
    } else if (e < H * kD + H) {
      if (gb1) gb1[e - H * kD] = v;
    } else if (e < 2 * H * kD + H) {
      if (gW2) gW2[e - H * kD - H] = v;
    } else if (gb2) {
      gb2[e - 2 * H * kD - H] = v;
    }
  }
}

// ------------------------------------------------------------ workspace ----

struct Layout {
  size_t total = 0;
  size_t keys_in, keys, idx_in, order, cub, cub_bytes, count, hi, lo, t_old, h, y, kb, rec, yb, Ybar,
      uT, AT, YT, gT, wfwd, wadj, w1t, w2t, part;
  Layout(int64_t n, int64_t H, int S, int parts) {
    auto take = [&](size_t bytes) {
      const size_t o = total;
      total += (bytes + 255) & ~(size_t)255;
      return o;
    };
    const int64_t pmax = (n + 127) / 128 * 128;
    cub_bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, cub_bytes, (const int32_t*)nullptr,
                                              (int32_t*)nullptr, (const int32_t*)nullptr,
                                              (int32_t*)nullptr, (int)n);
    keys_in = take(4 * n), keys = take(4 * n), idx_in = take(4 * n), order = take(4 * n);
    cub = take(cub_bytes), count = take(8);
    hi = take(8 * n), lo = take(8 * n), t_old = take(8 * n), h = take(8 * n);
    y = take(8 * n * kD), kb = take(8 * (size_t)S * n * kD), rec = take(8 * n);
    Ybar = take(4 * (size_t)S * n * kD);
    yb = take(8 * n * kD);
    uT = take(4 * (size_t)H * S * pmax), AT = take(4 * (size_t)H * S * pmax);
    YT = take(4 * (size_t)kD * S * pmax), gT = take(4 * (size_t)kD * S * pmax);
    wfwd = take(mlp_tc_prep_bytes(H)), wadj = take(mlp_tc_prep_bytes(H));
    w1t = take(4 * H * kD), w2t = take(4 * H * kD);
    part = take(4 * (size_t)parts * kPartFloats);
  }
};

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int M>
cudaError_t run(AdjParams A, char* ws, cudaStream_t st, int64_t* launches) {
  constexpr int S = Tab<M>::S;
  if (!A.traj_stages) return cudaErrorInvalidValue;  // (bode_abi.cu reports it)
  const int64_t n = A.n, H = A.H;
  const int sms = sm_count();
  const Layout L(n, H, S, sms);
  const int64_t pmax = (n + 127) / 128 * 128;
  auto at = [&](size_t o) { return ws + o; };
  RowState R;
  R.n = n;
  R.pmax = pmax;
  R.order = (const int32_t*)at(L.order);
  R.nrec = (const int32_t*)at(L.keys);
  R.count = (int32_t*)at(L.count);
  R.hi = (int64_t*)at(L.hi);
  R.lo = (int64_t*)at(L.lo);
  R.t_old = (double*)at(L.t_old);
  R.h = (double*)at(L.h);
  R.y = (double*)at(L.y);
  R.kb = (double*)at(L.kb);
  R.yb = (double*)at(L.yb);
  R.rec = (int64_t*)at(L.rec);
  float* wfwd = (float*)at(L.wfwd);
  float* wadj = (float*)at(L.wadj);
  cudaError_t e;
  int64_t nl = 0;
  const unsigned gb = (unsigned)((n * kD + 255) / 256 < sms * 16 ? (n * kD + 255) / 256 : sms * 16);
  // weights: the forward's pre-split chunks and the adjoint's (W2^T | W1^T)
  transpose_kernel<<<sms, 256, 0, st>>>(A.W1, (int)H, kD, (float*)at(L.w1t));  // (64, H)
  transpose_kernel<<<sms, 256, 0, st>>>(A.W2, kD, (int)H, (float*)at(L.w2t));  // (H, 64)
  if ((e = mlp_tc_prep(A.W1, A.W2, H, wfwd, st)) != cudaSuccess) return e;
  if ((e = mlp_tc_prep((float*)at(L.w2t), (float*)at(L.w1t), H, wadj, st)) != cudaSuccess) return e;
  nl += 4;
  // rows longest trajectory first (stable: ties by index)
  keys_kernel<<<gb, 256, 0, st>>>(A.traj_offsets, n, (int32_t*)at(L.keys_in), (int32_t*)at(L.idx_in));
  size_t cb = L.cub_bytes;
  e = cub::DeviceRadixSort::SortPairsDescending(at(L.cub), cb, (const int32_t*)at(L.keys_in),
                                                (int32_t*)at(L.keys), (const int32_t*)at(L.idx_in),
                                                (int32_t*)at(L.order), (int)n, 0, 32, st);
  if (e != cudaSuccess) return e;
  nl += 1 + 4;  // keys + the radix sort passes (approximate)
  int32_t maxn = 0;
  if ((e = cudaMemcpyAsync(&maxn, at(L.keys), 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  init_kernel<<<gb, 256, 0, st>>>(R, A.n_emitted);
  if ((e = cudaMemsetAsync(at(L.part), 0, 4 * (size_t)sms * kPartFloats, st)) != cudaSuccess) return e;
  nl += 1;

  static bool attr = false;
  const size_t vjp_smem = sizeof(VjpSmem) + 1024, wg_smem = sizeof(WgSmem) + 1024;
  if (!attr) {
    if ((e = cudaFuncSetAttribute(vjp_kernel<BODE_METHOD_DOPRI5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vjp_smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(vjp_kernel<BODE_METHOD_TSIT5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vjp_smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(vjp_kernel<BODE_METHOD_HEUN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vjp_smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(wg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wg_smem)) != cudaSuccess) return e;
    attr = true;
  }
  const int max_tiles = (int)((n + kRows - 1) / kRows);
  const int grid = max_tiles < sms ? max_tiles : sms;
  VjpArgs V{n, pmax, (int)H, 0, R.count, R.y, A.traj_stages, R.rec, R.h, R.kb, (float*)at(L.Ybar), wfwd, wadj, A.b1,
            (float*)at(L.uT), (float*)at(L.AT), (float*)at(L.YT), (float*)at(L.gT)};
  WgArgs G{(int)H, S, pmax, (int64_t)S * pmax, R.count, V.uT, V.AT, V.YT, V.gT, (float*)at(L.part)};
  for (int64_t it = 0; it < maxn; it++) {
    count_kernel<<<1, 1, 0, st>>>(R, it);
    load_kernel<<<gb, 256, 0, st>>>(R, A.traj, A.traj_offsets, it);
    seeds_kernel<M><<<gb, 256, 0, st>>>(R, A.t_eval, A.t_eval_offsets, A.t_eval_len, A.grad_ys);
    for (int s = S - 1; s >= 0; s--) {
      V.stage = s;
      vjp_kernel<M><<<grid, kVjpThreads, vjp_smem, st>>>(V);
    }
    fold_kernel<M><<<gb, 256, 0, st>>>(R, (const float*)at(L.Ybar));
    wg_kernel<<<sms, 256, wg_smem, st>>>(G);
    nl += 5 + S;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  finish_kernel<<<gb, 256, 0, st>>>(R, A.grad_ys, A.t_eval_offsets, A.t_eval_len, A.grad_y0);
  wg_reduce_kernel<<<64, 256, 0, st>>>((const float*)at(L.part), sms, (int)H, A.gW1, A.gb1, A.gW2, A.gb2);
  nl += 2;
  *launches += nl;
  return cudaGetLastError();
}

}  // namespace adjtc

#ifdef BODE_ADJ_PROF
extern "C" int bode_debug_adj_prof(long long* out) {
  cudaMemcpyFromSymbol(out, adjtc::g_adj_prof, sizeof(adjtc::g_adj_prof));
  int n[2];
  cudaMemcpyFromSymbol(n, adjtc::g_adj_prof_n, sizeof(n));
  return n[0] * 1000 + n[1];
}
#endif

bool mlp_adjoint_tc_supported(int64_t d, int64_t H) {
  return d == tc::kD && H % tc::kHc == 0 && H >= 32 && H <= 256;
}

size_t mlp_adjoint_tc_bytes(int64_t n, int64_t H, int method) {
  const int S = method == BODE_METHOD_HEUN ? Tab<BODE_METHOD_HEUN>::S
              : method == BODE_METHOD_TSIT5 ? Tab<BODE_METHOD_TSIT5>::S
                                            : Tab<BODE_METHOD_DOPRI5>::S;
  return adjtc::Layout(n, H, S, adjtc::sm_count()).total;
}

cudaError_t mlp_adjoint_tc_run(int method, AdjParams A, void* ws, cudaStream_t st, int64_t* launches) {
  switch (method) {
    case BODE_METHOD_DOPRI5: return adjtc::run<BODE_METHOD_DOPRI5>(A, (char*)ws, st, launches);
    case BODE_METHOD_TSIT5: return adjtc::run<BODE_METHOD_TSIT5>(A, (char*)ws, st, launches);
    default: return adjtc::run<BODE_METHOD_HEUN>(A, (char*)ws, st, launches);
  }
}

}  // namespace bode
