// bode_mlp_fused.cu -- the neural-ODE solve as ONE persistent tcgen05 kernel.
//
// Each CTA (one per SM) owns a tile of 128 instances -- one per TMEM lane --
// and runs the reference's whole per-instance loop (solver.py:208-322) for
// them: stage inputs, the stage MLPs on the tensor cores, y_next / err, the
// NumPy-order RMS norm, the PID update, accept/reject, dense output,
// statuses.  When an instance terminates its row is refilled from a global
// queue, so there is no lockstep iteration, no per-stage launch and no host
// round trip; the lockstep path (bode_mlp.cu + bode_mlp_tc.cu) launches 9
// kernels per iteration and re-reads every stage vector from HBM per stage.
//
// TMEM (512 columns x 128 lanes, fp32):
//   columns 64 s .. 64 s + 63   stage derivative k_s of every row (s < 7)
//   columns 448 .. 511          two 32-column GEMM1 chunk accumulators
// Shared memory (~226 KB): y (fp64, [column][row]), the stage-input tile Y_s
// as TF32 hi/lo core matrices (reused as the y_next buffer by the control
// step), one hidden chunk H_c hi/lo, a 4-slot ring of 16 KB weight chunks
// streamed with cp.async.bulk.
//
// Warp roles (288 threads):
//   warps 0-3 (WG0)  row owners: refill, control; plus half of every stage
//                    input and of every tanh epilogue (columns 0-31 / 0-15)
//   warps 4-7 (WG1)  the other half of the stage inputs and epilogues
//   warp 8           one elected thread issues every MMA and weight copy
// Per stage s and hidden chunk c (3xTF32: hi*hi + hi*lo + lo*hi, fp32 acc):
//   GEMM1  acc1[c&1] = Y_s W1_c^T        (M=128, N=32, K=64: 24 MMAs)
//   epi    H_c = tanh(acc1 + b1) -> hi/lo (both groups, 16 columns each)
//   GEMM2  k_s += H_c W2_c^T             (M=128, N=64, K=32: 12 MMAs)
// GEMM1 of chunk c+2 is issued as soon as the epilogue of chunk c released
// its accumulator, so the tensor core works while the epilogue runs.  The
// MMA sequence (order of chunks, K steps and hi/lo terms) is the lockstep
// tensor-core path's, so stage values are bit-identical to it; the fp64
// stage combination, control and dense output replay the reference order.
#include <cuda_runtime.h>

#include <type_traits>

#include "bode_mlp.cuh"
#include "bode_tc.cuh"

namespace bode {
namespace fused {
using namespace tc;

// -DBODE_FUSED_PROF: per-CTA cycle counters of each phase (debug builds)
#ifdef BODE_FUSED_PROF
#define PROF_DECL unsigned long long pf[32] = {0}; long long pt = clock64();
#define PROF_MARK(k) { const long long now = clock64(); pf[k] += now - pt; pt = now; }
#else
#define PROF_DECL
#define PROF_MARK(k)
#endif

constexpr int kNS = 4;            // weight ring slots
constexpr int kWItem = 2 * kW1;   // one W1 or W2 chunk, hi | lo (16 KB)
constexpr int kThreads = 320;
constexpr int kMaxChunks = 8;     // H <= 256 (TMEM: 7 x 64 stage columns + 64)
constexpr int kItemsMax = 16;     // weight items per stage (H / 16)

// GEMM1 unit width of stage s: stage vectors k_0..k_s occupy TMEM columns
// [0, 64 (s+1)); the two GEMM1 accumulators take the top 2 W columns, and a
// wider unit means fewer, more efficient MMAs (measured on B200: a
// kind::tf32 M=128 MMA costs 46 / 54 / 66 cycles at N = 32 / 64 / 128 --
// smem operand bandwidth -- for 1x / 2x / 4x the work).
//
// Where 64 more columns fit, the tanh outputs H_c (GEMM2's A operand, TF32
// hi/lo for each group's 16 columns) are kept in TMEM as well
// (tcgen05.mma with A in tensor memory): GEMM2 then reads only the weights
// from shared memory, and the H stores never touch it.  For dopri5/tsit5
// that holds for stages 1-5 (widths 128, 128, 64, 64, 32); stage 6 keeps H in
// shared memory.
__host__ __device__ __forceinline__ bool h_in_tmem(int s, int H, int* width) {
  const int used = 64 * (s + 1);
  for (int w = 128; w >= 32; w >>= 1)
    if (H % w == 0 && used + 2 * w + 64 <= 512) {
      *width = w;
      return true;
    }
  const int free_cols = 512 - used;
  *width = (free_cols >= 256 && H % 128 == 0) ? 128 : (free_cols >= 128 && H % 64 == 0) ? 64 : 32;
  return false;
}
__host__ __device__ __forceinline__ int unit_width(int s, int H) {
  int w;
  h_in_tmem(s, H, &w);
  return w;
}

struct Smem {
  double ys[kD][kRows];       // 64 KB  state y, [column][row]
  uint8_t a[2][kATile];       // 64 KB  Y_s hi, lo  |  y_next (fp64 [column][row])
  uint8_t h[2][2][kHTile / 2]; // 32 KB  [group][hi, lo] 16-column halves of H_c
  uint8_t w[kNS][kWItem];     // 64 KB  weight ring
  float b2[kD];
  double hs[kRows];           // dt_used of the pending attempt, per row
  int32_t act[kRows];         // row holds an instance
  int32_t ridx[kRows];        // instance just loaded into the row (-1: none)
  uint32_t seq[7][kItemsMax];  // weight item byte offsets, per stage, in consumption order
  uint64_t a_full, epidone[2], g1done[2], g2done[2], stage_done, wfull[kNS], wempty[kNS];
  uint32_t tmem_base;
};

__device__ __forceinline__ void store_hilo(uint8_t* hi_base, uint8_t* lo_base, uint32_t off,
                                           const float* x) {
  float4 hi, lo;
  hi.x = tf32_hi(x[0]), hi.y = tf32_hi(x[1]), hi.z = tf32_hi(x[2]), hi.w = tf32_hi(x[3]);
  lo.x = x[0] - hi.x, lo.y = x[1] - hi.y, lo.z = x[2] - hi.z, lo.w = x[3] - hi.w;
  *reinterpret_cast<float4*>(hi_base + off) = hi;
  *reinterpret_cast<float4*>(lo_base + off) = lo;
}

// FAST (bode_solve_args.mode == BODE_MODE_FAST): the fp64 stage
// combinations, error estimate and dense output fuse where written
// (FastOps), the error ratio multiplies by a reciprocal, and an I / PI
// controller runs on the squared norm with one exp (adapt_pi_ms) -- the
// analytic kernels' fast mode; the hidden activation is tanh_fast (ex2 / rcp,
// absolute error ~2e-7) instead of libdevice tanhf.  The MLP itself is fp32
// either way, so its
// stage values already differ from the reference at fp32-ulp level; the
// MLP parity bar (aggregate step counts 2%, y(T) 1e-4) holds for both.
template <int M, bool FAST>
__global__ void __launch_bounds__(kThreads, 1) mlp_fused_kernel(const MlpFusedArgs A) {
  using T = Tab<M>;
  using O = typename std::conditional<FAST, FastOps, ExactOps>::type;
  constexpr int S = T::S;
  constexpr int S0 = T::FSAL ? 1 : 0;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wg = warp >> 2;                 // 0, 1: row groups; 2: MMA warp
  const int row = (warp & 3) * 32 + lane;   // tile row == TMEM lane (groups 0, 1)
  const int nc = A.H / kHc;

  if (tid == 0) {
    mbar_init(&sm.a_full, 256);
    mbar_init(&sm.epidone[0], 128);
    mbar_init(&sm.epidone[1], 128);
    mbar_init(&sm.g1done[0], 1);
    mbar_init(&sm.g1done[1], 1);
    mbar_init(&sm.g2done[0], 1);
    mbar_init(&sm.g2done[1], 1);
    mbar_init(&sm.stage_done, 1);
    for (int q = 0; q < kNS; q++) {
      mbar_init(&sm.wfull[q], 1);
      mbar_init(&sm.wempty[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // weight items in the order the MMA thread consumes them in stage s:
    // the K slices of GEMM1 units 0 and 1, then per 32-column hidden chunk q
    // the W2 chunk of q and, after a unit's last chunk, unit u+2's slices
    for (int st = S0; st < S; st++) {
      const int Wd = unit_width(st, A.H), nu = A.H / Wd, spu = Wd / kHc;
      int p = 0;
      auto g1items = [&](int u) {
        for (int q = 0; q < spu; q++)  // spu K slices of 16 KB per unit
          sm.seq[st][p++] = Wd == kHc ? (uint32_t)(u * kWChunk)
                                      : (uint32_t)(mlp_w1_items_offset(A.H, Wd) + (size_t)(u * spu + q) * 16384);
      };
      g1items(0);
      if (nu > 1) g1items(1);
      for (int q = 0; q < nc; q++) {
        sm.seq[st][p++] = (uint32_t)(q * kWChunk + 2 * kW1);
        if (q % spu == spu - 1 && q / spu + 2 < nu) g1items(q / spu + 2);
      }
    }
  }
  for (int e = tid; e < kD; e += kThreads) sm.b2[e] = A.b2[e];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t lrow = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's lanes
  const int count = *A.count;
  const bool b1_vec = (reinterpret_cast<unsigned long long>(A.b1) & 15) == 0;

  // ---- row state (WG0 threads)
  bool have = false;
  int64_t idx = 0, nsteps = 0, nacc = 0, cursor = 0, m = 0;
  int64_t trow = 0, tlen = 0;  // (gradients) this row's trajectory rows
  double t = 0.0, dt = 0.0, t_end = 0.0, atol = 0.0, rtol = 0.0, n1 = 1.0, n2 = 1.0, h = 0.0;
  LogCache L1{0.0, 0.0, true};  // (FAST I / PI) log of the previous norm: log(1) = 0
  bool trunc = false;
  const double* te = nullptr;
  double* yout = nullptr;
  unsigned long long my_max = 0;
  // ---- barrier phases
  uint32_t ph_afull = 0, ph_epi = 0, ph_sd = 0, ph_g1[2] = {0u, 0u};
  uint32_t g2_base = 0;            // G2 completions before the current stage
  uint32_t wq_load = 0, wq_use = 0;  // MMA thread: weight items issued / consumed
  const unsigned lt_mask = (1u << lane) - 1u;
  PROF_DECL

  while (true) {
    // ================= refill free rows (WG0 takes instances from the queue;
    // both row groups keep identical copies of the row state)
    auto load_row = [&](int64_t i) {
      idx = i;
      t = A.t[i];
      dt = A.dt[i];
      t_end = A.t_end[i];
      atol = A.atol_v ? A.atol_v[i] : A.atol;
      rtol = A.rtol_v ? A.rtol_v[i] : A.rtol;
      cursor = A.n_emitted[i];
      if (A.t_eval_offsets) {
        const int64_t o = A.t_eval_offsets[i];
        te = A.t_eval + o;
        m = A.t_eval_offsets[i + 1] - o;
        yout = A.ys ? A.ys + o * kD : nullptr;
      } else {
        te = A.t_eval;
        m = A.t_eval_len;
        yout = A.ys ? A.ys + i * A.t_eval_len * kD : nullptr;
      }
      n1 = 1.0;
      n2 = 1.0;
      L1 = LogCache{0.0, 0.0, true};
      nsteps = 0;
      nacc = 0;
      if (A.traj_y) {
        trow = A.traj_offsets[i];
        tlen = A.traj_offsets[i + 1] - trow;
      }
      have = true;
    };
    if (wg == 0) {
      const unsigned need = __ballot_sync(0xffffffffu, !have);
      bool got = false;
      int32_t rid = -1;
      if (need) {
        const int leader = __ffs(need) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(A.queue, (unsigned long long)__popc(need));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (!have) {
          const unsigned long long pos = base + __popc(need & lt_mask);
          if (pos < (unsigned long long)count) {
            const int64_t i = A.act[pos];
            rid = (int32_t)i;
            load_row(i);
            const double2* yp = reinterpret_cast<const double2*>(A.y + i * kD);
#pragma unroll 8
            for (int c = 0; c < kD / 2; c++) {
              const double2 v = yp[c];
              sm.ys[2 * c][row] = v.x;
              sm.ys[2 * c + 1][row] = v.y;
            }
            got = true;
          }
        }
      }
      sm.ridx[row] = rid;
      if (T::FSAL && __any_sync(0xffffffffu, got)) {  // k_0 = f0 of refilled rows
#pragma unroll
        for (int ch = 0; ch < 4; ch++) {
          float v[16];
          tmem_ld16(lrow + 16 * ch, v);
          if (got) {
            const float4* fp = reinterpret_cast<const float4*>(A.f0 + idx * kD + 16 * ch);
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const float4 f = fp[q];
              v[4 * q] = f.x, v[4 * q + 1] = f.y, v[4 * q + 2] = f.z, v[4 * q + 3] = f.w;
            }
          }
          tmem_st16(lrow + 16 * ch, v);
        }
        tmem_wait_st();
      }
      if (have) {
        const double rem = ExactOps::sub(t_end, t);
        trunc = fabs(dt) >= fabs(rem);
        h = trunc ? rem : dt;
      }
      sm.hs[row] = h;
      sm.act[row] = have;
    }
    PROF_MARK(0)
    fence_before();
    const int any = __syncthreads_or(wg == 0 && have);
    fence_after();
    PROF_MARK(1)
    if (!any) break;
    if (wg == 1) {  // mirror WG0's row state
      const int32_t rid = sm.ridx[row];
      if (rid >= 0) load_row(rid);
      if (have) {
        const double rem = ExactOps::sub(t_end, t);
        trunc = fabs(dt) >= fabs(rem);
        h = trunc ? rem : dt;
      }
    }

    for (int s = S0; s < S; s++) {
      if (wg < 2) {
        // ============ stage input Y_s = y + h sum_{j<s} a_sj k_j (my 32 columns)
        {
          const bool live = sm.act[row] != 0;
          const double hr = sm.hs[row];
#pragma unroll
          for (int ch = 0; ch < 2; ch++) {
            const int c0 = 32 * wg + 16 * ch;
            double acc[16];
#pragma unroll
            for (int e = 0; e < 16; e++) acc[e] = 0.0;
#pragma unroll
            for (int j = 0; j < S - 1; j++) {
              if (j >= s) break;
              float kv[16];
              tmem_ld16(lrow + 64 * j + c0, kv);
              const double aj = T::a(s, j);
#pragma unroll
              for (int e = 0; e < 16; e++)
                acc[e] = j == 0 ? O::mul(aj, (double)kv[e])
                                : O::mad(aj, (double)kv[e], acc[e]);
            }
            float x[16];
#pragma unroll
            for (int e = 0; e < 16; e++) {
              const double y = sm.ys[c0 + e][row];
              x[e] = live ? (float)(s > 0 ? O::mad(hr, acc[e], y) : y) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < 4; q++)
              store_hilo(sm.a[0], sm.a[1], cm_off(row, c0 + 4 * q, kD), x + 4 * q);
            // gradients: this attempt's stage input into the row of the step
            // being tried (a rejected attempt is overwritten by the next one)
            if (A.traj_y && live && nacc < tlen) {
              float4* dst = reinterpret_cast<float4*>(A.traj_y + ((trow + nacc) * S + s) * kD + c0);
#pragma unroll
              for (int q = 0; q < 4; q++)
                dst[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
            }
          }
        }
        fence_async_smem();
        mbar_arrive(&sm.a_full);
        PROF_MARK(2)
        // ============ tanh epilogues of the hidden chunks
        int Wd;
        const bool htm = h_in_tmem(s, A.H, &Wd);
        const int spu = Wd / kHc, lspu = 31 - __clz(spu);  // (a power of two: shifts, not divisions)
        const uint32_t acc1_base = 512 - 2 * Wd, h_base = acc1_base - 64;
        for (int c = 0; c < nc; c++) {
          const int u = c >> lspu, b = u & 1;
          if ((c & (spu - 1)) == 0) {
            mbar_wait(&sm.g1done[b], ph_g1[b]);
            ph_g1[b] ^= 1;
            fence_after();
          }
          PROF_MARK(3)
          float v[16];
          tmem_ld16(lrow + acc1_base + Wd * b + 32 * (c & (spu - 1)) + 16 * wg, v);
          const float* b1 = A.b1 + c * kHc + 16 * wg;
          float bb[16];
          if (b1_vec) {
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const float4 t4 = __ldg(reinterpret_cast<const float4*>(b1) + q);
              bb[4 * q] = t4.x, bb[4 * q + 1] = t4.y, bb[4 * q + 2] = t4.z, bb[4 * q + 3] = t4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; j++) bb[j] = __ldg(b1 + j);
          }
#pragma unroll
          for (int j = 0; j < 16; j++) v[j] = FAST ? tanh_fast(v[j] + bb[j]) : tanhf(v[j] + bb[j]);
          PROF_MARK(4)
          if (c > 0) {  // GEMM2 of chunk c-1 has finished reading H
            mbar_wait(&sm.g2done[wg], (g2_base + c - 1) & 1);
          }
          PROF_MARK(5)
          if (htm) {  // TF32 hi/lo into this group's TMEM columns (A of GEMM2)
            float hi[16], lo[16];
#pragma unroll
            for (int j = 0; j < 16; j++) {
              hi[j] = tf32_hi(v[j]);
              lo[j] = v[j] - hi[j];
            }
            tmem_st16(lrow + h_base + 32 * wg, hi);
            tmem_st16(lrow + h_base + 32 * wg + 16, lo);
            tmem_wait_st();
          } else {
#pragma unroll
            for (int q = 0; q < 4; q++)
              store_hilo(sm.h[wg][0], sm.h[wg][1], cm_off(row, 4 * q, 16), v + 4 * q);
            fence_async_smem();
          }
          fence_before();
          mbar_arrive(&sm.epidone[wg]);
          PROF_MARK(6)
        }
        mbar_wait(&sm.stage_done, ph_sd);
        ph_sd ^= 1;
        // the last chunk's GEMM2 completion (already complete once stage_done
        // is: tcgen05.commit tracks every earlier MMA) is consumed here, so
        // every g2done phase has a waiter
        mbar_wait(&sm.g2done[wg], (g2_base + nc - 1) & 1);
        g2_base += nc;
        fence_after();
        PROF_MARK(7)
        // ============ k_s = acc + b2 (the reference adds b2 after the sum)
#pragma unroll
        for (int hf = 0; hf < 2; hf++) {
          const int c0 = 32 * wg + 16 * hf;
          float v[16];
          tmem_ld16(lrow + 64 * s + c0, v);
#pragma unroll
          for (int j = 0; j < 16; j++) v[j] += sm.b2[c0 + j];
          tmem_st16(lrow + 64 * s + c0, v);
        }
        tmem_wait_st();
        PROF_MARK(8)
      } else if (warp == 8) {
        // ============ MMA issue.  The whole warp runs this code so descriptors
        // and TMEM addresses stay in uniform registers; one elected lane
        // issues each MMA / commit.  Weights arrive from the loader warp.
        auto next_w = [&]() -> uint32_t {
          const uint32_t sl = wq_use % kNS;
          PROF_MARK(20)
          mbar_wait(&sm.wfull[sl], (wq_use / kNS) & 1);
          PROF_MARK(18)
          wq_use++;
          return sl;
        };
        // descriptor of K step k = descriptor of the tile + 16 k (256 B >> 4)
        const uint64_t dA_hi = smem_desc(smem_u32(sm.a[0]), 2048);
        const uint64_t dA_lo = smem_desc(smem_u32(sm.a[1]), 2048);
        const uint64_t dW2 = smem_desc(smem_u32(sm.w[0]), 1024);
        int Wd;
        const bool htm = h_in_tmem(s, A.H, &Wd);
        const int spu = Wd / kHc, nu = A.H / Wd, lspu = 31 - __clz(spu);
        const int KS = 2048 / Wd;                     // K per 16 KB item
        const uint32_t acc1_base = 512 - 2 * Wd, h_base = acc1_base - 64;
        // GEMM1 unit u: acc1[u&1] (N = Wd) = Y_s W1[u Wd .. u Wd + Wd)^T,
        // K-step major, the three 3xTF32 products inner
        auto gemm1 = [&](int u) {
          const uint32_t acc = tmem + acc1_base + Wd * (u & 1);
          for (int q = 0; q < spu; q++) {
            const uint32_t sl = next_w();
            const uint64_t wdesc = smem_desc(smem_u32(sm.w[sl]), (uint32_t)(KS * 32));
            const uint64_t wh = wdesc, wl = wdesc + (8192 >> 4);
            PROF_MARK(20)
            if (elect_one()) {
              fence_after();
              for (int kl = 0; kl < KS / 8; kl++) {
                const int k = q * (KS / 8) + kl;
                mma_tf32(acc, dA_hi + 16 * k, wh + 16 * kl, idesc(Wd), k ? 1u : 0u);
                mma_tf32(acc, dA_hi + 16 * k, wl + 16 * kl, idesc(Wd), 1u);
                mma_tf32(acc, dA_lo + 16 * k, wh + 16 * kl, idesc(Wd), 1u);
              }
              mma_commit(&sm.wempty[sl]);
              if (q == spu - 1) mma_commit(&sm.g1done[u & 1]);
            }
            __syncwarp();
            PROF_MARK(22)
          }
        };
        // GEMM2 of hidden chunk c, half g (K steps 2g, 2g+1): A = group g's
        // 16-column H buffer, so each group refills its buffer as soon as its
        // own half has been read
        auto gemm2_half = [&](int c, int g, uint32_t sl) {
          const uint64_t wh = dW2 + (uint64_t)((sl * kWItem) >> 4), wl = wh + (kW2 >> 4);
          const uint64_t hh = smem_desc(smem_u32(sm.h[g][0]), 512), hl = smem_desc(smem_u32(sm.h[g][1]), 512);
          const uint32_t acc = tmem + 64 * s;
          const uint32_t th = tmem + h_base + 32 * g, tl = th + 16;  // TMEM H (htm)
          PROF_MARK(20)
          if (elect_one()) {
            fence_after();
            if (htm) {
#pragma unroll
              for (int kk = 0; kk < 2; kk++) {
                const int k = 2 * g + kk;
                mma_tf32_ts(acc, th + 8 * kk, wh + 16 * k, idesc(kD), (c | k) ? 1u : 0u);
                mma_tf32_ts(acc, th + 8 * kk, wl + 16 * k, idesc(kD), 1u);
                mma_tf32_ts(acc, tl + 8 * kk, wh + 16 * k, idesc(kD), 1u);
              }
            } else {
#pragma unroll
              for (int kk = 0; kk < 2; kk++) {
                const int k = 2 * g + kk;
                mma_tf32(acc, hh + 16 * kk, wh + 16 * k, idesc(kD), (c | k) ? 1u : 0u);
                mma_tf32(acc, hh + 16 * kk, wl + 16 * k, idesc(kD), 1u);
                mma_tf32(acc, hl + 16 * kk, wh + 16 * k, idesc(kD), 1u);
              }
            }
            mma_commit(&sm.g2done[g]);
            if (g == 1) {
              mma_commit(&sm.wempty[sl]);
              if (c == nc - 1) mma_commit(&sm.stage_done);
            }
          }
          __syncwarp();
          PROF_MARK(23)
        };
        PROF_MARK(20)
        mbar_wait(&sm.a_full, ph_afull);
        ph_afull ^= 1;
        fence_after();
        PROF_MARK(16)
        gemm1(0);
        if (nu > 1) gemm1(1);
        for (int c = 0; c < nc; c++) {
          const uint32_t sl = next_w();
#pragma unroll
          for (int g = 0; g < 2; g++) {
            PROF_MARK(20)
            mbar_wait(&sm.epidone[g], ph_epi);
            fence_after();
            PROF_MARK(17)
            gemm2_half(c, g, sl);
          }
          ph_epi ^= 1;
          if ((c & (spu - 1)) == spu - 1 && (c >> lspu) + 2 < nu) gemm1((c >> lspu) + 2);
        }
        PROF_MARK(20)
      } else if (s == S0) {
        // ============ weight loader (warp 9): every item of this step, in
        // consumption order, as ring slots free up
        const uint32_t per = (uint32_t)(A.H / 16);  // items per stage
        const uint32_t n_items = per * (uint32_t)(S - S0);
        for (uint32_t i = 0; i < n_items; i++, wq_load++) {
          const uint32_t sl = wq_load % kNS;
          if (wq_load >= (uint32_t)kNS) mbar_wait(&sm.wempty[sl], ((wq_load / kNS) - 1) & 1);
          if (elect_one()) {
            mbar_expect_tx(&sm.wfull[sl], kWItem);
            bulk_g2s(sm.w[sl], (const char*)A.wprep + sm.seq[S0 + i / per][i % per], kWItem,
                     &sm.wfull[sl]);
          }
          __syncwarp();
        }
      }
    }

    // ================= control: the rest of step_once.  Each row group
    // handles its 32 columns; the NumPy-order norm is finished by both groups
    // from the exchanged partial sums, so both keep identical row state.
    fence_before();
    PROF_MARK(21)
    if (wg < 2) asm volatile("bar.sync 1, 256;" ::: "memory");
    fence_after();
    PROF_MARK(9)
    if (wg < 2) {
      double* ynb = reinterpret_cast<double*>(sm.a[0]);   // y_next, [column][row]
      double* p0 = reinterpret_cast<double*>(sm.w[0]);    // group 0's 8 partial sums
      double* q1 = reinterpret_cast<double*>(sm.h);       // group 1's squared ratios
      double sq[8];
#pragma unroll
      for (int ch = 0; ch < 2; ch++) {
        const int c0 = 32 * wg + 16 * ch;
        double sb[16], se[16];
#pragma unroll
        for (int j = 0; j < S; j++) {
          float kv[16];
          tmem_ld16(lrow + 64 * j + c0, kv);
          const double bj = T::b(j), ej = T::e(j);
#pragma unroll
          for (int e = 0; e < 16; e++) {
            const double kd = (double)kv[e];
            sb[e] = j == 0 ? O::mul(bj, kd) : O::mad(bj, kd, sb[e]);
            se[e] = j == 0 ? O::mul(ej, kd) : O::mad(ej, kd, se[e]);
          }
        }
#pragma unroll
        for (int e = 0; e < 16; e++) {
          const int c = c0 + e;
          const double y = sm.ys[c][row];
          const double yn = O::mad(h, sb[e], y);
          const double err = O::mul(h, se[e]);
          const double scale = O::mad(rtol, np_max(fabs(y), fabs(yn)), atol);
          const double r = FAST ? __dmul_rn(err, fast_rcp1(scale)) : ddiv(err, scale);
          const double q = O::mul(r, r);
          if (wg == 0) {
            sq[c & 7] = c < 8 ? q : ExactOps::add(sq[c & 7], q);  // NumPy pairwise, n = 64
          } else {
            q1[(c - 32) * kRows + row] = q;
          }
          ynb[c * kRows + row] = yn;
        }
      }
      if (wg == 0) {
#pragma unroll
        for (int j = 0; j < 8; j++) p0[j * kRows + row] = sq[j];
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 8; j++) sq[j] = p0[j * kRows + row];
#pragma unroll
      for (int c = 32; c < kD; c++) sq[c & 7] = ExactOps::add(sq[c & 7], q1[(c - 32) * kRows + row]);
      double nrm = ExactOps::add(ExactOps::add(ExactOps::add(sq[0], sq[1]), ExactOps::add(sq[2], sq[3])),
                                 ExactOps::add(ExactOps::add(sq[4], sq[5]), ExactOps::add(sq[6], sq[7])));
      bool accept = false;
      double dtn = h;
      if (FAST && A.ctrl.plain_pi) {  // squared norm, one exp (bode_device.cuh)
        double ms = __dmul_rn(nrm, 1.0 / kD);  // (exact: kD is a power of two)
        ms = ms < INFINITY ? ms : __longlong_as_double(0x7ff0000000000000LL);  // NaN -> inf
        if (have) accept = adapt_pi_ms(A.ctrl, ms, L1, dtn, g_pow_tables);
      } else {
        nrm = dsqrt(ddiv(nrm, (double)kD));
        if (!isfinite(nrm)) nrm = __longlong_as_double(0x7ff0000000000000LL);
        if (have) accept = adapt(A.ctrl, nrm, n1, n2, dtn);
      }
      const int64_t cursor_before = cursor;
      // dense output for every crossed point (solver.py:284-322), pre-commit state
      bool pend = have && accept && cursor < m && h != 0.0;
      while (__any_sync(0xffffffffu, pend)) {
        double th = 0.0;
        if (pend) {
          th = ddiv(ExactOps::sub(te[cursor], t), h);
          if (!(th <= 1.0)) pend = false;
          th = np_max(th, 0.0);
        }
        if (!__any_sync(0xffffffffu, pend)) break;
        double w[S];
#pragma unroll
        for (int q = 0; q < S; q++) {
          double v = T::w(q, T::NI - 1);
#pragma unroll
          for (int r = T::NI - 2; r >= 0; r--) v = O::mad(v, th, T::w(q, r));
          w[q] = O::mul(v, th);
        }
#pragma unroll
        for (int ch = 0; ch < 2; ch++) {
          const int c0 = 32 * wg + 16 * ch;
          double sa[16];
#pragma unroll
          for (int j = 0; j < S; j++) {
            float kv[16];
            tmem_ld16(lrow + 64 * j + c0, kv);
#pragma unroll
            for (int e = 0; e < 16; e++)
              sa[e] = j == 0 ? O::mul(w[0], (double)kv[e])
                             : O::mad(w[j], (double)kv[e], sa[e]);
          }
          if (pend && yout) {
#pragma unroll
            for (int e = 0; e < 16; e++)
              yout[cursor * kD + c0 + e] = O::mad(h, sa[e], sm.ys[c0 + e][row]);
          }
        }
        if (pend) {
          cursor++;
          pend = cursor < m;
        }
      }
      // gradients: record (t_old, h, cursor before the step, y_old) of an
      // accepted step; each row group writes its 32 columns, group 0 the
      // scalars (rows bounded: they were sized by an identical solve)
      if (A.traj && have && accept) {
        const int64_t r0 = A.traj_offsets[idx];
        if (nacc < A.traj_offsets[idx + 1] - r0) {
          double* rec = A.traj + (r0 + nacc) * BODE_TRAJ_STRIDE(kD);
          if (wg == 0) {
            rec[0] = t;
            rec[1] = h;
            rec[2] = (double)cursor_before;
          }
#pragma unroll 8
          for (int c = 32 * wg; c < 32 * wg + 32; c++) rec[BODE_TRAJ_EXTRA + c] = sm.ys[c][row];
        }
      }
      // commit: y <- y_next, FSAL k_0 <- k_{S-1} on accepted rows (my columns)
      if (have && accept) {
#pragma unroll 8
        for (int c = 32 * wg; c < 32 * wg + 32; c++) sm.ys[c][row] = ynb[c * kRows + row];
      }
      if (T::FSAL && __any_sync(0xffffffffu, have && accept)) {
#pragma unroll
        for (int ch = 0; ch < 2; ch++) {
          const int c0 = 32 * wg + 16 * ch;
          float k0[16], kl[16];
          tmem_ld16(lrow + c0, k0);
          tmem_ld16(lrow + 64 * (S - 1) + c0, kl);
          if (have && accept) {
#pragma unroll
            for (int e = 0; e < 16; e++) k0[e] = kl[e];
          }
          tmem_st16(lrow + c0, k0);
        }
        tmem_wait_st();
      }
      if (have) {
        int status = BODE_RUNNING;
        if (accept) {
          nacc++;
          t = trunc ? t_end : ExactOps::add(t, h);
          if (trunc) status = BODE_SUCCESS;
        }
        nsteps++;
        dt = dtn;
        if (status == BODE_RUNNING && ExactOps::add(t, dt) == t) status = BODE_STEP_UNDERFLOW;
        if (status == BODE_RUNNING && nsteps >= A.max_steps) status = BODE_MAX_STEPS_EXCEEDED;
        if (wg == 0 && !accept && status == BODE_RUNNING) {
          const uint64_t bit = (uint64_t)nsteps;  // rejected at iteration nsteps-1
          atomicOr(&A.refresh[bit >> 5], 1u << (bit & 31));
        }
        if (status != BODE_RUNNING) {
          if (wg == 0) {
            A.n_steps[idx] = nsteps;
            A.n_accepted[idx] = nacc;
            A.n_emitted[idx] = cursor;
            A.final_dt[idx] = dt;
            A.status[idx] = status;
            if ((unsigned long long)nsteps > my_max) my_max = (unsigned long long)nsteps;
          }
          have = false;
        }
      }
    }
#ifdef BODE_FUSED_PROF
    PROF_MARK(10)
    pf[30] += 1;
#endif
  }
#ifdef BODE_FUSED_PROF
  if (A.prof && (tid == 0 || tid == 128 || tid == 256)) {
    for (int k = 0; k < 32; k++) A.prof[(blockIdx.x * 3 + (tid >> 7)) * 32 + k] = pf[k];
  }
#endif

  // ---- teardown: no bulk copy may still be landing in this CTA's smem
  // (the loader issues exactly the items the MMA warp consumes, so no bulk
  // copy is in flight here)
  if (wg == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, my_max, o);
      my_max = v > my_max ? v : my_max;
    }
    if (lane == 0 && my_max) atomicMax(A.max_n, my_max);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(sm.tmem_base));
}

}  // namespace fused

bool mlp_fused_supported(int64_t D, int64_t H, int method) {
  (void)method;
  return D == tc::kD && H % tc::kHc == 0 && H / tc::kHc <= fused::kMaxChunks;
}

template <int M>
cudaError_t mlp_fused_launch(const MlpFusedArgs& A, cudaStream_t st) {
  const size_t smem = sizeof(fused::Smem);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fused::mlp_fused_kernel<M, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fused::mlp_fused_kernel<M, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (A.fast)
    fused::mlp_fused_kernel<M, true><<<sms, fused::kThreads, smem, st>>>(A);
  else
    fused::mlp_fused_kernel<M, false><<<sms, fused::kThreads, smem, st>>>(A);
  return cudaGetLastError();
}

template cudaError_t mlp_fused_launch<BODE_METHOD_DOPRI5>(const MlpFusedArgs&, cudaStream_t);
template cudaError_t mlp_fused_launch<BODE_METHOD_TSIT5>(const MlpFusedArgs&, cudaStream_t);
template cudaError_t mlp_fused_launch<BODE_METHOD_HEUN>(const MlpFusedArgs&, cudaStream_t);

}  // namespace bode
