// bode_mlp_tc.cu -- MLP stage evaluation on the 5th-generation tensor cores.
//
// f(Y) = W2 tanh(W1 Y + b1) + b2 for tiles of 128 running instances, one
// persistent CTA per SM, two warp groups:
//   producer (warps 4-7)  forms the stage input Y = y + h * sum_j a_sj k_j in
//                         fp64 (reference order, stepper.py:81-89), rounds to
//                         fp32, splits into TF32 hi + lo and writes the UMMA
//                         K-major core-matrix tile into one of two A buffers;
//   consumer (warps 0-3)  per 32-wide hidden chunk c (H = 256 -> 8 chunks):
//     GEMM1    acc1[128x32] = Y W1_c^T as 3xTF32 (hi*hi + hi*lo + lo*hi),
//              24 tcgen05.mma kind::tf32 (M=128, N=32, K=8), fp32 in TMEM;
//     epilogue tcgen05.ld acc1, + b1, tanh, split hi/lo -> smem (A of GEMM2);
//     GEMM2    acc2[128x64] += H_c W2_c^T (3xTF32, 12 MMAs, N=64);
//   and finally tcgen05.ld acc2, + b2 -> the k_s rows of the instances.
// Weight chunks (pre-split to TF32 hi/lo tiles once per solve) stream in
// with cp.async.bulk (TMA engine) into separate W1/W2 buffers, each
// prefetched as soon as the MMA that read it has completed; the producer
// fills the next tile's A buffer while the consumer works on this one.
// One elected lane of warp 0 issues every MMA; completions are tcgen05.commit ->
// mbarrier.  3xTF32 keeps ~fp32 accuracy: plain TF32 inflates step counts
// by +613% at rtol = 1e-6 (SURVEY.md finding 6).
#include <cuda_runtime.h>

#include "bode_mlp.cuh"
#include "bode_tc.cuh"

namespace bode {
namespace tc {

struct Smem {
  uint8_t a[2][2][kATile];  // [buffer][hi, lo]
  uint8_t h[2][kHTile];     // [hi, lo]
  uint8_t w1[2][kW1];
  uint8_t w2[2][kW2];
  uint64_t full[2], empty[2], mb_w1, mb_w2, mb_g1, mb_g2;
  uint32_t tmem_base;
};

// weight chunk c in global: [W1hi | W1lo | W2hi | W2lo] (8 KB each), already
// in the core-matrix layouts the MMAs read
__global__ void mlp_tc_prep_kernel(const float* __restrict__ W1, const float* __restrict__ W2,
                                   int H, float* __restrict__ out) {
  const int nchunk = H / kHc;
  const int total = nchunk * kHc * kD;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int c = e / (kHc * kD), rem = e % (kHc * kD);
    char* base = (char*)out + (size_t)c * kWChunk;
    {  // W1 chunk: row = hidden j in chunk (32), K = input k (64)
      const int j = rem / kD, k = rem % kD;
      const float w = W1[(size_t)(c * kHc + j) * kD + k];
      const float hi = tf32_hi(w);
      *(float*)(base + cm_off(j, k, kD)) = hi;
      *(float*)(base + kW1 + cm_off(j, k, kD)) = w - hi;
    }
    {  // W2 chunk: row = output o (64), K = hidden j in chunk (32)
      const int o = rem / kHc, j = rem % kHc;
      const float w = W2[(size_t)o * H + c * kHc + j];
      const float hi = tf32_hi(w);
      *(float*)(base + 2 * kW1 + cm_off(o, j, kHc)) = hi;
      *(float*)(base + 2 * kW1 + kW2 + cm_off(o, j, kHc)) = w - hi;
    }
  }
  // W1 again as 16 KB items for wide GEMM1 units (bode_mlp_fused.cu): for
  // unit width Wd in {64, 128}, item (unit u, K slice q) holds rows
  // [u Wd, u Wd + Wd) x K [q KS, q KS + KS), KS = 2048 / Wd, hi then lo
  const int tot1 = H * kD;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * tot1; e += gridDim.x * blockDim.x) {
    const int which = e / tot1, rem = e % tot1;
    const int Wd = which == 0 ? 64 : 128;
    if (H % Wd) continue;
    const int KS = 2048 / Wd;
    const int j = rem / kD, k = rem % kD;  // hidden row, input column
    const int u = j / Wd, r = j % Wd, q = k / KS, kk = k % KS;
    char* item = (char*)out + mlp_w1_items_offset(H, Wd) + (size_t)(u * (kD / KS) + q) * 16384;
    const uint32_t o = (uint32_t)((r >> 3) * (KS / 4) * 128 + (kk >> 2) * 128 + (r & 7) * 16 + (kk & 3) * 4);
    const float w = W1[(size_t)j * kD + k];
    const float hi = tf32_hi(w);
    *(float*)(item + o) = hi;
    *(float*)(item + 8192 + o) = w - hi;
  }
}

template <int M>
__device__ __forceinline__ void produce_tile(const MlpTcArgs& A, int tile, int cnt, uint8_t* ahi,
                                             uint8_t* alo, int pwarp, int lane) {
  using T = Tab<M>;
  // lane -> (row r of an 8-row group, 4-column chunk q): every load is a
  // 16/32-byte vector, all of a lane's loads are issued before the fp64
  // combination, and the 16-byte result rows land in core matrix (g, q)
  const int stage = A.Yin ? -1 : A.stage;
  for (int it = pwarp; it < kRows / 8 * 4; it += 4) {  // 16 row groups x 4 column quarters
    const int g = it >> 2, r = g * 8 + (lane & 7);
    const int q = (it & 3) * 4 + (lane >> 3);           // 4-column chunk 0..15
    const int pr = tile * kRows + r;
    const bool lv = pr < cnt;
    const int64_t ir = lv ? (A.act ? A.act[pr] : pr) : 0;
    float x[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (lv) {
      if (stage < 0) {
        const float4 v = *reinterpret_cast<const float4*>(A.Yin + (size_t)pr * kD + 4 * q);
        x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
      } else {
        const double2* yp = reinterpret_cast<const double2*>(A.y + ir * kD + 4 * q);
        const double2 y01 = __ldg(yp), y23 = __ldg(yp + 1);
        const double yv[4] = {y01.x, y01.y, y23.x, y23.y};
        if (stage == 0) {
#pragma unroll
          for (int e = 0; e < 4; e++) x[e] = (float)yv[e];
        } else {
          float4 kv[T::S];
#pragma unroll
          for (int j = 0; j < T::S; j++)
            if (j < stage)
              kv[j] = __ldg(reinterpret_cast<const float4*>(A.k + ((int64_t)j * A.n + ir) * kD + 4 * q));
          const double hr = A.h[ir];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < T::S; j++) {
              if (j >= stage) break;
              const float kf = e == 0 ? kv[j].x : e == 1 ? kv[j].y : e == 2 ? kv[j].z : kv[j].w;
              s = j == 0 ? ExactOps::mul(T::a(stage, 0), (double)kf)
                         : ExactOps::mad(T::a(stage, j), (double)kf, s);
            }
            x[e] = (float)ExactOps::mad(hr, s, yv[e]);
          }
        }
      }
    }
    if (A.Yout && lv)
      *reinterpret_cast<float4*>(A.Yout + (size_t)ir * kD + 4 * q) = make_float4(x[0], x[1], x[2], x[3]);
    float4 hi, lo;
    hi.x = tf32_hi(x[0]), hi.y = tf32_hi(x[1]), hi.z = tf32_hi(x[2]), hi.w = tf32_hi(x[3]);
    lo.x = x[0] - hi.x, lo.y = x[1] - hi.y, lo.z = x[2] - hi.z, lo.w = x[3] - hi.w;
    const uint32_t o = (uint32_t)((g * 16 + q) * 128 + (r & 7) * 16);
    *reinterpret_cast<float4*>(ahi + o) = hi;
    *reinterpret_cast<float4*>(alo + o) = lo;
  }
}

template <int M>
__global__ void __launch_bounds__(256, 1) mlp_tc_kernel(MlpTcArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cnt = *A.count;
  const int ntiles = (cnt + kRows - 1) / kRows;
  if ((int)blockIdx.x >= ntiles) return;
  const int nchunk = A.H / kHc;

  if (tid == 0) {
    for (int b = 0; b < 2; b++) {
      mbar_init(&S.full[b], 1);
      mbar_init(&S.empty[b], 1);
    }
    mbar_init(&S.mb_w1, 1);
    mbar_init(&S.mb_w2, 1);
    mbar_init(&S.mb_g1, 1);
    mbar_init(&S.mb_g2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        smem_u32(&S.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();

  if (tid >= 128) {
    // ===================== producer: stage-input tiles =====================
    int kl = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, kl++) {
      const int b = kl & 1;
      if (kl >= 2) mbar_wait(&S.empty[b], ((kl >> 1) - 1) & 1);
      produce_tile<M>(A, tile, cnt, S.a[b][0], S.a[b][1], warp - 4, lane);
      fence_async_smem();
      group_sync(1);
      if (tid == 128) mbar_arrive(&S.full[b]);
    }
  } else {
    // ===================== consumer: MMAs + epilogues =====================
    const uint32_t tmem = S.tmem_base;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t acc1 = tmem, acc2 = tmem + 64;
    const uint32_t h_hi = smem_u32(S.h[0]), h_lo = smem_u32(S.h[1]);
    const uint32_t w1h = smem_u32(S.w1[0]), w1l = smem_u32(S.w1[1]);
    const uint32_t w2h = smem_u32(S.w2[0]), w2l = smem_u32(S.w2[1]);
    uint32_t ph_w1 = 0, ph_w2 = 0, ph_g1 = 0, ph_g2 = 0;
    const char* wsrc = (const char*)A.wprep;
    auto load_w1 = [&](int c) {
      mbar_expect_tx(&S.mb_w1, 2 * kW1);
      bulk_g2s(S.w1[0], wsrc + (size_t)c * kWChunk, kW1, &S.mb_w1);
      bulk_g2s(S.w1[1], wsrc + (size_t)c * kWChunk + kW1, kW1, &S.mb_w1);
    };
    auto load_w2 = [&](int c) {
      mbar_expect_tx(&S.mb_w2, 2 * kW2);
      bulk_g2s(S.w2[0], wsrc + (size_t)c * kWChunk + 2 * kW1, kW2, &S.mb_w2);
      bulk_g2s(S.w2[1], wsrc + (size_t)c * kWChunk + 2 * kW1 + kW2, kW2, &S.mb_w2);
    };
    if (tid == 0) {
      load_w1(0);
      load_w2(0);
    }
    int kl = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, kl++) {
      const int b = kl & 1;
      const bool more_tiles = tile + (int)gridDim.x < ntiles;
      const uint32_t a_hi = smem_u32(S.a[b][0]), a_lo = smem_u32(S.a[b][1]);
      mbar_wait(&S.full[b], (kl >> 1) & 1);
      for (int c = 0; c < nchunk; c++) {
        const bool last = c == nchunk - 1;
        const int cn = last ? 0 : c + 1;
        const bool prefetch = !last || more_tiles;
        // ---- GEMM1: acc1 = Y W1_c^T  (3xTF32, K = 64 in 8 steps)
        mbar_wait(&S.mb_w1, ph_w1);
        ph_w1 ^= 1;
        if (warp == 0) {  // warp-uniform descriptors, one elected lane issues
          const uint64_t da[3] = {smem_desc(a_hi, 2048), smem_desc(a_hi, 2048), smem_desc(a_lo, 2048)};
          const uint64_t db[3] = {smem_desc(w1h, 2048), smem_desc(w1l, 2048), smem_desc(w1h, 2048)};
          if (elect_one()) {
            fence_after();
#pragma unroll
            for (int s = 0; s < kD / 8; s++)
#pragma unroll
              for (int term = 0; term < 3; term++)
                mma_tf32(acc1, da[term] + 16 * s, db[term] + 16 * s, idesc(kHc), (term | s) ? 1u : 0u);
            mma_commit(&S.mb_g1);
            if (last) mma_commit(&S.empty[b]);  // A[b] free once this GEMM1 is done
          }
          __syncwarp();
        }
        mbar_wait(&S.mb_g1, ph_g1);
        ph_g1 ^= 1;
        fence_after();
        if (tid == 0 && prefetch) load_w1(cn);
        // ---- epilogue 1: tanh(acc1 + b1) -> H_c hi/lo (row = tid)
        {
          float v[32];
          tmem_ld32(acc1 + lane_off, v);
          float* hh = reinterpret_cast<float*>(S.h[0]);
          float* hl = reinterpret_cast<float*>(S.h[1]);
#pragma unroll
          for (int j = 0; j < kHc; j++) {
            const float hv = tanhf(v[j] + __ldg(A.b1 + c * kHc + j));
            const float hi = tf32_hi(hv);
            const uint32_t o = cm_off(tid, j, kHc) >> 2;
            hh[o] = hi;
            hl[o] = hv - hi;
          }
        }
        fence_async_smem();
        fence_before();
        group_sync(2);
        // ---- GEMM2: acc2 += H_c W2_c^T  (3xTF32, K = 32 in 4 steps)
        mbar_wait(&S.mb_w2, ph_w2);
        ph_w2 ^= 1;
        if (warp == 0) {
          const uint64_t da[3] = {smem_desc(h_hi, 1024), smem_desc(h_hi, 1024), smem_desc(h_lo, 1024)};
          const uint64_t db[3] = {smem_desc(w2h, 1024), smem_desc(w2l, 1024), smem_desc(w2h, 1024)};
          if (elect_one()) {
            fence_after();
#pragma unroll
            for (int s = 0; s < kHc / 8; s++)
#pragma unroll
              for (int term = 0; term < 3; term++)
                mma_tf32(acc2, da[term] + 16 * s, db[term] + 16 * s, idesc(kD), (c | term | s) ? 1u : 0u);
            mma_commit(&S.mb_g2);
          }
          __syncwarp();
        }
        mbar_wait(&S.mb_g2, ph_g2);
        ph_g2 ^= 1;
        fence_after();
        if (tid == 0 && prefetch) load_w2(cn);
      }
      // ---- epilogue 2: k_s = acc2 + b2 for the live rows
      {
        const int p = tile * kRows + tid;
        float v[32];
        const bool live = p < cnt;
        const int64_t i = live ? (A.act ? A.act[p] : p) : 0;
        float* dst = A.out + (size_t)i * kD;
#pragma unroll
        for (int half = 0; half < 2; half++) {
          tmem_ld32(acc2 + lane_off + 32 * half, v);
          if (live) {
#pragma unroll
            for (int o = 0; o < 32; o += 4)
              *reinterpret_cast<float4*>(dst + 32 * half + o) =
                  make_float4(v[o] + __ldg(A.b2 + 32 * half + o), v[o + 1] + __ldg(A.b2 + 32 * half + o + 1),
                              v[o + 2] + __ldg(A.b2 + 32 * half + o + 2),
                              v[o + 3] + __ldg(A.b2 + 32 * half + o + 3));
          }
        }
      }
      fence_before();
      group_sync(2);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(S.tmem_base));
}

}  // namespace tc

size_t mlp_tc_prep_bytes(int64_t H) { return mlp_w1_items_offset(H, 256); }

bool mlp_tc_supported(int64_t D, int64_t H) { return D == tc::kD && H % tc::kHc == 0 && H <= 1024; }

cudaError_t mlp_tc_prep(const float* W1, const float* W2, int64_t H, float* out, cudaStream_t st) {
  tc::mlp_tc_prep_kernel<<<148, 256, 0, st>>>(W1, W2, (int)H, out);
  return cudaGetLastError();
}

template <int M>
cudaError_t mlp_tc_launch(const MlpTcArgs& A, int max_tiles, cudaStream_t st) {
  const size_t smem = sizeof(tc::Smem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc::mlp_tc_kernel<M>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = max_tiles < sms ? (max_tiles < 1 ? 1 : max_tiles) : sms;
  tc::mlp_tc_kernel<M><<<grid, 256, smem, st>>>(A);
  return cudaGetLastError();
}

template cudaError_t mlp_tc_launch<BODE_METHOD_DOPRI5>(const MlpTcArgs&, int, cudaStream_t);
template cudaError_t mlp_tc_launch<BODE_METHOD_TSIT5>(const MlpTcArgs&, int, cudaStream_t);
template cudaError_t mlp_tc_launch<BODE_METHOD_HEUN>(const MlpTcArgs&, int, cudaStream_t);

}  // namespace bode
