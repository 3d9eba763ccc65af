// bode_mlp_tc.cu -- MLP stage evaluation on the 5th-generation tensor cores.
//
// One persistent CTA per SM (128 threads, 192 KB shared memory, 128 TMEM
// columns) streams tiles of 128 running instances:
//   prologue   threads form the stage input Y = y + h * sum_j a_sj k_j in
//              fp64 (reference order, stepper.py:81-89), round to fp32 and
//              split it into TF32 hi + lo, written to shared memory in the
//              UMMA K-major core-matrix layout;
//   per 64-wide hidden chunk c (H = 256 -> 4 chunks):
//     TMA      cp.async.bulk of the pre-split W1/W2 chunk (64 KB) into smem;
//     GEMM1    acc1[128x64] = Y W1_c^T as 3xTF32 (hi*hi + hi*lo + lo*hi),
//              24 tcgen05.mma kind::tf32 (M=128, N=64, K=8), fp32 in TMEM;
//     epilogue tcgen05.ld acc1, + b1, tanh, split hi/lo -> smem (A of GEMM2);
//     GEMM2    acc2[128x64] += H_c W2_c^T, 3xTF32, accumulating over chunks;
//   epilogue2  tcgen05.ld acc2, + b2 -> k_s rows (fp32, scattered to the
//              instance rows of the compacted running list).
// One elected thread issues all MMAs; completion is tracked with
// tcgen05.commit on an mbarrier.  3xTF32 keeps ~fp32 accuracy: plain TF32
// inflates step counts by +613% at rtol = 1e-6 (SURVEY.md finding 6).
#include <cuda_runtime.h>

#include "bode_mlp.cuh"

namespace bode {
namespace tc {

constexpr int kD = 64;         // state width handled by this kernel
constexpr int kChunk = 64;     // hidden units per chunk
constexpr int kRows = 128;     // instances per tile (UMMA M)
constexpr int kTileBytes = kRows * kD * 4;     // 32 KB (one 128x64 fp32 operand)
constexpr int kWBytes = kChunk * kD * 4;       // 16 KB (one 64x64 fp32 operand)
constexpr uint32_t kSBO = 2048, kLBO = 128;    // core-matrix strides (bytes)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// byte offset of element (r, k) in a K-major, no-swizzle core-matrix tile
// with 64 K-elements per row: 8-row x 16-byte core matrices, K-chunks 128 B
// apart (LBO), 8-row groups 2048 B apart (SBO)
__host__ __device__ __forceinline__ uint32_t cm_off(int r, int k) {
  return (uint32_t)((r >> 3) * kSBO + (k >> 2) * kLBO + (r & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((kSBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;                 // base offset 0, layout SWIZZLE_NONE
}
// kind::tf32, fp32 accumulate, A/B K-major, M = 128, N = 64
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) |
                            ((128u >> 4) << 24);

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 64 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]),
        "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]),
        "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),
        "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]),
        "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 64; j++) v[j] = __uint_as_float(r[j]);
}

struct Smem {
  uint8_t a_hi[kTileBytes];
  uint8_t a_lo[kTileBytes];
  uint8_t h_hi[kTileBytes];
  uint8_t h_lo[kTileBytes];
  uint8_t w1[2][kWBytes];  // hi, lo
  uint8_t w2[2][kWBytes];
  uint64_t mb_w;
  uint64_t mb_mma;
  uint32_t tmem_base;
};

// weight chunk c in global: [W1hi | W1lo | W2hi | W2lo], 16 KB each
__global__ void mlp_tc_prep_kernel(const float* __restrict__ W1, const float* __restrict__ W2,
                                   int H, float* __restrict__ out) {
  const int nchunk = H / kChunk;
  const int total = nchunk * kChunk * kD;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int c = e / (kChunk * kD), r = (e / kD) % kChunk, k = e % kD;
    char* base = (char*)out + (size_t)c * 4 * kWBytes;
    const float w1 = W1[(size_t)(c * kChunk + r) * kD + k];  // hidden r of chunk, input k
    const float w1h = tf32_hi(w1);
    *(float*)(base + cm_off(r, k)) = w1h;
    *(float*)(base + kWBytes + cm_off(r, k)) = w1 - w1h;
    const float w2 = W2[(size_t)r * H + c * kChunk + k];     // output r, hidden k of chunk
    const float w2h = tf32_hi(w2);
    *(float*)(base + 2 * kWBytes + cm_off(r, k)) = w2h;
    *(float*)(base + 3 * kWBytes + cm_off(r, k)) = w2 - w2h;
  }
}

template <int M>
__global__ void __launch_bounds__(128, 1) mlp_tc_kernel(MlpTcArgs A) {
  using T = Tab<M>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int cnt = *A.count;
  const int ntiles = (cnt + kRows - 1) / kRows;
  if ((int)blockIdx.x >= ntiles) return;
  const int nchunk = A.H / kChunk;

  if (tid == 0) {
    mbar_init(&S.mb_w, 1);
    mbar_init(&S.mb_mma, 1);
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
  const uint32_t tmem = S.tmem_base;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  uint32_t ph_w = 0, ph_mma = 0;

  const uint32_t a_hi = smem_u32(S.a_hi), a_lo = smem_u32(S.a_lo);
  const uint32_t h_hi = smem_u32(S.h_hi), h_lo = smem_u32(S.h_lo);
  const uint32_t w1h = smem_u32(S.w1[0]), w1l = smem_u32(S.w1[1]);
  const uint32_t w2h = smem_u32(S.w2[0]), w2l = smem_u32(S.w2[1]);

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // ---- prologue: stage input rows -> TF32 hi/lo operand tiles.  A warp
    // fills whole 8x4 core matrices (128 contiguous bytes: conflict-free
    // stores); its lanes read 8 rows x 4 consecutive columns per core
    // matrix, 16 consecutive core matrices covering the same 8 rows.
    const int p = tile * kRows + tid;
    const bool live = p < cnt;
    const int64_t i = live ? (A.act ? A.act[p] : p) : 0;
    {
      float* ah = reinterpret_cast<float*>(S.a_hi);
      float* al = reinterpret_cast<float*>(S.a_lo);
      const int lane = tid & 31;
      for (int g = warp; g < kRows / 8; g += 4) {   // 8-row group
        const int r = g * 8 + (lane >> 2);
        const int pr = tile * kRows + r;
        const bool lv = pr < cnt;
        const int64_t ir = lv ? (A.act ? A.act[pr] : pr) : 0;
        const double hr = (lv && !A.Yin && A.stage > 0) ? A.h[ir] : 0.0;
#pragma unroll 4
        for (int q = 0; q < kD / 4; q++) {            // 4-column chunk
          const int k = q * 4 + (lane & 3);
          float x = 0.0f;
          if (lv) {
            if (A.Yin) {
              x = A.Yin[(size_t)pr * kD + k];
            } else if (A.stage == 0) {
              x = (float)__ldg(A.y + ir * kD + k);
            } else {
              double s = 0.0;
#pragma unroll
              for (int j = 0; j < T::S; j++) {
                if (j >= A.stage) break;
                const double kj = (double)__ldg(A.k + ((int64_t)j * A.n + ir) * kD + k);
                s = j == 0 ? ExactOps::mul(T::a(A.stage, 0), kj)
                           : ExactOps::mad(T::a(A.stage, j), kj, s);
              }
              x = (float)ExactOps::mad(hr, s, __ldg(A.y + ir * kD + k));
            }
          }
          const float hi = tf32_hi(x);
          const int o = (g * 16 + q) * 32 + lane;  // core matrix (g, q), element lane
          ah[o] = hi;
          al[o] = x - hi;
        }
      }
    }
    fence_async_smem();
    for (int c = 0; c < nchunk; c++) {
      // ---- weights of chunk c (the previous chunk's MMAs have completed)
      if (tid == 0) {
        const char* src = (const char*)A.wprep + (size_t)c * 4 * kWBytes;
        mbar_expect_tx(&S.mb_w, 4 * kWBytes);
        bulk_g2s(S.w1[0], src, kWBytes, &S.mb_w);
        bulk_g2s(S.w1[1], src + kWBytes, kWBytes, &S.mb_w);
        bulk_g2s(S.w2[0], src + 2 * kWBytes, kWBytes, &S.mb_w);
        bulk_g2s(S.w2[1], src + 3 * kWBytes, kWBytes, &S.mb_w);
      }
      __syncthreads();  // A tile (and H of the previous chunk) visible
      mbar_wait(&S.mb_w, ph_w);
      ph_w ^= 1;
      // ---- GEMM1: acc1 = Y W1_c^T  (3xTF32, K = 64 in 8 steps)
      if (tid == 0) {
        fence_after();
        const uint32_t aa[3] = {a_hi, a_hi, a_lo}, bb[3] = {w1h, w1l, w1h};
        for (int term = 0; term < 3; term++)
          for (int s = 0; s < kD / 8; s++)
            mma_tf32(tmem, smem_desc(aa[term] + 256 * s), smem_desc(bb[term] + 256 * s),
                     (term | s) ? 1u : 0u);
        mma_commit(&S.mb_mma);
      }
      __syncwarp();
      mbar_wait(&S.mb_mma, ph_mma);
      ph_mma ^= 1;
      fence_after();
      // ---- epilogue 1: tanh(acc1 + b1) -> H_c hi/lo
      {
        float v[64];
        tmem_ld64(tmem + lane_off, v);
        float* hh = reinterpret_cast<float*>(S.h_hi);
        float* hl = reinterpret_cast<float*>(S.h_lo);
#pragma unroll
        for (int j = 0; j < kChunk; j++) {
          const float hv = tanhf(v[j] + A.b1[c * kChunk + j]);
          const float hi = tf32_hi(hv);
          const uint32_t o = cm_off(tid, j) >> 2;
          hh[o] = hi;
          hl[o] = hv - hi;
        }
      }
      fence_async_smem();
      fence_before();
      __syncthreads();
      // ---- GEMM2: acc2 += H_c W2_c^T
      if (tid == 0) {
        fence_after();
        const uint32_t aa[3] = {h_hi, h_hi, h_lo}, bb[3] = {w2h, w2l, w2h};
        for (int term = 0; term < 3; term++)
          for (int s = 0; s < kChunk / 8; s++)
            mma_tf32(tmem + 64, smem_desc(aa[term] + 256 * s), smem_desc(bb[term] + 256 * s),
                     (c | term | s) ? 1u : 0u);
        mma_commit(&S.mb_mma);
      }
      __syncwarp();
      mbar_wait(&S.mb_mma, ph_mma);
      ph_mma ^= 1;
      fence_after();
    }
    // ---- epilogue 2: k_s = acc2 + b2 for the live rows
    {
      float v[64];
      tmem_ld64(tmem + lane_off + 64, v);
      if (live) {
        float* dst = A.out + (size_t)i * kD;
#pragma unroll
        for (int o = 0; o < kD; o += 4)
          *reinterpret_cast<float4*>(dst + o) =
              make_float4(v[o] + A.b2[o], v[o + 1] + A.b2[o + 1], v[o + 2] + A.b2[o + 2],
                          v[o + 3] + A.b2[o + 3]);
      }
    }
    fence_before();
    __syncthreads();
  }
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

}  // namespace tc

size_t mlp_tc_prep_bytes(int64_t H) { return (size_t)(H / tc::kChunk) * 4 * tc::kWBytes; }

bool mlp_tc_supported(int64_t D, int64_t H) { return D == tc::kD && H % tc::kChunk == 0 && H <= 1024; }

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
  tc::mlp_tc_kernel<M><<<grid, 128, smem, st>>>(A);
  return cudaGetLastError();
}

template cudaError_t mlp_tc_launch<BODE_METHOD_DOPRI5>(const MlpTcArgs&, int, cudaStream_t);
template cudaError_t mlp_tc_launch<BODE_METHOD_TSIT5>(const MlpTcArgs&, int, cudaStream_t);
template cudaError_t mlp_tc_launch<BODE_METHOD_HEUN>(const MlpTcArgs&, int, cudaStream_t);

}  // namespace bode
