// bode_probe.cu -- roofline denominators measured on the running GPU.
// MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only; the solver is
// FP64-pipe bound, so bench.py measures the FP64 FMA peak with this kernel
// (8 independent DFMA chains per thread, full occupancy, 2 flops per DFMA).
#include "../../include/bode.h"
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) bode_fp64_probe_kernel(int64_t iters, double* out) {
  double a[8];
  const double m = 1.0 + 1e-9 * threadIdx.x, c = 1e-12;
#pragma unroll
  for (int j = 0; j < 8; j++) a[j] = 1.0 + j * 1e-3 + blockIdx.x * 1e-7;
  for (int64_t i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = fma(a[j], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += a[j];
  if (s == 42.0) out[0] = s;  // keep the chains alive
}

extern "C" int bode_probe_fp64(int64_t iters, int32_t blocks, double* out, void* stream) {
  bode_fp64_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, out);
  return cudaGetLastError() == cudaSuccess ? BODE_OK : BODE_ECUDA;
}

// TF32 tensor-core peak (the C4 MLP roofline): one CTA per SM issues
// back-to-back tcgen05.mma kind::tf32, M = 128, N = 256, K = 8 (smem
// operands, fp32 accumulation in TMEM); 2 * 128 * 256 * 8 flops per MMA.
#include "bode_tc.cuh"

__global__ void __launch_bounds__(128, 1) bode_tf32_probe_kernel(int32_t reps) {
  using namespace bode::tc;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < (32768 + 65536) / 4; i += 128) ((float*)smem)[i] = 0.0f;
  fence_async_smem();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) {
    const uint64_t da = smem_desc(smem_u32(smem), 2048), db = smem_desc(smem_u32(smem + 32768), 2048);
    for (int r = 0; r < reps; r++) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; k++) mma_tf32(tbase, da + 16 * k, db + 16 * k, idesc(256), (r | k) ? 1u : 0u);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

extern "C" int bode_probe_tf32(int32_t reps, int32_t blocks, void* stream) {
  const int smem = 32768 + 65536 + 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(bode_tf32_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return BODE_ECUDA;
    attr = true;
  }
  bode_tf32_probe_kernel<<<blocks, 128, smem, (cudaStream_t)stream>>>(reps);
  return cudaGetLastError() == cudaSuccess ? BODE_OK : BODE_ECUDA;
}
