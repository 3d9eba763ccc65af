// mma_cost.cu -- cycles per tcgen05.mma kind::tf32 (M = 128, K = 8) on one
// SM, A from shared memory (SS) or from tensor memory (TS), N = 32..256:
// a chain of back-to-back MMAs into one accumulator, timed from the first
// issue to the commit's mbarrier completing.  Sizes the operand choices of
// the fused MLP kernel and the adjoint's VJP kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 --expt-relaxed-constexpr -I../paper_2210_12375_b200/csrc -o mma_cost mma_cost.cu
#include <cstdio>

#include "bode_tc.cuh"

using namespace bode::tc;

template <int N, bool TS>
__device__ __forceinline__ long long chain(uint32_t tm, uint8_t* sm, uint64_t* bar, uint32_t ph, int n8) {
  // K-major core matrices (8 rows x 16 B): A as a 64-column tile (SBO 2048,
  // K step = +256 B), B as an N x 8 slice per K step (SBO 256, +N * 32 B)
  const uint64_t da = smem_desc(smem_u32(sm), 2048);
  const uint64_t db = smem_desc(smem_u32(sm + 64 * 1024), 256);
  const long long t0 = clock64();
  for (int i = 0; i < n8; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if (TS)
        mma_tf32_ts(tm, tm + 256 + 8 * k, db + ((N * 32 * k) >> 4), idesc(N), (i | k) ? 1u : 0u);
      else
        mma_tf32(tm, da + 16 * k, db + ((N * 32 * k) >> 4), idesc(N), (i | k) ? 1u : 0u);
    }
  }
  mma_commit(bar);
  mbar_wait(bar, ph);
  return clock64() - t0;
}

template <int N, bool TS>
__device__ void measure(uint32_t tm, uint8_t* sm, uint64_t* bar, uint32_t& ph, long long* out, int& slot,
                        int n8) {
  long long c = 0;
  for (int rep = 0; rep < 2; rep++) {
    if (threadIdx.x < 32) {
      if (elect_one()) c = chain<N, TS>(tm, sm, bar, ph, n8);
      __syncwarp();
    }
    ph ^= 1;
    __syncthreads();
  }
  if (threadIdx.x < 32 && c) {
    out[2 * slot] = N * 10 + (TS ? 1 : 0);
    out[2 * slot + 1] = c / (8 * n8);
  }
  slot++;
}

__global__ void cost(long long* out, int n8) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.0f;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = tbase;
  uint32_t ph = 0;
  int slot = 0;
  // accumulator at column 0 (N columns); a TS operand at column 256 (8
  // columns per K step); A in smem at 0 (4 KB per K step), B at 64 KB
  measure<32, false>(tm, sm, &bar, ph, out, slot, n8);
  measure<32, true>(tm, sm, &bar, ph, out, slot, n8);
  measure<64, false>(tm, sm, &bar, ph, out, slot, n8);
  measure<64, true>(tm, sm, &bar, ph, out, slot, n8);
  measure<128, false>(tm, sm, &bar, ph, out, slot, n8);
  measure<128, true>(tm, sm, &bar, ph, out, slot, n8);
  measure<256, false>(tm, sm, &bar, ph, out, slot, n8);
  measure<256, true>(tm, sm, &bar, ph, out, slot, n8);
  fence_before();
  __syncthreads();
  fence_after();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  cudaFuncSetAttribute(cost, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cost<<<1, 128, 200 * 1024>>>(d, 24);
  long long h[64];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  for (int s = 0; s < 8; s++)
    printf("tf32 M=128 N=%lld %s: %lld cycles per MMA\n", h[2 * s] / 10, h[2 * s] % 10 ? "TS (A in TMEM)" : "SS",
           h[2 * s + 1]);
  return 0;
}
