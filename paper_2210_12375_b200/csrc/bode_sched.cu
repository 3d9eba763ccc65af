// bode_sched.cu -- longest-processing-time-first queue order on the device.
//
// The persistent solver hands instances to lanes in queue order; with a
// heavy-tailed step-count distribution (p50 241 vs p99
// 8,483 steps) the solve time is set by whatever long instance is picked up
// last.  Queuing instances in decreasing cost makes the tail short (LPT).
// An exact sort is unnecessary: a counting sort over 1/16-octave buckets of
// the cost (the top 15 bits of a positive IEEE double, which order like the
// values) costs three small launches and no host round trip.  Order within
// a bucket is arbitrary -- results never depend on the order, only the
// schedule does (batch independence).
#include <cuda_runtime.h>

#include "bode_sched.cuh"

namespace bode {

namespace {
constexpr int kBuckets = 1 << 15;

__device__ __forceinline__ uint32_t bucket_of(double c) {
  if (!(c > 0.0)) return 0;  // non-positive / NaN costs go last
  const unsigned long long bits = (unsigned long long)__double_as_longlong(c);
  return (uint32_t)(bits >> 48) & (kBuckets - 1);
}

__global__ void lpt_hist_kernel(const double* cost, int64_t n, uint32_t* hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[bucket_of(cost[i])], 1u);
}

// exclusive scan over buckets in DESCENDING key order; one block of 1024
// threads, 32 buckets per thread
__global__ void __launch_bounds__(1024) lpt_scan_kernel(uint32_t* hist) {
  __shared__ uint32_t part[1024];
  const int t = threadIdx.x;
  uint32_t v[32], s = 0;
#pragma unroll
  for (int j = 0; j < 32; j++) {
    v[j] = hist[kBuckets - 1 - (t * 32 + j)];
    s += v[j];
  }
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const uint32_t x = t >= off ? part[t - off] : 0u;
    __syncthreads();
    part[t] += x;
    __syncthreads();
  }
  uint32_t run = part[t] - s;
#pragma unroll
  for (int j = 0; j < 32; j++) {
    hist[kBuckets - 1 - (t * 32 + j)] = run;
    run += v[j];
  }
}

__global__ void lpt_scatter_kernel(const double* cost, int64_t n, uint32_t* cursor,
                                   int64_t* order) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    order[atomicAdd(&cursor[bucket_of(cost[i])], 1u)] = i;
}
}  // namespace

size_t lpt_workspace_bytes(int64_t n) { return (size_t)kBuckets * 4 + 8 * (size_t)n; }

cudaError_t lpt_order(const double* cost, int64_t n, void* ws, int64_t** order_out,
                      cudaStream_t st) {
  uint32_t* hist = (uint32_t*)ws;
  int64_t* order = (int64_t*)((char*)ws + (size_t)kBuckets * 4);
  cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)kBuckets * 4, st);
  if (e != cudaSuccess) return e;
  const int64_t nb = (n + 255) / 256;
  const unsigned grid = (unsigned)(nb < 148 * 16 ? nb : 148 * 16);
  lpt_hist_kernel<<<grid, 256, 0, st>>>(cost, n, hist);
  lpt_scan_kernel<<<1, 1024, 0, st>>>(hist);
  lpt_scatter_kernel<<<grid, 256, 0, st>>>(cost, n, hist, order);
  *order_out = order;
  return cudaGetLastError();
}

}  // namespace bode
