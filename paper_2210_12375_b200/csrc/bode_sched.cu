// bode_sched.cu -- longest-processing-time-first queue order on the device.
//
// The persistent solver hands instances to lanes in queue order; with a
// heavy-tailed step-count distribution (p50 241 vs p99
// 8,483 steps) the solve time is set by whatever long instance is picked up
// last.  Queuing instances in decreasing cost makes the tail short (LPT).
// An exact sort is unnecessary: a counting sort over 1/8-octave buckets of
// the cost (binary exponent clamped to [-64, 63] and the top 3 mantissa bits,
// 1024 buckets) is enough.  Histograms and ranks live in shared memory; each
// block reserves one contiguous output range per non-empty bucket with a
// single global atomic, so there is no global-atomic hot spot even when all
// costs fall into a handful of buckets.  Order within a bucket is arbitrary:
// results never depend on the order, only the schedule does.
#include <cuda_runtime.h>

#include "bode_sched.cuh"

namespace bode {

namespace {
constexpr int kBuckets = 1024;
constexpr int kThreads = 1024;

__device__ __forceinline__ int bucket_of(double c) {
  if (!(c > 0.0)) return 0;  // non-positive / NaN costs go last
  const long long bits = __double_as_longlong(c);
  int ex = (int)((bits >> 52) & 0x7ff) - 1023;
  ex = ex < -64 ? -64 : (ex > 63 ? 63 : ex);
  return (ex + 64) * 8 + (int)((bits >> 49) & 7);
}

// per-block shared histogram, merged into the global one
__global__ void __launch_bounds__(kThreads) lpt_hist_kernel(const double* cost, int64_t n,
                                                            uint32_t* hist) {
  __shared__ uint32_t s[kBuckets];
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) s[b] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&s[bucket_of(cost[i])], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x)
    if (s[b]) atomicAdd(&hist[b], s[b]);
}

// exclusive scan of the histogram in DESCENDING bucket order
__global__ void __launch_bounds__(kThreads) lpt_scan_kernel(uint32_t* hist) {
  __shared__ uint32_t part[kBuckets];
  const int t = threadIdx.x;
  const uint32_t v = hist[kBuckets - 1 - t];
  part[t] = v;
  __syncthreads();
  for (int off = 1; off < kBuckets; off <<= 1) {
    const uint32_t x = t >= off ? part[t - off] : 0u;
    __syncthreads();
    part[t] += x;
    __syncthreads();
  }
  hist[kBuckets - 1 - t] = part[t] - v;
}

// each block re-counts its (same) elements, reserves one range per bucket
// with one global atomic, then ranks locally with shared atomics
__global__ void __launch_bounds__(kThreads) lpt_scatter_kernel(const double* cost, int64_t n,
                                                               uint32_t* cursor, int64_t* order) {
  __shared__ uint32_t s[kBuckets];
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) s[b] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&s[bucket_of(cost[i])], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x)
    if (s[b]) s[b] = atomicAdd(&cursor[b], s[b]);
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    order[atomicAdd(&s[bucket_of(cost[i])], 1u)] = i;
}
}  // namespace

size_t lpt_workspace_bytes(int64_t n) { return (size_t)kBuckets * 4 + 8 * (size_t)n; }

cudaError_t lpt_order(const double* cost, int64_t n, void* ws, int64_t** order_out,
                      cudaStream_t st) {
  uint32_t* hist = (uint32_t*)ws;
  int64_t* order = (int64_t*)((char*)ws + (size_t)kBuckets * 4);
  cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)kBuckets * 4, st);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nb = (n + kThreads - 1) / kThreads;
  const unsigned grid = (unsigned)(nb < sms ? nb : sms);
  lpt_hist_kernel<<<grid, kThreads, 0, st>>>(cost, n, hist);
  lpt_scan_kernel<<<1, kThreads, 0, st>>>(hist);
  lpt_scatter_kernel<<<grid, kThreads, 0, st>>>(cost, n, hist, order);
  *order_out = order;
  return cudaGetLastError();
}

}  // namespace bode
