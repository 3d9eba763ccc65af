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

#include "../../include/bode.h"
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


// ------------------------------------------------------------ partition --
// Multi-GPU shard plan: instances dealt to `world` shards
// in decreasing cost in a snake pattern over the longest-first order
// (positions p = j*W + k go to shard k on even laps j, W-1-k on odd ones),
// which keeps per-shard cost sums within one instance's cost of each other.
// perm = shard 0's instances, then shard 1's, ...; inside a shard they stay
// longest-first, so a shard's own queue order is its row order.
namespace {
// first position of shard r (snake sizes: laps, plus one for the shards the
// last, partial lap reaches -- the first rem on an even lap, the last rem on
// an odd one)
__device__ __forceinline__ int64_t shard_off(int64_t r, int64_t laps, int64_t rem, int64_t w) {
  const int64_t ex = (laps & 1) ? (r > w - rem ? r - (w - rem) : 0) : (r < rem ? r : rem);
  return r * laps + ex;
}

__global__ void shard_perm_kernel(const int64_t* order, int64_t n, int32_t world, int64_t* perm) {
  const int64_t laps = n / world, rem = n % world;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = 0;
    while (r + 1 < world && q >= shard_off(r + 1, laps, rem, world)) r++;
    const int64_t j = q - shard_off(r, laps, rem, world);
    perm[q] = order ? order[j * world + ((j & 1) ? world - 1 - r : r)] : q;
  }
}
}  // namespace

void compute_shard_sizes(int64_t n, int32_t world, bool snake, int64_t* sizes) {
  const int64_t laps = n / world, rem = n % world;
  for (int r = 0; r < world; r++) {
    if (!snake) {
      sizes[r] = n * (r + 1) / world - n * r / world;
    } else {
      const bool extra = (laps & 1) ? (r >= world - rem) : (r < rem);
      sizes[r] = laps + (extra ? 1 : 0);
    }
  }
}

cudaError_t shard_partition(const double* cost, int64_t n, int32_t world, int64_t* perm,
                            void* ws, cudaStream_t st) {
  int64_t* order = nullptr;
  if (cost) {
    const cudaError_t e = lpt_order(cost, n, ws, &order, st);
    if (e != cudaSuccess) return e;
  }
  const int64_t nb = (n + 255) / 256;
  shard_perm_kernel<<<(unsigned)(nb < 148 * 8 ? nb : 148 * 8), 256, 0, st>>>(order, n, world, perm);
  return cudaGetLastError();
}

namespace {
__global__ void inverse_order_kernel(const int64_t* order, int64_t n, int64_t* inv) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    inv[order[q]] = q;
}
}  // namespace

cudaError_t inverse_order(const int64_t* order, int64_t n, int64_t* inv, cudaStream_t st) {
  const int64_t nb = (n + 255) / 256;
  inverse_order_kernel<<<(unsigned)(nb < 148 * 16 ? nb : 148 * 16), 256, 0, st>>>(order, n, inv);
  return cudaGetLastError();
}

}  // namespace bode
