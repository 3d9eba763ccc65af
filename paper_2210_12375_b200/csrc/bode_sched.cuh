// bode_sched.cuh -- LPT queue ordering (bode_sched.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace bode {
size_t lpt_workspace_bytes(int64_t n);
// Builds a longest-first permutation of [0, n) from per-instance costs into
// the workspace; *order_out points into ws.
cudaError_t lpt_order(const double* cost, int64_t n, void* ws, int64_t** order_out,
                      cudaStream_t st);
// inv[order[q]] = q (queue position of every instance)
cudaError_t inverse_order(const int64_t* order, int64_t n, int64_t* inv, cudaStream_t st);
// multi-GPU shard plan (bode_partition in bode.h): sizes on the host,
// the rank-major permutation on the device
void compute_shard_sizes(int64_t n, int32_t world, bool snake, int64_t* sizes);
cudaError_t shard_partition(const double* cost, int64_t n, int32_t world, int64_t* perm,
                            void* ws, cudaStream_t st);
}  // namespace bode
