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
