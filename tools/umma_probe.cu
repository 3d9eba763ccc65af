// umma_probe.cu -- checks the tcgen05 operand/accumulator layouts the MLP
// adjoint kernel relies on (kind::tf32, no swizzle), against a host
// reference:
//   T1  M=64 accumulator at TMEM lane 0 (rows -> lanes 0-15 of each warp
//       quadrant), A and B MN-major views of K-major-stored row tiles:
//       D0[c][j] = sum_r Y[r][c] U[r][j]
//   T2  a second M=64 accumulator interleaved at lane 16, same columns:
//       D1[o][j] = sum_r G[r][o] U[r][j]
//   T3  M=128, A K-major (G rows), B MN-major view of a K-major [o][j]
//       weight chunk: D2[r][j] = sum_o G[r][o] W[o][j]
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ __forceinline__ uint32_t cm_off(int r, int k, int kcols) {
  return (uint32_t)((r >> 3) * (kcols / 4) * 128 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amn, int bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(t), "l"(a), "l"(b),
               "r"(id), "r"(acc));
}

struct Sm {
  float y[128 * 64];   // Y rows, K-major cm_off(r, c, 64)
  float g[128 * 64];   // G rows
  float u[128 * 32];   // U rows, cm_off(r, j, 32)
  float w[64 * 32];    // W chunk [o][j], cm_off(o, j, 32)
  float wt[32 * 64];   // the same chunk transposed, K-major [j][o], cm_off(j, o, 64)
  float yt[64 * 128];  // Y^T K-major: (c, r) at cm_off(c, r, 128)
  float gt[64 * 128];  // G^T
  float ut[32 * 128];  // U^T: (j, r) at cm_off(j, r, 128)
  uint64_t bar;
  uint32_t tmem;
};

__global__ void probe(const float* Y, const float* G, const float* U, const float* W, float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  Sm& s = *reinterpret_cast<Sm*>(raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * 64; e += 128) {
    const int r = e / 64, c = e % 64;
    s.y[cm_off(r, c, 64) / 4] = Y[e];
    s.g[cm_off(r, c, 64) / 4] = G[e];
  }
  for (int e = tid; e < 128 * 32; e += 128) s.u[cm_off(e / 32, e % 32, 32) / 4] = U[e];
  for (int e = tid; e < 128 * 64; e += 128) {
    const int r = e / 64, c = e % 64;
    s.yt[cm_off(c, r, 128) / 4] = Y[e];
    s.gt[cm_off(c, r, 128) / 4] = G[e];
  }
  for (int e = tid; e < 128 * 32; e += 128) s.ut[cm_off(e % 32, e / 32, 128) / 4] = U[e];
  for (int e = tid; e < 64 * 32; e += 128) {
    s.w[cm_off(e / 32, e % 32, 32) / 4] = W[e];
    s.wt[cm_off(e % 32, e / 32, 64) / 4] = W[e];
  }
  {  // poison the rest of shared memory: a read outside the tiles shows as NaN
    float* rest = reinterpret_cast<float*>(raw + sizeof(Sm));
    for (int e = tid; e < (200 * 1024 - (int)sizeof(Sm)) / 4; e += 128) rest[e] = __int_as_float(0x7fc00000);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s.bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&s.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = s.tmem;
  if (tid == 0) {
    // T1 / T2: K = 128 rows in 16 steps of 8; A MN-major (SBO 128 between
    // 4-column groups, one 8-row K group per MMA), B MN-major likewise
    for (int k = 0; k < 16; k++) {
      mma(t, desc(su32(s.yt) + 256 * k, 128, 4096), desc(su32(s.ut) + 256 * k, 128, 4096),
          idesc(64, 32, 0, 0), k ? 1u : 0u);
      mma(t + (16u << 16), desc(su32(s.gt) + 256 * k, 128, 4096), desc(su32(s.ut) + 256 * k, 128, 4096),
          idesc(64, 32, 0, 0), k ? 1u : 0u);
    }
    // T3: K = 64 (o) in 8 steps; A K-major G, B MN-major view of W;
    // variants v: (LBO, SBO) = (1024, 128), (128, 1024)
    for (int v = 0; v < 2; v++)
      for (int k = 0; k < 8; k++)
        mma(t + 32 + 32 * v, desc(su32(s.g) + 256 * k, 128, 2048),
            desc(su32(s.w) + 1024 * k, v ? 128 : 1024, v ? 1024 : 128), idesc(128, 32, 0, 1), k ? 1u : 0u);
    // sweep: (LBO, SBO) in {128, 256, 512, 1024}^2 into columns 128 + 32 v
    for (int v = 0; v < 12; v++)
      for (int k = 0; k < 8; k++)
        mma(t + 128 + 32 * v, desc(su32(s.g) + 256 * k, 128, 2048),
            desc(su32(s.w) + 1024 * k, 128u << (v & 3), 128u << (v >> 2)), idesc(128, 32, 0, 1), k ? 1u : 0u);
    // T0: the same product with B K-major (the forward's layout): sanity
    for (int k = 0; k < 8; k++)
      mma(t + 96, desc(su32(s.g) + 256 * k, 128, 2048), desc(su32(s.wt) + 256 * k, 128, 2048),
          idesc(128, 32, 0, 0), k ? 1u : 0u);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&s.bar))
                 : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
                   su32(&s.bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int half = 0; half < 16; half++) {
    uint32_t r[32];
    const uint32_t a = t + ((uint32_t)(warp * 32) << 16) + 32 * half;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; j++) out[(half * 128 + tid) * 32 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

int main() {
  float *Y, *G, *U, *W, *out;
  cudaMallocManaged(&Y, 128 * 64 * 4);
  cudaMallocManaged(&G, 128 * 64 * 4);
  cudaMallocManaged(&U, 128 * 32 * 4);
  cudaMallocManaged(&W, 64 * 32 * 4);
  cudaMallocManaged(&out, 16 * 128 * 32 * 4);
  srand(1);
  auto v = []() { return (float)((rand() % 17) - 8) / 8.0f; };  // exact in tf32
  for (int e = 0; e < 128 * 64; e++) Y[e] = v(), G[e] = v();
  for (int e = 0; e < 128 * 32; e++) U[e] = v();
  for (int e = 0; e < 64 * 32; e++) W[e] = v();
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe<<<1, 128, 200 * 1024>>>(Y, G, U, W, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  double e1 = 0, e2 = 0, e3 = 0, e4 = 0, e0 = 0;
  for (int lane = 0; lane < 128; lane++) {
    const int w = lane / 32, l = lane % 32;
    const int m = 16 * w + (l & 15);
    for (int j = 0; j < 32; j++) {
      double ref = 0;
      for (int r = 0; r < 128; r++) ref += (double)(l < 16 ? Y[r * 64 + m] : G[r * 64 + m]) * U[r * 32 + j];
      const double got = out[lane * 32 + j];
      (l < 16 ? e1 : e2) = fmax(l < 16 ? e1 : e2, fabs(got - ref));
      double r3 = 0;
      for (int o = 0; o < 64; o++) r3 += (double)G[lane * 64 + o] * W[o * 32 + j];
      e3 = fmax(e3, fabs(out[(128 + lane) * 32 + j] - r3));
      e4 = fmax(e4, fabs(out[(256 + lane) * 32 + j] - r3));
      e0 = fmax(e0, fabs(out[(384 + lane) * 32 + j] - r3));
    }
  }
  printf("T0 (M=128, K-major sanity) %g\nT1 (M=64 lane0, A/B MN-major) max err %g\nT2 (M=64 lane16) max err %g\n"
         "T3 (M=128, B MN-major, LBO=K stride) %g\nT3' (swapped) %g\n", e0, e1, e2, e3, e4);
  for (int v = 0; v < 12; v++) {
    double ev = 0;
    for (int lane = 0; lane < 128; lane++)
      for (int j = 0; j < 32; j++) {
        double r3 = 0;
        for (int o = 0; o < 64; o++) r3 += (double)G[lane * 64 + o] * W[o * 32 + j];
        ev = fmax(ev, fabs(out[((4 + v) * 128 + lane) * 32 + j] - r3));
      }
    printf("sweep LBO=%d SBO=%d err %g  first %g %g\n", 128 << (v & 3), 128 << (v >> 2), ev,
           out[((4 + v) * 128) * 32], out[((4 + v) * 128) * 32 + 1]);
  }
  for (int j = 0; j < 8; j++) printf("%g/%g ", out[(128) * 32 + j], out[(384) * 32 + j]);
  printf("\n");
  return (e1 == 0 && e2 == 0 && e3 == 0) ? 0 : 3;
}
