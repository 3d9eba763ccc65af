// bode_mlp_adjoint.cu -- gradients through a neural-ODE solve,
// f(y) = W2 tanh(W1 y + b1) + b2 (fp32 MLP on the fp64 state), the MLP half
// of SURVEY.md §8(f) row 1 (torchode's AutoDiffAdjoint backward; the
// reference has no gradients).
//
// Same definition as the analytic adjoint (bode_adjoint.cu): reverse mode
// through the recorded accepted steps -- stages, solution update, dense
// output -- with step sizes and accept decisions held fixed.  Outputs
// dL/dy0 per instance and dL/dW1, db1, dW2, db2 summed over the batch.
//
// One CTA (256 threads) owns one instance at a time and walks its steps
// backwards; thread j owns hidden unit j, thread c < D state component c.
// Both weight matrices sit in shared memory with padded rows (conflict-free
// for row- and column-wise access), the seven stages' fp32 inputs and
// hidden activations of the step being reversed are kept in shared memory,
// and the weight gradients accumulate in registers of the owning thread
// (row j of dW1, column j of dW2) for every instance the CTA processes;
// per-CTA partials are summed by a second kernel at the end (deterministic
// order).  Per step: 7 MLP evaluations (forward recompute) + 7 VJPs
// (W2^T g, tanh', W1^T v) + the rank-1 weight-gradient updates, fp32 FMA on
// CUDA cores.
#include "bode_adjoint.cuh"
#include "bode_sched.cuh"
#include "bode_solver.cuh"

namespace bode {
namespace {

constexpr int kThreads = 256;

template <int D>
constexpr size_t mlp_adj_smem(int S) {
  return 4 * ((size_t)kThreads * (D + 1) + (size_t)D * (kThreads + 1) + (size_t)S * kThreads +
              (size_t)S * D + 4 * 64 + 64 + kThreads) +
         8 * ((size_t)2 * S * D + 3 * D) + 64;
}

template <int M, int D>
__global__ void __launch_bounds__(kThreads, 1) mlp_adjoint_kernel(const AdjParams A) {
  using T = Tab<M>;
  constexpr int S = T::S, NI = T::NI, W = BODE_TRAJ_STRIDE(D);
  const int H = A.H;
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char smraw[];
  double* kk = reinterpret_cast<double*>(smraw);  // [S][D] stage derivatives
  double* kb = kk + S * D;                           // [S][D] their adjoints
  double* yv = kb + S * D;                           // [D] y_old
  double* yb = yv + D;                               // [D] running dL/dy_old
  double* ab = yb + D;                               // [D] dL/dy_next
  float* W1p = reinterpret_cast<float*>(ab + D);    // [H][D+1]
  float* W2p = W1p + kThreads * (D + 1);             // [D][H+1]
  float* Hs = W2p + D * (kThreads + 1);              // [S][256] tanh activations
  float* Yf = Hs + S * kThreads;                     // [S][D] fp32 stage inputs
  float* Pp = Yf + S * D;                            // [4][64] partial sums
  float* gf = Pp + 4 * 64;                           // [64] fp32 stage adjoint
  float* Vs = gf + 64;                               // [256] tanh' * W2^T g
  __shared__ int64_t s_inst;
  __shared__ double s_rec[3];

  for (int e = tid; e < H * D; e += kThreads) {
    const int j = e / D, c = e % D;
    W1p[j * (D + 1) + c] = A.W1[e];
    const int o = e / H, jj = e % H;
    W2p[o * (kThreads + 1) + jj] = A.W2[e];
  }
  const bool own_j = tid < H, own_c = tid < D;
  const float b1j = own_j ? A.b1[tid] : 0.0f;
  const float b2c = own_c ? A.b2[tid] : 0.0f;
  float gW1[D], gW2[D], gb1 = 0.0f, gb2 = 0.0f;
#pragma unroll
  for (int c = 0; c < D; c++) gW1[c] = gW2[c] = 0.0f;
  const int po = tid & 63, part = tid >> 6, jp = (H + 3) / 4;
  const int j_lo = part * jp, j_hi = min(H, j_lo + jp);
  __syncthreads();

  while (true) {
    if (tid == 0) {
      const unsigned long long q = atomicAdd(A.queue, 1ull);
      s_inst = q < (unsigned long long)A.n ? (A.order ? A.order[q] : (int64_t)q) : -1;
    }
    __syncthreads();
    const int64_t i = s_inst;
    if (i < 0) break;
    const double* te = A.t_eval_offsets ? A.t_eval + A.t_eval_offsets[i] : A.t_eval;
    const double* gy = A.t_eval_offsets ? A.grad_ys + A.t_eval_offsets[i] * D
                                        : A.grad_ys + i * A.t_eval_len * D;
    const int64_t r0 = A.traj_offsets[i], nrec = A.traj_offsets[i + 1] - r0;
    int64_t hi = A.n_emitted[i];
    if (own_c) ab[tid] = 0.0;
    for (int64_t r = nrec - 1; r >= 0; r--) {
      const double* rec = A.traj + (r0 + r) * W;
      if (tid < 3) s_rec[tid] = rec[tid];
      if (own_c) yv[tid] = rec[kTrajExtra + tid];
      __syncthreads();
      const double t = s_rec[0], h = s_rec[1];
      const int64_t lo = (int64_t)s_rec[2];
      (void)t;  // autonomous dynamics
      // ---- forward recompute of the step: Yf[s], Hs[s], kk[s]
      for (int s = 0; s < S; s++) {
        if (own_c) {
          double acc = 0.0;
          if (s > 0) {
            acc = T::a(s, 0) * kk[tid];
            for (int j = 1; j < s; j++) acc = fma(T::a(s, j), kk[j * D + tid], acc);
          }
          Yf[s * D + tid] = (float)(s > 0 ? fma(h, acc, yv[tid]) : yv[tid]);
        }
        __syncthreads();
        if (own_j) {
          float z = b1j;
          const float* w = W1p + tid * (D + 1);
          const float* yf = Yf + s * D;
#pragma unroll 16
          for (int c = 0; c < D; c++) z = fmaf(w[c], yf[c], z);
          Hs[s * kThreads + tid] = tanhf(z);
        }
        __syncthreads();
        if (po < D) {
          float acc = 0.0f;
          const float* w = W2p + po * (kThreads + 1);
          const float* hs = Hs + s * kThreads;
          for (int j = j_lo; j < j_hi; j++) acc = fmaf(w[j], hs[j], acc);
          Pp[part * 64 + po] = acc;
        }
        __syncthreads();
        if (own_c)
          kk[s * D + tid] = (double)(((Pp[tid] + Pp[64 + tid]) + (Pp[128 + tid] + Pp[192 + tid])) + b2c);
        __syncthreads();
      }
      // ---- seeds: y_next = y + h sum b_s k_s and the points of this step
      if (own_c) {
        const double a0 = ab[tid];
        double y_b = a0;
#pragma unroll
        for (int s = 0; s < S; s++) kb[s * D + tid] = (h * T::b(s)) * a0;
        for (int64_t p = lo; p < hi; p++) {
          double theta = ddiv(te[p] - s_rec[0], h);
          theta = np_max(theta, 0.0);
          const double g = gy[p * D + tid];
          y_b += g;
#pragma unroll
          for (int s = 0; s < S; s++) {
            double v = T::w(s, NI - 1);
#pragma unroll
            for (int j = NI - 2; j >= 0; j--) v = fma(v, theta, T::w(s, j));
            kb[s * D + tid] = fma(h * (v * theta), g, kb[s * D + tid]);
          }
        }
        yb[tid] = y_b;
      }
      hi = lo;
      __syncthreads();
      // ---- reverse sweep through the stages
      for (int s = S - 1; s >= 0; s--) {
        if (own_c) {
          const float g = (float)kb[s * D + tid];
          gf[tid] = g;
          gb2 += g;
        }
        __syncthreads();
        if (own_j) {
          float u = 0.0f;
          const float* w = W2p + tid;
#pragma unroll 16
          for (int o = 0; o < D; o++) u = fmaf(w[o * (kThreads + 1)], gf[o], u);
          const float hj = Hs[s * kThreads + tid];
          const float v = u * (1.0f - hj * hj);
          Vs[tid] = v;
          gb1 += v;
          const float* yf = Yf + s * D;
#pragma unroll
          for (int c = 0; c < D; c++) {
            gW1[c] = fmaf(v, yf[c], gW1[c]);
            gW2[c] = fmaf(gf[c], hj, gW2[c]);
          }
        }
        __syncthreads();
        if (po < D) {
          float acc = 0.0f;
          for (int j = j_lo; j < j_hi; j++) acc = fmaf(W1p[j * (D + 1) + po], Vs[j], acc);
          Pp[part * 64 + po] = acc;
        }
        __syncthreads();
        if (own_c) {
          const double Yb = (double)((Pp[tid] + Pp[64 + tid]) + (Pp[128 + tid] + Pp[192 + tid]));
          yb[tid] += Yb;
          for (int j = 0; j < s; j++)
            if (T::za(s, j) != 0.0) kb[j * D + tid] = fma(h * T::a(s, j), Yb, kb[j * D + tid]);
        }
        __syncthreads();
      }
      if (own_c) ab[tid] = yb[tid];
      __syncthreads();
    }
    if (own_c) {
      double a0 = ab[tid];
      for (int64_t p = 0; p < hi; p++) a0 += gy[p * D + tid];  // points at t_start
      A.grad_y0[i * D + tid] = a0;
    }
    if (A.grad_params && tid < 8) A.grad_params[i * 8 + tid] = 0.0;
    __syncthreads();
  }
  // per-CTA partial weight gradients: [dW1 (H,D) | dW2 (D,H) | db1 (H) | db2 (D)]
  float* out = A.mlp_part + (size_t)blockIdx.x * (2 * D * H + H + D);
  if (own_j) {
#pragma unroll
    for (int c = 0; c < D; c++) {
      out[tid * D + c] = gW1[c];
      out[D * H + c * H + tid] = gW2[c];
    }
    out[2 * D * H + tid] = gb1;
  }
  if (own_c) out[2 * D * H + H + tid] = gb2;
}

__global__ void mlp_grad_reduce_kernel(const float* part, int blocks, int D, int H, float* gW1,
                                       float* gb1, float* gW2, float* gb2) {
  const int len = 2 * D * H + H + D;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < blocks; b++) s += (double)part[(size_t)b * len + e];
    const float v = (float)s;
    if (e < D * H) {
      if (gW1) gW1[e] = v;
    } else if (e < 2 * D * H) {
      if (gW2) gW2[e - D * H] = v;
    } else if (e < 2 * D * H + H) {
      if (gb1) gb1[e - 2 * D * H] = v;
    } else if (gb2) {
      gb2[e - 2 * D * H - H] = v;
    }
  }
}

template <int M, int D>
cudaError_t launch_mlp_adjoint(const AdjParams& A, int blocks, cudaStream_t st) {
  auto kern = mlp_adjoint_kernel<M, D>;
  const size_t smem = mlp_adj_smem<D>(Tab<M>::S);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<blocks, kThreads, smem, st>>>(A);
  return cudaGetLastError();
}

template <int M>
cudaError_t dispatch_mlp_adjoint(int64_t d, const AdjParams& A, int blocks, cudaStream_t st) {
  switch (d) {
    case 4: return launch_mlp_adjoint<M, 4>(A, blocks, st);
    case 8: return launch_mlp_adjoint<M, 8>(A, blocks, st);
    case 16: return launch_mlp_adjoint<M, 16>(A, blocks, st);
    case 32: return launch_mlp_adjoint<M, 32>(A, blocks, st);
    case 64: return launch_mlp_adjoint<M, 64>(A, blocks, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

int mlp_adjoint_blocks() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

size_t mlp_adjoint_part_bytes(int64_t d, int64_t H) {
  return 4 * (size_t)mlp_adjoint_blocks() * (size_t)(2 * d * H + H + d);
}

cudaError_t mlp_adjoint_run(int method, int64_t d, AdjParams A, cudaStream_t st, int64_t* launches) {
  if (A.H < 1 || A.H > kThreads) return cudaErrorNotSupported;
  const int blocks = mlp_adjoint_blocks();
  cudaError_t e;
  switch (method) {
    case BODE_METHOD_DOPRI5: e = dispatch_mlp_adjoint<BODE_METHOD_DOPRI5>(d, A, blocks, st); break;
    case BODE_METHOD_TSIT5: e = dispatch_mlp_adjoint<BODE_METHOD_TSIT5>(d, A, blocks, st); break;
    default: e = dispatch_mlp_adjoint<BODE_METHOD_HEUN>(d, A, blocks, st); break;
  }
  if (e != cudaSuccess) return e;
  mlp_grad_reduce_kernel<<<64, 256, 0, st>>>(A.mlp_part, blocks, (int)d, (int)A.H, A.gW1, A.gb1,
                                             A.gW2, A.gb2);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace bode
