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
// One CTA (256 threads) reverses kRows instances at a time in lockstep
// (consecutive entries of the longest-first queue, so their trajectory
// lengths match); thread j owns hidden unit j for all rows, thread
// (r, c) < kRows*D row r's state component c.  Every weight read from
// shared memory serves the kRows rows.
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
constexpr int kRows = 4;  // instances reversed together by one CTA

// weight rows padded by 4 floats: 16-byte aligned rows for float4 reads
// along a row, and conflict-free (row stride = 4 banks) for both row- and
// column-wise access
constexpr int kPad = 4;

template <int D>
constexpr size_t mlp_adj_smem(int S) {
  return 8 * ((size_t)2 * S * kRows * D + 3 * kRows * D + 4 * kRows) +
         4 * ((size_t)kThreads * (D + kPad) + (size_t)D * (kThreads + kPad) +
              (size_t)S * kRows * kThreads + (size_t)S * kRows * D + kRows * 4 * 64 +
              kRows * 64 + kRows * kThreads) + 64;
}

// Rows r < kRows of a CTA are kRows consecutive instances of the
// longest-first queue, reversed in lockstep (iteration `it` reverses each
// row's (nrec - 1 - it)-th step; a row whose trajectory is exhausted is
// inactive and contributes exactly zero: its stage adjoints are zero).
template <int M, int D>
__global__ void __launch_bounds__(kThreads, 1) mlp_adjoint_kernel(const AdjParams A) {
  using T = Tab<M>;
  constexpr int S = T::S, NI = T::NI, W = BODE_TRAJ_STRIDE(D), R = kRows;
  const int H = A.H;
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char smraw[];
  double* kk = reinterpret_cast<double*>(smraw);  // [S][R][D] stage derivatives
  double* kb = kk + S * R * D;                       // [S][R][D] their adjoints
  double* yv = kb + S * R * D;                       // [R][D] y_old
  double* yb = yv + R * D;                           // [R][D] running dL/dy_old
  double* ab = yb + R * D;                           // [R][D] dL/dy_next
  double* rs = ab + R * D;                           // [R][4] t_old, h, lo, active
  constexpr int L1 = D + kPad, L2 = kThreads + kPad;  // padded row lengths
  float* W1p = reinterpret_cast<float*>(rs + 4 * R);  // [H][L1]
  float* W2p = W1p + kThreads * L1;                  // [D][L2]
  float* Hs = W2p + D * L2;                          // [S][R][256] tanh activations
  float* Yf = Hs + S * R * kThreads;                 // [S][R][D] fp32 stage inputs
  float* Pp = Yf + S * R * D;                        // [R][4][64] partial sums
  float* gf = Pp + R * 4 * 64;                       // [R][64] fp32 stage adjoint
  float* Vs = gf + R * 64;                           // [R][256]
  __shared__ int64_t s_inst[R], s_nrec[R], s_r0[R], s_hi[R];
  __shared__ int64_t s_it;

  for (int e = tid; e < H * D; e += kThreads) {
    const int j = e / D, c = e % D;
    W1p[j * L1 + c] = A.W1[e];
    const int o = e / H, jj = e % H;
    W2p[o * L2 + jj] = A.W2[e];
  }
  const bool own_j = tid < H;
  const int er = tid / D, ec = tid % D;  // (row, component) of this thread
  const bool own_e = tid < R * D;
  const float b1j = own_j ? A.b1[tid] : 0.0f;
  const float b2c = own_e ? A.b2[ec] : 0.0f;
  float gW1[D], gW2[D], gb1 = 0.0f, gb2 = 0.0f;
#pragma unroll
  for (int c = 0; c < D; c++) gW1[c] = gW2[c] = 0.0f;
  const int po = tid & 63, part = tid >> 6, jp = (H + 3) / 4;
  const int j_lo = part * jp, j_hi = min(H, j_lo + jp);
  __syncthreads();

  while (true) {
    if (tid == 0) {
      const unsigned long long q = atomicAdd(A.queue, (unsigned long long)R);
      int64_t mx = -1;
      for (int r = 0; r < R; r++) {
        const int64_t i = q + r < (unsigned long long)A.n ? (A.order ? A.order[q + r] : (int64_t)(q + r)) : -1;
        s_inst[r] = i;
        s_r0[r] = i >= 0 ? A.traj_offsets[i] : 0;
        s_nrec[r] = i >= 0 ? A.traj_offsets[i + 1] - s_r0[r] : -1;
        s_hi[r] = i >= 0 ? A.n_emitted[i] : 0;
        mx = s_nrec[r] > mx ? s_nrec[r] : mx;
      }
      s_it = q < (unsigned long long)A.n ? mx : -1;
    }
    __syncthreads();
    const int64_t iters = s_it;
    if (iters < 0) break;
    if (own_e) ab[tid] = 0.0;
    for (int64_t it = 0; it < iters; it++) {
      // ---- load this iteration's record of every active row
      if (tid < R) {
        const int64_t k = s_nrec[tid] - 1 - it;
        double* q = rs + 4 * tid;
        if (k >= 0) {
          const double* rec = A.traj + (s_r0[tid] + k) * W;
          q[0] = rec[0];
          q[1] = rec[1];
          q[2] = rec[2];
          q[3] = 1.0;
        } else {
          q[0] = q[1] = q[2] = 0.0;
          q[3] = 0.0;
        }
      }
      __syncthreads();
      const bool act_e = own_e && rs[4 * er + 3] != 0.0;
      const double h_e = own_e ? rs[4 * er + 1] : 0.0;
      if (own_e)
        yv[tid] = act_e ? A.traj[(s_r0[er] + s_nrec[er] - 1 - it) * W + kTrajExtra + ec] : 0.0;
      __syncthreads();
      // ---- forward recompute: Yf[s], Hs[s], kk[s] for all rows
      for (int s = 0; s < S; s++) {
        if (own_e) {
          double acc = 0.0;
          if (s > 0) {
            acc = T::a(s, 0) * kk[tid];
            for (int j = 1; j < s; j++) acc = fma(T::a(s, j), kk[(j * R) * D + tid], acc);
          }
          Yf[(s * R) * D + tid] = (float)(s > 0 ? fma(h_e, acc, yv[tid]) : yv[tid]);
        }
        __syncthreads();
        if (own_j) {
          float z[R];
#pragma unroll
          for (int r = 0; r < R; r++) z[r] = b1j;
          const float4* w = reinterpret_cast<const float4*>(W1p + tid * L1);
          const float* yf = Yf + (s * R) * D;
#pragma unroll 4
          for (int c4 = 0; c4 < D / 4; c4++) {
            const float4 wc = w[c4];
#pragma unroll
            for (int r = 0; r < R; r++) {
              const float4 y4 = reinterpret_cast<const float4*>(yf + r * D)[c4];
              z[r] = fmaf(wc.x, y4.x, fmaf(wc.y, y4.y, fmaf(wc.z, y4.z, fmaf(wc.w, y4.w, z[r]))));
            }
          }
#pragma unroll
          for (int r = 0; r < R; r++) Hs[(s * R + r) * kThreads + tid] = tanhf(z[r]);
        }
        __syncthreads();
        if (po < D) {
          float acc[R];
#pragma unroll
          for (int r = 0; r < R; r++) acc[r] = 0.0f;
          const float* w = W2p + po * L2;
          const float* hs = Hs + (s * R) * kThreads;
          for (int j = j_lo; j < j_hi; j += 4) {
            const float4 w4 = *reinterpret_cast<const float4*>(w + j);
#pragma unroll
            for (int r = 0; r < R; r++) {
              const float4 h4 = *reinterpret_cast<const float4*>(hs + r * kThreads + j);
              acc[r] = fmaf(w4.x, h4.x, fmaf(w4.y, h4.y, fmaf(w4.z, h4.z, fmaf(w4.w, h4.w, acc[r]))));
            }
          }
#pragma unroll
          for (int r = 0; r < R; r++) Pp[(r * 4 + part) * 64 + po] = acc[r];
        }
        __syncthreads();
        if (own_e) {
          const float* pp = Pp + er * 256 + ec;
          kk[(s * R) * D + tid] = (double)(((pp[0] + pp[64]) + (pp[128] + pp[192])) + b2c);
        }
        __syncthreads();
      }
      // ---- seeds: y_next = y + h sum b_s k_s and the points of this step
      if (own_e) {
        const double a0 = act_e ? ab[tid] : 0.0;
        double y_b = a0;
#pragma unroll
        for (int s = 0; s < S; s++) kb[(s * R) * D + tid] = (h_e * T::b(s)) * a0;
        if (act_e) {
          const int64_t i = s_inst[er];
          const double* te = A.t_eval_offsets ? A.t_eval + A.t_eval_offsets[i] : A.t_eval;
          const double* gy = A.t_eval_offsets ? A.grad_ys + A.t_eval_offsets[i] * D
                                              : A.grad_ys + i * A.t_eval_len * D;
          const double t_old = rs[4 * er];
          const int64_t lo = (int64_t)rs[4 * er + 2];
          for (int64_t p = lo; p < s_hi[er]; p++) {
            double theta = ddiv(te[p] - t_old, h_e);
            theta = np_max(theta, 0.0);
            const double g = gy[p * D + ec];
            y_b += g;
#pragma unroll
            for (int s = 0; s < S; s++) {
              double v = T::w(s, NI - 1);
#pragma unroll
              for (int j = NI - 2; j >= 0; j--) v = fma(v, theta, T::w(s, j));
              kb[(s * R) * D + tid] = fma(h_e * (v * theta), g, kb[(s * R) * D + tid]);
            }
          }
        }
        yb[tid] = y_b;
      }
      __syncthreads();
      if (tid < R && rs[4 * tid + 3] != 0.0) s_hi[tid] = (int64_t)rs[4 * tid + 2];
      // ---- reverse sweep through the stages
      for (int s = S - 1; s >= 0; s--) {
        if (own_e) {
          const float g = (float)kb[(s * R) * D + tid];
          gf[er * 64 + ec] = g;
          gb2 += g;
        }
        __syncthreads();
        if (own_j) {
          float u[R];
#pragma unroll
          for (int r = 0; r < R; r++) u[r] = 0.0f;
          const float* w = W2p + tid;
#pragma unroll 4
          for (int o4 = 0; o4 < D / 4; o4++) {
            const float w0 = w[(4 * o4) * L2], w1 = w[(4 * o4 + 1) * L2];
            const float w2 = w[(4 * o4 + 2) * L2], w3 = w[(4 * o4 + 3) * L2];
#pragma unroll
            for (int r = 0; r < R; r++) {
              const float4 g4 = reinterpret_cast<const float4*>(gf + r * 64)[o4];
              u[r] = fmaf(w0, g4.x, fmaf(w1, g4.y, fmaf(w2, g4.z, fmaf(w3, g4.w, u[r]))));
            }
          }
          float v[R], hj[R];
#pragma unroll
          for (int r = 0; r < R; r++) {
            hj[r] = Hs[(s * R + r) * kThreads + tid];
            v[r] = u[r] * (1.0f - hj[r] * hj[r]);
            Vs[r * kThreads + tid] = v[r];
            gb1 += v[r];
          }
          const float* yf = Yf + (s * R) * D;
#pragma unroll
          for (int c4 = 0; c4 < D / 4; c4++) {
#pragma unroll
            for (int r = 0; r < R; r++) {
              const float4 y4 = reinterpret_cast<const float4*>(yf + r * D)[c4];
              const float4 g4 = reinterpret_cast<const float4*>(gf + r * 64)[c4];
              gW1[4 * c4] = fmaf(v[r], y4.x, gW1[4 * c4]);
              gW1[4 * c4 + 1] = fmaf(v[r], y4.y, gW1[4 * c4 + 1]);
              gW1[4 * c4 + 2] = fmaf(v[r], y4.z, gW1[4 * c4 + 2]);
              gW1[4 * c4 + 3] = fmaf(v[r], y4.w, gW1[4 * c4 + 3]);
              gW2[4 * c4] = fmaf(g4.x, hj[r], gW2[4 * c4]);
              gW2[4 * c4 + 1] = fmaf(g4.y, hj[r], gW2[4 * c4 + 1]);
              gW2[4 * c4 + 2] = fmaf(g4.z, hj[r], gW2[4 * c4 + 2]);
              gW2[4 * c4 + 3] = fmaf(g4.w, hj[r], gW2[4 * c4 + 3]);
            }
          }
        }
        __syncthreads();
        if (po < D) {
          float acc[R];
#pragma unroll
          for (int r = 0; r < R; r++) acc[r] = 0.0f;
          for (int j = j_lo; j < j_hi; j += 4) {
            const float w0 = W1p[j * L1 + po], w1 = W1p[(j + 1) * L1 + po];
            const float w2 = W1p[(j + 2) * L1 + po], w3 = W1p[(j + 3) * L1 + po];
#pragma unroll
            for (int r = 0; r < R; r++) {
              const float4 v4 = *reinterpret_cast<const float4*>(Vs + r * kThreads + j);
              acc[r] = fmaf(w0, v4.x, fmaf(w1, v4.y, fmaf(w2, v4.z, fmaf(w3, v4.w, acc[r]))));
            }
          }
#pragma unroll
          for (int r = 0; r < R; r++) Pp[(r * 4 + part) * 64 + po] = acc[r];
        }
        __syncthreads();
        if (own_e) {
          const float* pp = Pp + er * 256 + ec;
          const double Yb = (double)((pp[0] + pp[64]) + (pp[128] + pp[192]));
          yb[tid] += Yb;
          for (int j = 0; j < s; j++)
            if (T::za(s, j) != 0.0) kb[(j * R) * D + tid] = fma(h_e * T::a(s, j), Yb, kb[(j * R) * D + tid]);
        }
        __syncthreads();
      }
      if (act_e) ab[tid] = yb[tid];
      __syncthreads();
    }
    if (own_e && s_inst[er] >= 0) {
      const int64_t i = s_inst[er];
      const double* gy = A.t_eval_offsets ? A.grad_ys + A.t_eval_offsets[i] * D
                                          : A.grad_ys + i * A.t_eval_len * D;
      double a0 = ab[tid];
      for (int64_t p = 0; p < s_hi[er]; p++) a0 += gy[p * D + ec];  // points at t_start
      A.grad_y0[i * D + ec] = a0;
    }
    __syncthreads();
  }
  // per-CTA partial weight gradients: [dW1 (H,D) | dW2 (D,H) | db1 (H) | db2 (D)]
  // (gb2 partials of the R row-threads of a component are summed through smem)
  float* red = Pp;
  if (own_e) red[tid] = gb2;
  __syncthreads();
  float* out = A.mlp_part + (size_t)blockIdx.x * (2 * D * H + H + D);
  if (own_j) {
#pragma unroll
    for (int c = 0; c < D; c++) {
      out[tid * D + c] = gW1[c];
      out[D * H + c * H + tid] = gW2[c];
    }
    out[2 * D * H + tid] = gb1;
  }
  if (tid < D) {
    float sb = 0.0f;
    for (int r = 0; r < R; r++) sb += red[r * D + tid];
    out[2 * D * H + H + tid] = sb;
  }
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
