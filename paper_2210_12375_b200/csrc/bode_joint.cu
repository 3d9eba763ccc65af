// bode_joint.cu -- solve_joint (solver.py:372-427) on the GPU: launchers of
// the single-CTA kernel in bode_joint_dev.cuh for the registered functors.
#include "bode_joint.cuh"
#include "bode_joint_dev.cuh"
#include "bode_program_host.cuh"

namespace bode {
namespace {

template <int M, class O, class F>
cudaError_t joint_launch(const SolveParams& P, const JointWs& W, cudaStream_t st) {
  bode_joint_kernel<M, F, O><<<1, kJT, 0, st>>>(P, W);
  return cudaGetLastError();
}

template <int M, class O>
cudaError_t joint_dispatch_ops(int kind, int64_t d, const SolveParams& P, const JointWs& W,
                               cudaStream_t st) {
  switch (kind) {
    case BODE_DYN_VDP:
      return d == 2 ? joint_launch<M, O, VdP<O>>(P, W, st) : cudaErrorInvalidValue;
    case BODE_DYN_LORENZ:
      return d == 3 ? joint_launch<M, O, Lorenz<O>>(P, W, st) : cudaErrorInvalidValue;
    case BODE_DYN_HARMONIC:
      return d == 2 ? joint_launch<M, O, Harmonic<O>>(P, W, st) : cudaErrorInvalidValue;
    case BODE_DYN_DAMPED:
      return d == 2 ? joint_launch<M, O, Damped<O>>(P, W, st) : cudaErrorInvalidValue;
    default:
      switch (d) {
        case 1: return joint_launch<M, O, Elementwise<O, 1>>(P, W, st);
        case 2: return joint_launch<M, O, Elementwise<O, 2>>(P, W, st);
        case 3: return joint_launch<M, O, Elementwise<O, 3>>(P, W, st);
        case 4: return joint_launch<M, O, Elementwise<O, 4>>(P, W, st);
        default: return cudaErrorNotSupported;
      }
  }
}

template <int M>
cudaError_t joint_dispatch(int mode, int kind, int64_t d, const SolveParams& P, const JointWs& W,
                           cudaStream_t st) {
  return mode == BODE_MODE_FAST ? joint_dispatch_ops<M, FastOps>(kind, d, P, W, st)
                                : joint_dispatch_ops<M, ExactOps>(kind, d, P, W, st);
}

size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace

size_t joint_workspace_bytes(int64_t n, int64_t d, int stages) {
  const size_t N = (size_t)(n * d), S = (size_t)stages;
  return a256(8 * N) * 3 + a256(8 * N * S) + a256(8 * (N / 64 + 2)) * 2;
}

cudaError_t joint_solve(int method, int mode, int kind, int64_t d, SolveParams P, char* ws,
                        int64_t* n_f_evals, cudaStream_t st, const bode_program* prog,
                        int stages) {
  const size_t N = (size_t)(P.n * d), S = (size_t)stages;
  JointWs W;
  char* p = ws;
  W.y = (double*)p;
  p += a256(8 * N);
  W.yn = (double*)p;
  p += a256(8 * N);
  W.sq = (double*)p;
  p += a256(8 * N);
  W.k = (double*)p;
  p += a256(8 * N * S);
  W.leaf_off = (int64_t*)p;
  p += a256(8 * (N / 64 + 2));
  W.leaf_sum = (double*)p;
  W.n_f_evals = n_f_evals;
  cudaError_t e;
  if (prog) return program_joint(prog, mode, P, W, st);
  switch (method) {
    case BODE_METHOD_DOPRI5: e = joint_dispatch<BODE_METHOD_DOPRI5>(mode, kind, d, P, W, st); break;
    case BODE_METHOD_TSIT5: e = joint_dispatch<BODE_METHOD_TSIT5>(mode, kind, d, P, W, st); break;
    default: e = joint_dispatch<BODE_METHOD_HEUN>(mode, kind, d, P, W, st); break;
  }
  return e;
}

}  // namespace bode
