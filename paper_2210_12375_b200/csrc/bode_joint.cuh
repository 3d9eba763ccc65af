// bode_joint.cuh -- solve_joint (solver.py:372-427) on the GPU (bode_joint.cu).
#pragma once
#include "bode_solver.cuh"

namespace bode {
size_t joint_workspace_bytes(int64_t n, int64_t d, int stages);
// one single-CTA launch: the whole batch as one problem of size n*d; P.ys is
// the shared-t_eval dense layout (n, t_eval_len, d); scalar tolerances
cudaError_t joint_solve(int method, int mode, int kind, int64_t d, SolveParams P, char* ws,
                        int64_t* n_f_evals, cudaStream_t st, const bode_program* prog = nullptr,
                        int stages = 7);
}  // namespace bode
