// bode_joint_dev.cuh -- the solve_joint kernel (device templates, shared by
// bode_joint.cu and run-time programs).
//
// The reference's pathology mode integrates the whole batch as ONE problem
// of size N = n*d: one RMS error norm over all N components (NumPy's
// pairwise summation over the flattened row), one shared step size, one
// accept decision, one trajectory whose statistics are replicated per
// instance.  It exists to show what independent solving avoids.
//
// One CTA runs the whole loop: each thread owns whole instances (their
// dynamics need all d components) for the stage evaluations, y_next / err,
// commit and dense output; the norm is a block reduction that reproduces
// NumPy's pairwise_sum tree exactly -- leaves of <= 128 elements (8
// accumulators) summed in parallel, then combined in the recursion's order
// by one thread; the controller, statuses and counters are scalar (thread
// 0).  Bit-identical to the reference in exact mode (tests/test_gpu_joint.py
// against fixtures produced by batchode.solve_joint).

#pragma once
#include "bode_solver.cuh"

namespace bode {

constexpr int kJT = 512;  // threads of the single CTA

// NumPy's pairwise_sum recursion (numpy/_core/src/umath/loops_utils.h.src):
// n <= 128 is a leaf; otherwise split at n/2 rounded down to a multiple of 8
__device__ inline void jt_build_leaves(int64_t off, int64_t n, int64_t* leaf_off, int32_t* nl) {
  if (n <= 128) {
    leaf_off[(*nl)++] = off;
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  jt_build_leaves(off, n2, leaf_off, nl);
  jt_build_leaves(off + n2, n - n2, leaf_off, nl);
}

__device__ inline double jt_combine(int64_t n, const double* leaf_sum, int32_t* li) {
  if (n <= 128) return leaf_sum[(*li)++];
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const double a = jt_combine(n2, leaf_sum, li);
  const double b = jt_combine(n - n2, leaf_sum, li);
  return __dadd_rn(a, b);
}

struct JointWs {
  double* y;         // (N) state
  double* k;         // (S, N) stage derivatives
  double* yn;        // (N) y_next / Euler probe state
  double* sq;        // (N) squared scaled errors
  int64_t* leaf_off; // pairwise leaves
  double* leaf_sum;
  int64_t* n_f_evals;
};

// sqrt(mean(sq[0..N))) in NumPy order; all threads call it, the result is
// returned to every thread
__device__ inline double jt_rms(const JointWs& W, int64_t N, int32_t nl, double* s_bcast) {
  __syncthreads();
  for (int32_t l = threadIdx.x; l < nl; l += blockDim.x) {
    const int64_t a = W.leaf_off[l], b = l + 1 < nl ? W.leaf_off[l + 1] : N;
    W.leaf_sum[l] = pairwise_sum_rt<ExactOps>(W.sq + a, b - a);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t li = 0;
    const double s = jt_combine(N, W.leaf_sum, &li);
    *s_bcast = dsqrt(ddiv(s, (double)N));
  }
  __syncthreads();
  return *s_bcast;
}

template <int M, class F, class O>
__global__ void __launch_bounds__(kJT) bode_joint_kernel(const SolveParams P, const JointWs W) {
  using T = Tab<M>;
  constexpr int D = F::D, S = T::S;
  const int64_t n = P.n, N = n * D;
  const int tid = threadIdx.x;
  __shared__ double s_bc;
  __shared__ int32_t s_nl;

  const double atol = P.atol, rtol = P.rtol;  // scalar tolerances (solver.py:399-403)
  const double t0 = P.t_start[0], t_end = P.t_end[0];
  const double direction = (t_end - t0) > 0.0 ? 1.0 : -1.0;
  const int64_t m = P.t_eval_len;  // shared t_eval (solver.py:394-398)

  if (tid == 0) {
    int32_t nl = 0;
    jt_build_leaves(0, N, W.leaf_off, &nl);
    s_nl = nl;
  }
  // ---- init (BatchSolver.__init__ on the flat problem): y, f0
  bool bad = false;
  for (int64_t i = tid; i < n; i += blockDim.x) {
    F f;
    f.load(P.dyn, i);
    double y[D], f0[D];
#pragma unroll
    for (int c = 0; c < D; c++) y[c] = W.y[i * D + c] = P.y0[i * D + c];
    f(t0, y, f0);
#pragma unroll
    for (int c = 0; c < D; c++) {
      W.k[i * D + c] = f0[c];
      bad |= !isfinite(f0[c]);
    }
  }
  bad = __syncthreads_or(bad);
  const int32_t nl = s_nl;
  double dt;
  if (P.dt0_mode == BODE_DT0_HEURISTIC) {
    // initial_step (controller.py:145-197) over all N components
    for (int64_t j = tid; j < N; j += blockDim.x) {
      const double q = ddiv(W.y[j], ExactOps::mad(rtol, fabs(W.y[j]), atol));
      W.sq[j] = ExactOps::mul(q, q);
    }
    const double d0 = jt_rms(W, N, nl, &s_bc);
    for (int64_t j = tid; j < N; j += blockDim.x) {
      const double q = ddiv(W.k[j], ExactOps::mad(rtol, fabs(W.y[j]), atol));
      W.sq[j] = ExactOps::mul(q, q);
    }
    const double d1 = jt_rms(W, N, nl, &s_bc);
    const bool degenerate = (d0 < 1e-5) || (d1 < 1e-5) || !isfinite(d1);
    const double h0 = degenerate ? 1e-6 : ddiv(__dmul_rn(0.01, d0), d1);
    const double hd = __dmul_rn(h0, direction);
    for (int64_t i = tid; i < n; i += blockDim.x) {  // Euler probe f1 = f(t0 + hd, y0 + hd f0)
      F f;
      f.load(P.dyn, i);
      double y1[D], f1[D];
#pragma unroll
      for (int c = 0; c < D; c++) y1[c] = ExactOps::mad(hd, W.k[i * D + c], W.y[i * D + c]);
      f(__dadd_rn(t0, hd), y1, f1);
#pragma unroll
      for (int c = 0; c < D; c++) {
        const double q = ddiv(ExactOps::sub(f1[c], W.k[i * D + c]),
                              ExactOps::mad(rtol, fabs(W.y[i * D + c]), atol));
        W.sq[i * D + c] = ExactOps::mul(q, q);
      }
    }
    const double d2 = ddiv(jt_rms(W, N, nl, &s_bc), h0);
    const double dmax = np_max(d1, d2);
    const bool small = (dmax <= 1e-15) || !isfinite(dmax);
    const double h1 = small ? np_max(1e-6, __dmul_rn(h0, 1e-3))
                            : np_scalar_pow(ddiv(0.01, dmax), ddiv(1.0, (double)(T::ORDER + 1)));
    dt = __dmul_rn(np_min(__dmul_rn(100.0, h0), h1), direction);
  } else {
    dt = P.dt0;
  }
  if (bad) dt = __longlong_as_double(0x7ff8000000000000LL);
  int32_t status = BODE_RUNNING;
  if (!isfinite(dt)) {
    status = BODE_INFINITE_DYNAMICS;
    dt = 0.0;
  }
  // points at t_start: copies of y0
  int64_t cursor = 0;
  while (cursor < m && P.t_eval[cursor] == t0) {
    for (int64_t i = tid; i < n; i += blockDim.x)
#pragma unroll
      for (int c = 0; c < D; c++) P.ys[(i * m + cursor) * D + c] = W.y[i * D + c];
    cursor++;
  }

  // ---- the loop (step_once on the flat problem, solver.py:208-282)
  double t = t0, n1 = 1.0, n2 = 1.0;
  int64_t nsteps = 0, nacc = 0, refresh = 0;
  bool rejected_last = false;
  while (status == BODE_RUNNING) {
    const double remaining = ExactOps::sub(t_end, t);
    const bool trunc = fabs(dt) >= fabs(remaining);
    const double h = trunc ? remaining : dt;
    if (T::FSAL && rejected_last) refresh++;  // FSAL refresh evaluation (solver.py:220-226)
    for (int64_t i = tid; i < n; i += blockDim.x) {
      F f;
      f.load(P.dyn, i);
      double y[D], k[S][D], yn[D], err[D];
#pragma unroll
      for (int c = 0; c < D; c++) {
        y[c] = W.y[i * D + c];
        k[0][c] = W.k[i * D + c];
      }
      rk_step<T, F, O>(f, t, h, y, k, yn, err);
#pragma unroll
      for (int c = 0; c < D; c++) {
#pragma unroll
        for (int s = 1; s < S; s++) W.k[((int64_t)s * n + i) * D + c] = k[s][c];
        if (!T::FSAL) W.k[i * D + c] = k[0][c];
        W.yn[i * D + c] = yn[c];
        const double scale = O::mad(rtol, np_max(fabs(y[c]), fabs(yn[c])), atol);
        const double r = ddiv(err[c], scale);
        W.sq[i * D + c] = O::mul(r, r);
      }
    }
    double norm = jt_rms(W, N, nl, &s_bc);
    if (!isfinite(norm)) norm = __longlong_as_double(0x7ff0000000000000LL);
    double dtn = h;
    const bool accept = adapt(P.ctrl, norm, n1, n2, dtn);
    const int32_t j = (int32_t)nsteps;
    nsteps++;
    if (tid == 0 && P.trace_cap > 0 && j < P.trace_cap) {
      if (P.trace_t) P.trace_t[j] = t;
      if (P.trace_dt) P.trace_dt[j] = h;
      if (P.trace_accept) P.trace_accept[j] = accept;
    }
    if (accept) {
      nacc++;
      const double t_old = t;
      // dense output for the shared points crossed (solver.py:284-322)
      while (cursor < m && h != 0.0) {
        double theta = ddiv(ExactOps::sub(P.t_eval[cursor], t_old), h);
        if (!(theta <= 1.0)) break;
        theta = np_max(theta, 0.0);
        for (int64_t i = tid; i < n; i += blockDim.x) {
          double y[D], k[S][D], out[D];
#pragma unroll
          for (int c = 0; c < D; c++) {
            y[c] = W.y[i * D + c];
#pragma unroll
            for (int s = 0; s < S; s++) k[s][c] = W.k[((int64_t)s * n + i) * D + c];
          }
          interpolate<T, D, O>(k, y, h, theta, out);
#pragma unroll
          for (int c = 0; c < D; c++) P.ys[(i * m + cursor) * D + c] = out[c];
        }
        cursor++;
      }
      for (int64_t i = tid; i < n; i += blockDim.x) {
#pragma unroll
        for (int c = 0; c < D; c++) {
          W.y[i * D + c] = W.yn[i * D + c];
          if (T::FSAL) W.k[i * D + c] = W.k[((int64_t)(S - 1) * n + i) * D + c];
        }
      }
      t = trunc ? t_end : ExactOps::add(t_old, h);
      if (trunc) status = BODE_SUCCESS;
    }
    dt = dtn;
    if (status == BODE_RUNNING && ExactOps::add(t, dt) == t) status = BODE_STEP_UNDERFLOW;
    if (status == BODE_RUNNING && nsteps >= P.max_steps) status = BODE_MAX_STEPS_EXCEEDED;
    rejected_last = !accept && status == BODE_RUNNING;
    __syncthreads();  // commits visible before the next step's reads
  }
  // ---- outputs, replicated per instance (solver.py:415-427)
  for (int64_t i = tid; i < n; i += blockDim.x) {
    P.n_emitted[i] = cursor;
    P.n_steps[i] = nsteps;
    P.n_accepted[i] = nacc;
    P.final_dt[i] = dt;
    P.status[i] = status;
  }
  if (tid == 0)  // single-trajectory n_f_evals (solver.py:184,224,239)
    W.n_f_evals[0] = T::FSAL ? 1 + (S - 1) * nsteps + refresh : 1 + S * nsteps;
}

}  // namespace bode
