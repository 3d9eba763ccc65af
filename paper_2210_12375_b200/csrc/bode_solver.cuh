// bode_solver.cuh -- the persistent batched integrator (kernel K2).
//
// One lane (thread) owns one instance at a time and runs the reference's
// whole per-instance state machine to termination: FSAL stages, RK axpys,
// RMS error norm, PID update, accept/reject, t_end truncation, statuses,
// statistics and Horner dense output straight to ys.  This is the
// batch-independent restatement of the reference's lockstep loop
// (solver.py:148-322).  There is no per-step launch
// and no host sync: when a lane's instance terminates the warp pulls the
// next instance from a global queue (warp-aggregated atomicAdd), so lanes
// never idle on an "all done?" flag and step-count divergence costs only the
// tail.  The queue may be cost-sorted (longest first) by the caller.
//
// The batch-global n_f_evals (solver.py:184,224,239) is rebuilt exactly:
// every lane records "instance rejected at iteration j and still running"
// in a per-block shared-memory bitmap of iterations, blocks OR it into a
// global bitmap, and bode_finalize counts 1 + (S-1)*max n_steps + refreshes.
#pragma once
#include "bode_device.cuh"

namespace bode {

struct SolveParams {
  int64_t n;
  DynParams dyn;
  CtrlParams ctrl;
  const double* y0;
  const double* t_start;
  const double* t_end;
  const double* t_eval;
  const int64_t* t_eval_offsets;
  int64_t t_eval_len;
  const double* atol_v;
  const double* rtol_v;
  double atol, rtol;
  int64_t max_steps;
  int32_t dt0_mode;
  double dt0;
  const double* dt0_v;
  const int64_t* order;
  double* ys;
  int64_t* n_emitted;
  int64_t* n_steps;
  int64_t* n_accepted;
  double* final_dt;
  int64_t* status;
  double* trace_t;
  double* trace_dt;
  uint8_t* trace_accept;
  int64_t trace_cap;
  // optional accepted-step trajectory for the adjoint (bode_adjoint.cu):
  // row traj_offsets[i] + k = the k-th accepted step of instance i, laid out
  // as [t_old, h, cursor before the step, y_old[D], pad] (kTrajStride<D>)
  double* traj;
  const int64_t* traj_offsets;
  // workspace
  unsigned long long* queue;   // next instance position
  unsigned long long* max_n;   // max n_steps over the batch
  uint32_t* refresh;           // global bitmap over iterations
  int32_t smem_words;          // >0: per-block shared bitmap of this many words
  double* f0;                  // (n, D) FSAL seeds from the init pass
  double* te_next;             // (n) first pending output time from the init pass
  // optional: the init pass's resume records in QUEUE order (kRec* slots,
  // rec_stride doubles per position) -- a refill reads one contiguous
  // record at its queue position instead of gathering a dozen scattered
  // per-instance fields through the order permutation
  double* rec;
  int32_t rec_stride;
  const int64_t* rec_pos;      // queue position of instance i (NULL: i)
  void* ev_start;              // host side only: optional cudaEvent_t around
  void* ev_stop;               // the persistent launch (bench roofline)
};

// resume record slots (doubles; integers stored by bit pattern), then
// y0 (D), f0 (D) and the instance's per-instance parameters
enum : int { kRecT = 0, kRecTEnd, kRecDt, kRecTeNext, kRecIdx, kRecCursor, kRecM, kRecStatus,
             kRecTeOff, kRecY };
__host__ __device__ __forceinline__ int rec_stride(int64_t d, int n_inst) {
  return (int)((kRecY + 2 * d + n_inst + 3) / 4 * 4);
}

constexpr int kTrajExtra = BODE_TRAJ_EXTRA;
template <int D>
constexpr int kTrajStride = BODE_TRAJ_STRIDE(D);

struct Workspace {
  static constexpr size_t kHeader = 64;
  static size_t bitmap_words(int64_t max_steps) { return (size_t)((max_steps + 2 + 31) / 32); }
  static size_t bitmap_bytes(int64_t max_steps) { return (4 * bitmap_words(max_steps) + 255) & ~(size_t)255; }
  static size_t f0_offset(int64_t max_steps) { return kHeader + bitmap_bytes(max_steps); }
  static size_t bytes(int64_t max_steps, int64_t n, int64_t d) {
    return f0_offset(max_steps) + 8 * (size_t)n * (size_t)d;
  }
};

// a recording lane's trajectory rows (shared memory, set at refill)
struct TrajRows {
  double* base;
  double* end;
};

// per-lane output bases (t_eval row, ys row) kept in shared memory from
// the refill on, so a lane emitting a point does not stall its warp on a
// dependent offsets load
struct EmitBase {
  const double* te;
  double* ys;
};

template <int M, class F, class O>
struct Lane {
  using T = Tab<M>;
  static constexpr int D = F::D, S = T::S;
  F f;
  double y[D];
  double k[S][D];  // k[0] is the FSAL cache f0
  // Registers hold what every step touches: per-instance tolerances and the
  // t_eval / ys bases are re-derived from idx where used (scalar tolerances
  // stay uniform), the next output time is cached (te_next), counters are
  // 32-bit -- the 2-D kernels stay at 5 blocks / SM with few spills.
  double t, dt, t_end, n1, n2;
  double te_next;  // t_eval[cursor], cached: the per-step check needs no load
  LogCache L1;  // log(n1) for the PID history term (adapt_cached)
  int64_t idx;
  int32_t nsteps, nacc, cursor, m;
  int32_t status;

  __device__ __forceinline__ const double* te_of(const SolveParams& P) const {
    return P.t_eval_offsets ? P.t_eval + P.t_eval_offsets[idx] : P.t_eval;
  }
  __device__ __forceinline__ double* ys_of(const SolveParams& P) const {
    if (!P.ys) return nullptr;
    return P.t_eval_offsets ? P.ys + P.t_eval_offsets[idx] * D : P.ys + idx * P.t_eval_len * D;
  }

  __device__ __forceinline__ double atol_of(const SolveParams& P) const {
    return P.atol_v ? P.atol_v[idx] : P.atol;
  }
  __device__ __forceinline__ double rtol_of(const SolveParams& P) const {
    return P.rtol_v ? P.rtol_v[idx] : P.rtol;
  }

  __device__ __forceinline__ void load_problem(const SolveParams& P, int64_t i) {
    idx = i;
    f.load(P.dyn, i);
    t = P.t_start[i];
    t_end = P.t_end[i];
#pragma unroll
    for (int c = 0; c < D; c++) y[c] = P.y0[i * D + c];
    m = (int32_t)(P.t_eval_offsets ? P.t_eval_offsets[i + 1] - P.t_eval_offsets[i] : P.t_eval_len);
    n1 = 1.0;
    n2 = 1.0;
    nsteps = 0;
    nacc = 0;
  }

  // BatchSolver.__init__ for one row (solver.py:148-206): f0, dt0 and the
  // INFINITE_DYNAMICS check, then the points equal to t_start.  Runs in the
  // init pass (one non-divergent launch over the batch); its results go to
  // the output buffers (dt -> final_dt, cursor -> n_emitted, status) and the
  // f0 workspace, from which the persistent kernel resumes the row.
  __device__ __forceinline__ void initialize(const SolveParams& P, int64_t i) {
    load_problem(P, i);
    const double direction = (t_end - t) > 0.0 ? 1.0 : -1.0;
    if (P.dt0_mode == BODE_DT0_HEURISTIC) {
      dt = initial_step<F, O>(f, t, y, T::ORDER, atol_of(P), rtol_of(P), direction, k[0]);
    } else {
      dt = P.dt0_mode == BODE_DT0_SCALAR ? P.dt0 : P.dt0_v[i];
      f(t, y, k[0]);
      bool fin = true;
#pragma unroll
      for (int c = 0; c < D; c++) fin &= isfinite(k[0][c]);
      if (!fin) dt = __longlong_as_double(0x7ff8000000000000LL);
    }
    status = BODE_RUNNING;
    if (!isfinite(dt)) {
      status = BODE_INFINITE_DYNAMICS;
      dt = 0.0;
    }
    cursor = 0;
    const double* te = te_of(P);
    double* ys = ys_of(P);
    while (cursor < m && te[cursor] == t) {  // points at t_start: copies of y0
      if (ys) {
#pragma unroll
        for (int c = 0; c < D; c++) ys[cursor * D + c] = y[c];
      }
      cursor++;
    }
    if (status == BODE_RUNNING) {
      if (!P.rec) {
#pragma unroll
        for (int c = 0; c < D; c++) P.f0[i * D + c] = k[0][c];
        P.te_next[i] = cursor < m ? te[cursor] : 0.0;
      }
      P.final_dt[i] = dt;
      P.n_emitted[i] = cursor;
      P.status[i] = BODE_RUNNING;
    } else {
      finish(P);
    }
  }

  // the resume record of queue position pos (P.rec), after initialize():
  // assembled in registers and written as whole 32-byte sectors (256-bit
  // stores) -- the positions are scattered, partial-sector writes are not
  __device__ __forceinline__ void write_record(const SolveParams& P, int64_t pos) const {
    constexpr int NR = (kRecY + 2 * D + 8 + 3) / 4 * 4;  // (n_inst <= 8)
    double r[NR];
    const double* te = te_of(P);
    r[kRecT] = t;
    r[kRecTEnd] = t_end;
    r[kRecDt] = dt;
    r[kRecTeNext] = cursor < m ? te[cursor] : 0.0;
    r[kRecIdx] = __longlong_as_double(idx);
    r[kRecCursor] = __longlong_as_double((int64_t)cursor);
    r[kRecM] = __longlong_as_double((int64_t)m);
    r[kRecStatus] = __longlong_as_double((int64_t)status);
    r[kRecTeOff] = __longlong_as_double(P.t_eval_offsets ? P.t_eval_offsets[idx]
                                                         : idx * P.t_eval_len);
#pragma unroll
    for (int c = 0; c < D; c++) {
      r[kRecY + c] = y[c];
      r[kRecY + D + c] = k[0][c];
    }
#pragma unroll
    for (int q = 0; q < 8; q++)
      r[kRecY + 2 * D + q] = q < P.dyn.n_inst ? P.dyn.inst[idx * P.dyn.n_inst + q] : 0.0;
    double* dst = P.rec + pos * P.rec_stride;
#pragma unroll
    for (int q = 0; q < NR; q += 4)
      if (q < P.rec_stride) {
#ifdef __CUDACC_RTC__  // (run-time programs: the runtime NVRTC's PTX has no 256-bit vectors)
        reinterpret_cast<double2*>(dst + q)[0] = make_double2(r[q], r[q + 1]);
        reinterpret_cast<double2*>(dst + q)[1] = make_double2(r[q + 2], r[q + 3]);
#else
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + q), "d"(r[q]),
                     "d"(r[q + 1]), "d"(r[q + 2]), "d"(r[q + 3]) : "memory");
#endif
      }
  }

  // pick up the row of queue position pos from its record; returns the
  // row's t_eval / ys offset and status
  __device__ __forceinline__ int64_t resume_record(const SolveParams& P, int64_t pos,
                                                   int64_t& st) {
    const double* r = P.rec + pos * P.rec_stride;
    // every load at once: the record is 16-byte aligned (rec_stride % 4 == 0)
    constexpr int NV = (kRecY + 2 * D + 1) / 2;
    double2 v[NV];
#pragma unroll
    for (int q = 0; q < NV; q++) v[q] = reinterpret_cast<const double2*>(r)[q];
    const double* x = reinterpret_cast<const double*>(v);
    t = x[kRecT];
    t_end = x[kRecTEnd];
    dt = x[kRecDt];
    te_next = x[kRecTeNext];
    idx = __double_as_longlong(x[kRecIdx]);
    cursor = (int32_t)__double_as_longlong(x[kRecCursor]);
    m = (int32_t)__double_as_longlong(x[kRecM]);
    st = __double_as_longlong(x[kRecStatus]);
#pragma unroll
    for (int c = 0; c < D; c++) {
      y[c] = x[kRecY + c];
      k[0][c] = x[kRecY + D + c];
    }
    DynParams pr = P.dyn;  // per-instance parameters from the record (row 0)
    pr.inst = r + kRecY + 2 * D;
    f.load(pr, 0);
    n1 = 1.0;
    n2 = 1.0;
    nsteps = 0;
    nacc = 0;
    status = BODE_RUNNING;
    L1.ok = cr_log(1.0, g_pow_tables, L1.h, L1.l);  // log(1) = 0 exactly (both modes)
    return __double_as_longlong(x[kRecTeOff]);
  }

  // pick up a row prepared by the init pass
  __device__ __forceinline__ void resume(const SolveParams& P, int64_t i) {
    load_problem(P, i);
#pragma unroll
    for (int c = 0; c < D; c++) k[0][c] = P.f0[i * D + c];
    dt = P.final_dt[i];
    cursor = (int32_t)P.n_emitted[i];
    te_next = P.te_next[i];  // no load dependent on cursor
    status = BODE_RUNNING;
    L1.ok = cr_log(1.0, g_pow_tables, L1.h, L1.l);  // log(1) = 0 exactly (both modes)
  }

  // one iteration of step_once for this row (solver.py:208-282); returns
  // true when the row just rejected and is still running (FSAL refresh at
  // the next iteration, solver.py:220-226)
  // trec (recording only): shared-memory slot holding this lane's
  // trajectory rows [base, end), set at resume -- no per-step global load
  // PI (fast mode only): the launch was specialised for an I / PI
  // controller (CtrlParams::plain_pi), so the general controller is not
  // compiled into the loop
  // the arithmetic of one attempt: t_end truncation, the RK trial step, the
  // error norm and the controller (no memory traffic, no branches on the
  // fast I / PI path); commit() applies the decision
  // VT: the launch may carry per-instance tolerance vectors; false = the
  // caller passed scalars (atol_v == rtol_v == NULL), so the step loop keeps
  // no pointer tests or predicated loads for them
  template <bool PI, bool VT = true>
  __device__ __forceinline__ bool attempt(const SolveParams& P, const PowTables& PT, double* yn,
                                          double* err, double& dtn, double& h, bool& trunc) {
    const double remaining = O::sub(t_end, t);
    trunc = fabs(dt) >= fabs(remaining);
    h = trunc ? remaining : dt;
    rk_step<T, F, O>(f, t, h, y, k, yn, err);
    dtn = h;
    const double at = VT ? atol_of(P) : P.atol, rt = VT ? rtol_of(P) : P.rtol;
    if constexpr (O::kFast && PI) {
      return adapt_pi_ms(P.ctrl, error_ms<D, O>(err, y, yn, at, rt), L1, dtn, PT);
    } else {
      const double norm = error_norm<D, O>(err, y, yn, at, rt);
      return adapt_cached<O>(P.ctrl, norm, n1, n2, L1, dtn, PT);
    }
  }

  // the rest of step_once for this row: statistics, trace, dense output,
  // the masked commit and the statuses; returns true when the row just
  // rejected and is still running (FSAL refresh at the next iteration)
  __device__ __forceinline__ bool commit(const SolveParams& P, bool tracing, const TrajRows* trec,
                                         const EmitBase& eb, const double* yn, bool accept,
                                         double dtn, double h, bool trunc) {
    const int32_t j = nsteps;
    nsteps = j + 1;
    if (tracing && j < P.trace_cap) {
      const int64_t o = idx * P.trace_cap + j;  // (trace only)
      if (P.trace_t) P.trace_t[o] = t;
      if (P.trace_dt) P.trace_dt[o] = h;
      if (P.trace_accept) P.trace_accept[o] = accept;
    }
    if (accept) {
      if (trec) {  // (adjoint only) the pre-commit state of this step,
        // written as whole 32-byte sectors, one 256-bit store each
        double rec[kTrajStride<D>] = {t, h, (double)cursor};
#pragma unroll
        for (int c = 0; c < D; c++) rec[kTrajExtra + c] = y[c];
        double* r = trec->base + (int64_t)nacc * kTrajStride<D>;
        if (r < trec->end) {  // (the rows were sized by an identical solve)
#pragma unroll
          for (int q = 0; q < kTrajStride<D>; q += 4)
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(r + q), "d"(rec[q]),
                         "d"(rec[q + 1]), "d"(rec[q + 2]), "d"(rec[q + 3]) : "memory");
        }
      }
      nacc++;
      const double t_old = t;
      if (cursor < m && h != 0.0) {
        // theta = (t_eval[cursor] - t_old) / h is >= 0 (earlier points were
        // emitted); |t_eval[cursor] - t_old| > 2|h| means theta > 2, so the
        // exact division is only needed near a point
        const double diff = O::sub(te_next, t_old);
        if (!(fabs(diff) > 2.0 * fabs(h))) emit(eb, t_old, h);
      }
#pragma unroll
      for (int c = 0; c < D; c++) y[c] = yn[c];
      t = trunc ? t_end : O::add(t_old, h);
      if constexpr (T::FSAL) {
#pragma unroll
        for (int c = 0; c < D; c++) k[0][c] = k[S - 1][c];
      }
      if (trunc) status = BODE_SUCCESS;
    }
    dt = dtn;
    if (status == BODE_RUNNING && O::add(t, dt) == t) status = BODE_STEP_UNDERFLOW;
    if (status == BODE_RUNNING && nsteps >= (int32_t)P.max_steps)  // (max_steps < 2^31, bode_abi.cu)
      status = BODE_MAX_STEPS_EXCEEDED;
    return !accept && status == BODE_RUNNING;
  }

  // one iteration of step_once for this row (solver.py:208-282); returns
  // true when the row just rejected and is still running (FSAL refresh at
  // the next iteration, solver.py:220-226)
  // trec (recording only): shared-memory slot holding this lane's
  // trajectory rows [base, end), set at resume -- no per-step global load
  // PI (fast mode only): the launch was specialised for an I / PI
  // controller (CtrlParams::plain_pi), so the general controller is not
  // compiled into the loop
  template <bool PI, bool VT = true>
  __device__ __forceinline__ bool step(const SolveParams& P, const PowTables& PT, bool tracing,
                                       const TrajRows* trec, const EmitBase& eb) {
    double yn[D], err[D], dtn, h;
    bool trunc;
    const bool accept = attempt<PI, VT>(P, PT, yn, err, dtn, h, trunc);
    return commit(P, tracing, trec, eb, yn, accept, dtn, h, trunc);
  }

  // _emit, solver.py:284-322: every point with theta in (.., 1] is
  // interpolated from the pre-commit state (y is still y_old here)
  // Fast mode: one reciprocal per call (not an IEEE division per point --
  // the hottest stall of C3's kernel) and theta = diff / h as the product
  // refined by one residual step, i.e. the rounded quotient except at rare
  // near-ties; diff == h still gives theta == 1 exactly (a point at the end
  // of the step is emitted by this step).
  __device__ __forceinline__ void emit(const EmitBase& eb, double t_old, double h) {
    const double* te = eb.te;
    double* ys = eb.ys;
    const double rh = O::kFast ? fast_rcp(h) : 0.0;
    while (cursor < m) {
      const double diff = O::sub(te_next, t_old);
      double theta;
      if constexpr (O::kFast) {
        const double q = diff * rh;
        theta = fma(fma(-q, h, diff), rh, q);
      } else {
        theta = ddiv(diff, h);
      }
      if (!(theta <= 1.0)) break;
      theta = np_max(theta, 0.0);
      double out[D];
      interpolate<T, D, O>(k, y, h, theta, out);
      if (ys) {
        if (D == 2 && (reinterpret_cast<unsigned long long>(ys) & 15) == 0) {  // one 16-byte store
          reinterpret_cast<double2*>(ys)[cursor] = make_double2(out[0], out[D - 1]);
        } else {
#pragma unroll
          for (int c = 0; c < D; c++) ys[cursor * D + c] = out[c];
        }
      }
      cursor++;
      if (cursor < m) te_next = te[cursor];
    }
  }

  __device__ __forceinline__ void finish(const SolveParams& P) const {
    P.n_emitted[idx] = cursor;
    P.n_steps[idx] = nsteps;
    P.n_accepted[idx] = nacc;
    P.final_dt[idx] = dt;
    P.status[idx] = status;
  }
};

#ifdef BODE_EXIT_PROF
static __device__ unsigned long long g_exit_times[65536];
static __device__ unsigned g_exit_count;
#endif

// 2-D systems fit 5 blocks of 128 threads per SM (<= 102 registers); wider
// ones keep 4 (<= 128 registers) to avoid spilling the stage vectors.  The
// trajectory-recording instantiation (REC, gradients only) fits 5 blocks
// without spills only in the fast-mode I / PI specialisation; the general
// controller (exact mode, PID betas) spills at 96 registers, so those REC
// instantiations keep 4 blocks.
#ifndef BODE_BLOCKS_2D
#define BODE_BLOCKS_2D 5
#endif
#ifndef BODE_BLOCKS_WIDE
#define BODE_BLOCKS_WIDE 4
#endif
template <bool B>
struct BoolTag {  // (no <type_traits> under NVRTC)
  static constexpr bool value = B;
};
template <int M, class F, class O, bool REC, bool PI>
__global__ void __launch_bounds__(128, ((F::D <= 2 && (!REC || PI)) ? BODE_BLOCKS_2D : BODE_BLOCKS_WIDE)) bode_persistent_kernel(const SolveParams P) {
  extern __shared__ uint32_t s_refresh[];
  __shared__ PowTables s_pow;  // pow tables: divergent lookups, so shared not constant
  const int lane = threadIdx.x & 31;
  for (int w = threadIdx.x; w < P.smem_words; w += blockDim.x) s_refresh[w] = 0u;
  {
    const double* src = &g_pow_tables.log_tab[0][0];
    double* dst = &s_pow.log_tab[0][0];
    for (int w = threadIdx.x; w < (int)(sizeof(PowTables) / 8); w += blockDim.x) dst[w] = src[w];
  }
  __syncthreads();

  Lane<M, F, O> L;
  __shared__ TrajRows s_trec[REC ? 128 : 1];  // per-lane trajectory rows
  const TrajRows* trec = REC ? &s_trec[threadIdx.x] : nullptr;
  __shared__ EmitBase s_eb[128];
  bool have = false, done = false;
  unsigned long long my_max = 0;
  const unsigned lt_mask = (1u << lane) - 1u;

  // the step loop, compiled with and without the debug trace (record_trace)
  // and with and without per-instance tolerance vectors, so the solve loop
  // carries no trace test or trace stores and, for scalar tolerances, no
  // tolerance pointer tests
  auto loop = [&](auto trace_tag, auto vtol_tag) {
  constexpr bool tracing = decltype(trace_tag)::value;
  constexpr bool vtol = decltype(vtol_tag)::value;
  unsigned done_mask = 0u;  // lanes out of work for good (changes only at a refill)
  // the shared bitmap's 32-bit shared-window address, kept in a register
  // (not re-derived from the CTA id on every rejection)
  uint32_t s_ref;
  asm("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(s_ref) : "l"(s_refresh));
  const bool smem_bm = P.smem_words > 0;
  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, !have && !done);
    if (need) {
      const int leader = __ffs(need) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(P.queue, (unsigned long long)__popc(need));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (!have && !done) {
        const unsigned long long pos = base + __popc(need & lt_mask);
        if (pos >= (unsigned long long)P.n) {
          done = true;
        } else {
          int64_t st;
          if (P.rec) {  // one contiguous record in queue order
            const int64_t off = L.resume_record(P, (int64_t)pos, st);
            s_eb[threadIdx.x] = EmitBase{P.t_eval_offsets ? P.t_eval + off : P.t_eval,
                                         P.ys ? P.ys + off * F::D : nullptr};
          } else {
            const int64_t i = P.order ? P.order[pos] : (int64_t)pos;
            // every load of the refill issues at once (one round trip after
            // the order lookup); a row the init pass finalised is dropped
            st = P.status[i];
            L.resume(P, i);
            s_eb[threadIdx.x] = EmitBase{L.te_of(P), L.ys_of(P)};
          }
          const int64_t i = L.idx;
          if (st == BODE_RUNNING) {
            if constexpr (REC)
              s_trec[threadIdx.x] = TrajRows{P.traj + P.traj_offsets[i] * kTrajStride<F::D>,
                                             P.traj + P.traj_offsets[i + 1] * kTrajStride<F::D>};
            have = true;
          }
        }
      }
      done_mask = __ballot_sync(0xffffffffu, done);
    }
    // every lane has a row or is done (need == 0): one vote per iteration
    if (done_mask == 0xffffffffu) break;
    if (have) {
      const uint32_t j = (uint32_t)L.nsteps;  // (n_steps is 32-bit: 32-bit bit index)
      if (L.template step<PI, vtol>(P, s_pow, tracing, trec, s_eb[threadIdx.x])) {
        const uint32_t bit = j + 1u;
        const uint32_t w = bit >> 5, msk = 1u << (bit & 31);
        if (smem_bm) {
          const uint32_t a = s_ref + 4u * w;
          uint32_t v;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
          if (!(v & msk)) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(msk) : "memory");
        } else {
          if (!(__ldcg(&P.refresh[w]) & msk)) atomicOr(&P.refresh[w], msk);
        }
      }
      if (L.status != BODE_RUNNING) {
        if ((unsigned long long)L.nsteps > my_max) my_max = (unsigned long long)L.nsteps;
        L.finish(P);
        have = false;
      }
    }
  }
  };
  if (P.trace_cap > 0)
    loop(BoolTag<true>{}, BoolTag<true>{});
  else if (P.atol_v || P.rtol_v)
    loop(BoolTag<false>{}, BoolTag<true>{});
  else
    loop(BoolTag<false>{}, BoolTag<false>{});
#ifdef BODE_EXIT_PROF
  if (lane == 0) {  // debug builds: when did each warp run out of work
    unsigned long long ts;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
    const unsigned slot = atomicAdd(&g_exit_count, 1u);
    if (slot < 65536) g_exit_times[slot] = ts;
  }
#endif
  // max n_steps: warp reduce then one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, my_max, o);
    my_max = v > my_max ? v : my_max;
  }
  if (lane == 0 && my_max) atomicMax(P.max_n, my_max);
  __syncthreads();
  for (int w = threadIdx.x; w < P.smem_words; w += blockDim.x)
    if (s_refresh[w]) atomicOr(&P.refresh[w], s_refresh[w]);
}

template <int M, class F, class O>
__global__ void __launch_bounds__(128) bode_init_kernel(const SolveParams P) {
  Lane<M, F, O> L;
  // instances in their natural order (coalesced per-instance reads and
  // writes); each resume record goes to its queue position (whole sectors)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    L.initialize(P, i);
    if (P.rec) L.write_record(P, P.rec_pos ? P.rec_pos[i] : i);
  }
}

#if BODE_HOST_CODE
// n_f_evals = 1 + (S-1)*max_n + #refresh iterations in [1, max_n)  (FSAL)
//           = 1 + S*max_n                                        (non-FSAL)
__global__ void bode_finalize_kernel(const unsigned long long* max_n, const uint32_t* refresh,
                                     int stages, int fsal, int64_t* n_f_evals,
                                     int64_t* max_out, uint8_t* map_out, int64_t map_len);

template <int M, class F, class O>
cudaError_t launch_persistent(const SolveParams& P, int threads, int blocks, cudaStream_t st) {
  // fast mode with an I / PI controller takes the specialised loop
  const bool pi = O::kFast && P.ctrl.plain_pi;
  auto kern = P.traj ? (pi ? bode_persistent_kernel<M, F, O, true, O::kFast>
                           : bode_persistent_kernel<M, F, O, true, false>)
                     : (pi ? bode_persistent_kernel<M, F, O, false, O::kFast>
                           : bode_persistent_kernel<M, F, O, false, false>);
  const size_t smem = (size_t)P.smem_words * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (threads <= 0) threads = 128;
  if (threads > 128 || threads % 32) return cudaErrorInvalidConfiguration;
  if (blocks <= 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t need = (P.n + threads - 1) / threads;
    blocks = (int)((int64_t)sms * per_sm < need ? (int64_t)sms * per_sm : need);
    if (blocks < 1) blocks = 1;
  }
  {
    const int64_t ib = (P.n + 127) / 128;
    bode_init_kernel<M, F, O><<<(unsigned)(ib < 148 * 64 ? ib : 148 * 64), 128, 0, st>>>(P);
  }
  if (P.ev_start) cudaEventRecord((cudaEvent_t)P.ev_start, st);
  kern<<<blocks, threads, smem, st>>>(P);
  if (P.ev_stop) cudaEventRecord((cudaEvent_t)P.ev_stop, st);
  return cudaGetLastError();
}

#endif  // BODE_HOST_CODE

}  // namespace bode
