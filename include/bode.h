/*
 * bode.h -- C ABI of libbode.so, the B200 (sm_100a) batched adaptive ODE
 * solver behind the batchode / torchode-style Python facade.
 *
 * Plain C: pointers, sizes and PODs only (no torch or CUDA types in the
 * signatures; streams travel as void*).  Every entry point replaces one
 * function of the reference's solve path (reference = /root/reference,
 * package ``batchode``, paths relative to pkg/src/batchode/):
 *
 *   bode_solve / bode_solve_host  <- solve()            solver.py:352-369
 *                                    BatchSolver.__init__/run/solution
 *                                                       solver.py:148-206,324-349
 *                                    (whole loop: step_once solver.py:208-282,
 *                                     _emit solver.py:284-322)
 *   bode_rk_step                  <- Stepper.step / rk_step  stepper.py:54-110,142-152
 *   bode_interpolate              <- Stepper.interpolate / interpolate
 *                                                       stepper.py:112-139,155-165
 *   bode_error_norm               <- error_norm         controller.py:120-142
 *   bode_adapt_step               <- adapt_step         controller.py:200-238
 *   bode_initial_step             <- initial_step       controller.py:145-197
 *   bode_solve_adjoint            <- (no reference counterpart: gradients,
 *                                    torchode's AutoDiffAdjoint backward;
 *                                    SURVEY.md 8(f) row 1)
 *
 * Error behaviour mirrors the reference: invalid arguments (the cases where
 * batchode raises ValueError) return BODE_EINVAL with a message in
 * bode_last_error(); numerical failure is never an error code, it is a
 * per-instance status (SolveStatus, solver.py:45-50).
 *
 * Memory: the caller owns every buffer, including the workspace
 * (bode_workspace_size); the library allocates nothing persistent.  All
 * device entry points are stream-ordered and asynchronous; bode_solve_host
 * is the synchronous host-buffer convenience used for end-to-end timing.
 */
#ifndef BODE_H_
#define BODE_H_

#ifndef __CUDACC_RTC__
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BODE_ABI_VERSION 6

/* return codes */
#define BODE_OK 0
#define BODE_EINVAL 1       /* invalid argument (reference: ValueError) */
#define BODE_ECUDA 2        /* CUDA runtime / launch failure */
#define BODE_EUNSUPPORTED 3 /* valid request this build does not implement */

/* per-instance status codes == batchode.SolveStatus (solver.py:45-50) */
#define BODE_RUNNING 0
#define BODE_SUCCESS 1
#define BODE_MAX_STEPS_EXCEEDED 2
#define BODE_STEP_UNDERFLOW 3
#define BODE_INFINITE_DYNAMICS 4

/* methods (tableau.py:102 dopri5, :152 tsit5; heun per SURVEY.md 8(b)) */
#define BODE_METHOD_DOPRI5 0
#define BODE_METHOD_TSIT5 1
#define BODE_METHOD_HEUN 2
/* a user ButcherTableau (tableau.py:17-83): coefficients compiled into a
 * run-time program (bode_program_create), args->program required */
#define BODE_METHOD_CUSTOM 3

/* registered dynamics (the reference takes any NumPy callable f(t, y),
 * stepper.py:19-20; a device solver needs them compiled in).  Parameter
 * slots p0..p7 per dynamics; slot k is per-instance when bit k of
 * inst_mask is set (read from inst_params, row-major n x popcount(mask)),
 * else shared_params[k].
 *   VDP        d=2  p0=mu                         (problems.py:41-50)
 *   LORENZ     d=3  p0=sigma p1=rho p2=beta
 *   ZERO       any  f=0
 *   CONST      any  p0=c                          f=c
 *   LINEAR     any  p0=lam                        f=lam*y
 *   LINEAR_COS any  p0=lam p1=amp p2=omega        f=lam*y + amp*cos(omega*t)
 *   LINEAR_SIN any  p0=lam p1=amp p2=omega        f=lam*y + amp*sin(omega*t)
 *   RELAX_COS  any  p0=lam p1=omega               f=lam*(y - cos(omega*t))
 *   SQUARE     any  p0=thr                        f= y>thr ? inf : y*y
 *   LOGISTIC   any                                f=y*(1-y)   (problems.py:178-179)
 *   SIN_PLUS_T any                                f=sin(y)+t
 *   HARMONIC   d=2                                f=(y1,-y0)  (problems.py:169-170)
 *   DAMPED     d=2                                f=(y1,-y0-0.1*y1*|y1|)
 *   MLP        any  weights in bode_mlp_weights   f=W2 tanh(W1 y + b1) + b2 (fp32) */
#define BODE_DYN_VDP 1
#define BODE_DYN_LORENZ 2
#define BODE_DYN_ZERO 3
#define BODE_DYN_CONST 4
#define BODE_DYN_LINEAR 5
#define BODE_DYN_LINEAR_COS 6
#define BODE_DYN_LINEAR_SIN 7
#define BODE_DYN_RELAX_COS 8
#define BODE_DYN_SQUARE 9
#define BODE_DYN_LOGISTIC 10
#define BODE_DYN_SIN_PLUS_T 11
#define BODE_DYN_HARMONIC 12
#define BODE_DYN_DAMPED 13
#define BODE_DYN_MLP 20
/* user dynamics compiled into a run-time program (bode_program_create):
 * the facade translates the reference's NumPy callable f(t, y) into a
 * device functor; inst_params = (n, desc.n_params) per-instance values it
 * reads, args->program required */
#define BODE_DYN_PROGRAM 30

/* arithmetic mode: EXACT = unfused IEEE ops in the reference's operation
 * order; FAST = FMA contraction allowed. */
#define BODE_MODE_EXACT 0
#define BODE_MODE_FAST 1

/* dt0 modes (solver.py:176-183) */
#define BODE_DT0_HEURISTIC 0 /* initial_step(), controller.py:145-197 */
#define BODE_DT0_SCALAR 1
#define BODE_DT0_ARRAY 2

typedef struct bode_dynamics {
  int32_t kind;               /* BODE_DYN_* */
  uint32_t inst_mask;         /* bit k: slot k is per-instance */
  const double* inst_params;  /* (n, popcount(inst_mask)) or NULL */
  double shared_params[8];
  /* MLP only (BODE_DYN_MLP): fp32 row-major, device pointers */
  const float* W1; /* (H, d) */
  const float* b1; /* (H,)   */
  const float* W2; /* (d, H) */
  const float* b2; /* (d,)   */
  int64_t hidden;  /* H */
} bode_dynamics;

typedef struct bode_controller {
  /* PidCoefficients (controller.py:57-83); exponents -beta/k are formed
   * on the host exactly as the reference does (controller.py:221-226). */
  double beta1, beta2, beta3;
  double safety, factor_min, factor_max;
  int32_t update_history_on_reject;
  int32_t _pad;
} bode_controller;

typedef struct bode_solve_args {
  int32_t abi_version; /* = BODE_ABI_VERSION */
  int32_t method;      /* BODE_METHOD_* */
  int32_t mode;        /* BODE_MODE_* */
  int32_t dt0_mode;    /* BODE_DT0_* */
  int64_t n, d;
  bode_dynamics dyn;
  bode_controller ctrl;
  /* problem (IvpBatch, solver.py:53-101); device pointers for bode_solve,
   * host pointers for bode_solve_host */
  const double* y0;      /* (n, d) */
  const double* t_start; /* (n,) */
  const double* t_end;   /* (n,) */
  /* t_eval: CSR (values + (n+1) offsets) or, with offsets NULL, one shared
   * sorted array of t_eval_len points used by every instance */
  const double* t_eval;
  const int64_t* t_eval_offsets;
  int64_t t_eval_len;
  /* tolerances (Tolerances, controller.py:39-54): array (n,) or scalar */
  const double* atol_v;
  const double* rtol_v;
  double atol, rtol;
  int64_t max_steps;   /* solver.py:42,155; 1 <= max_steps < 2^31 - 2 (32-bit per-instance
                        * step counters), BODE_EINVAL otherwise */
  double dt0;          /* BODE_DT0_SCALAR */
  const double* dt0_v; /* BODE_DT0_ARRAY, (n,) */
  /* processing order (cost-sorted LPT queue); NULL = natural order */
  const int64_t* order;
  /* outputs.  ys follows the t_eval layout: CSR rows (offsets) or dense
   * (n, t_eval_len, d); only the first n_emitted[i] rows of an instance are
   * written (unreached points are absent, solver.py:126-131). */
  double* ys;
  int64_t* n_emitted;   /* (n,) */
  int64_t* n_steps;     /* (n,) */
  int64_t* n_accepted;  /* (n,) */
  double* final_dt;     /* (n,) */
  int64_t* status;      /* (n,) SolveStatus codes, int64 like the reference */
  int64_t* n_f_evals;   /* (1,) batch-global count (solver.py:184,224,239) */
  /* optional record_trace (solver.py:196-199,257-261): (n, trace_cap) */
  double* trace_t;
  double* trace_dt;
  uint8_t* trace_accept;
  int64_t trace_cap;
  /* scratch from bode_workspace_size(); device memory */
  void* workspace;
  size_t workspace_bytes;
  void* stream; /* cudaStream_t */
  /* launch shape overrides (0 = auto) */
  int32_t threads_per_block;
  int32_t blocks;
  /* optional per-instance cost estimate (n,): when set and `order` is NULL
   * the library queues instances longest-first (LPT) with an on-device
   * bucketed counting sort (1/8-octave buckets).  Scheduling only: results
   * are identical for any order (batch independence). */
  const double* cost_hint;
  /* bode_solve_host only: split the batch into this many chunks and overlap
   * chunk k's solve with chunk k+1's upload and chunk k-1's download
   * (0 or 1 = no pipelining).  n_f_evals stays batch-global. */
  int32_t pipeline_chunks;
  /* 1: solve_joint (solver.py:372-427) -- the batch as ONE problem of size
   * n*d with one error norm, step size and accept decision; requires the
   * same t_start / t_end for every instance, a shared t_eval (offsets NULL)
   * and scalar tolerances; statistics are replicated per instance */
  int32_t joint;
  /* optional outputs for combining n_f_evals across shards (multi-GPU):
   * the largest n_steps of this solve and a byte per loop iteration j in
   * [0, max_steps + 2) that is 1 iff some instance rejected at iteration
   * j-1 and was still running at j (an FSAL refresh evaluation,
   * solver.py:220-226).  The global count is 1 + (S-1) * max_j + #{j >= 1 :
   * OR over shards of map[j]} (FSAL), 1 + S * max_j otherwise. */
  int64_t* max_iterations_out;
  uint8_t* refresh_map_out;
  /* reserved, must be 0.  (MLP dynamics run one path: d == 64 with hidden
   * a multiple of 32 up to 256 -> the fused persistent tcgen05 integrator;
   * other shapes return BODE_EUNSUPPORTED -- the Python facade zero-pads
   * narrower networks to the 64-wide tile.  There is no backend switch.) */
  int32_t reserved_mlp;
  int32_t _pad3;
  /* optional cudaEvent_t pair recorded on `stream` immediately before and
   * after the persistent integrator launch (roofline timing in bench.py) */
  void* prof_event_start;
  void* prof_event_stop;
  /* optional HOST pointer: number of kernels this call launched */
  int64_t* launch_count_out;
  /* optional (gradients, bode_solve_adjoint): record every accepted step.
   * Row traj_offsets[i] + k (k < n_accepted[i]) receives the k-th accepted
   * step of instance i: t_old, h, the t_eval cursor before the step,
   * y_old[d], padded to BODE_TRAJ_STRIDE(d) doubles (whole 32-byte
   * sectors, so the scattered per-instance row writes never partially fill
   * one).  traj_offsets (n+1) is the exclusive prefix sum of n_accepted
   * from an earlier identical solve (the solve is deterministic).  Not with
   * joint. */
  double* traj;
  const int64_t* traj_offsets;
  /* run-time program (bode_program_create) for a BODE_METHOD_CUSTOM tableau
   * and/or BODE_DYN_PROGRAM dynamics; NULL for the built-in kernels */
  const struct bode_program* program;
  /* MLP dynamics with d == 64 (the fused tcgen05 integrator), with traj:
   * the fp32 stage inputs Y_s of every recorded step, row r of traj owning
   * (S, 64) floats at traj_stages + r * S * 64 (slot s for s >= 1 when the
   * tableau is FSAL -- Y_0 is y_old --, every slot otherwise).  Required by
   * bode_solve_adjoint for such dynamics (its backward runs on the tensor
   * cores and does not recompute the forward stages). */
  float* traj_stages;
} bode_solve_args;

#define BODE_TRAJ_EXTRA 3
#define BODE_TRAJ_STRIDE(d) ((((d) + BODE_TRAJ_EXTRA) + 3) / 4 * 4)

/* Reverse-mode gradients of a solve ("AutoDiffAdjoint" backward; the
 * reference has no gradients, SPEC.md:13 / SURVEY.md 8(f) row 1).
 * Discretise-then-optimise through the recorded accepted steps: every RK
 * stage, the solution update and the Horner dense output are differentiated
 * exactly; the step sizes, accept decisions and interpolation positions
 * theta are held fixed (no gradient through the step-size controller). */
typedef struct bode_adjoint_args {
  const double* traj;          /* recorded by bode_solve (fwd->traj) */
  const int64_t* traj_offsets; /* (n+1,) */
  const int64_t* n_emitted;    /* (n,) from the forward solve */
  const double* grad_ys;       /* dL/dys, same layout as the forward ys */
  double* grad_y0;             /* (n, d) out: dL/dy0 */
  double* grad_params;         /* (n, 8) out or NULL: dL/dp_k of instance i
                                  (slot k of bode_dynamics; a shared slot's
                                  gradient is the column sum) */
  void* workspace;             /* bode_adjoint_workspace_size bytes, device */
  size_t workspace_bytes;
  int64_t* launch_count_out;   /* optional HOST pointer */
  /* MLP dynamics: dL/dW1 (H,d), dL/db1 (H,), dL/dW2 (d,H), dL/db2 (d,),
   * fp32 device buffers summed over the batch, each optional (NULL) */
  float* grad_W1;
  float* grad_b1;
  float* grad_W2;
  float* grad_b2;
  /* MLP dynamics with d == 64: fwd->traj_stages of the recording solve */
  const float* traj_stages;
} bode_adjoint_args;


/* A ButcherTableau by value (tableau.py:17-57) for the unit ops of the
 * stepping API: row-major a (stride BODE_TABLEAU_MAX_STAGES), interp row i
 * = ascending theta^1..theta^n_interp coefficients (stride
 * BODE_TABLEAU_MAX_INTERP).  Device memory. */
#define BODE_TABLEAU_MAX_STAGES 16
#define BODE_TABLEAU_MAX_INTERP 8
typedef struct bode_tableau {
  int32_t stages, n_interp, fsal, _pad;
  double a[BODE_TABLEAU_MAX_STAGES * BODE_TABLEAU_MAX_STAGES];
  double b[BODE_TABLEAU_MAX_STAGES];
  double b_err[BODE_TABLEAU_MAX_STAGES];
  double c[BODE_TABLEAU_MAX_STAGES];
  double interp[BODE_TABLEAU_MAX_STAGES * BODE_TABLEAU_MAX_INTERP];
} bode_tableau;

#ifndef __CUDACC_RTC__ /* entry points: host code only */
int bode_abi_version(void);
/* sizeof(bode_solve_args) as compiled, for binding layout checks */
size_t bode_sizeof_args(void);
const char* bode_last_error(void);
size_t bode_workspace_size(const bode_solve_args* args);

/* Full batched solve on device buffers, asynchronous on args->stream. */
int bode_solve(const bode_solve_args* args);

/* Same, but every pointer in args is a HOST pointer: copies inputs to the
 * device, solves, copies outputs back and synchronises (end-to-end path). */
int bode_solve_host(const bode_solve_args* args);

size_t bode_adjoint_workspace_size(const bode_solve_args* fwd);

/* dL/dy0 and dL/dparams for the solve described by fwd (the same
 * arguments as the recording bode_solve: method, dynamics, t_eval layout,
 * stream); device buffers, asynchronous on fwd->stream. */
int bode_solve_adjoint(const bode_solve_args* fwd, const bode_adjoint_args* adj);

/* One embedded RK trial step on the full batch (Stepper.step):
 * k0 = f0 for FSAL methods, else f(t, y).  k: (stages, n, d). */
int bode_rk_step(int32_t method, int32_t mode, const bode_dynamics* dyn, int64_t n,
                 int64_t d, const double* t, const double* dt, const double* y,
                 const double* f0, double* y_next, double* err, double* k,
                 void* stream);

/* Dense output y(t + theta*dt) from a step's stage derivatives; theta in
 * [0,1] is checked on the host path by the facade (stepper.py:126-127). */
int bode_interpolate(int32_t method, int32_t mode, int64_t n, int64_t d,
                     const double* k, const double* y0, const double* dt,
                     const double* theta, double* out, void* stream);

/* f(t, y) of a registered functor on the batch (the reference's dynamics
 * are callables, problems.py:41-50): t (n), y (n, d), out (n, d). */
int bode_eval_dynamics(const bode_dynamics* dyn, int64_t n, int64_t d, const double* t,
                       const double* y, double* out, void* stream);

/* Mixed-tolerance RMS norm, NumPy pairwise summation order. */
int bode_error_norm(int64_t n, int64_t d, const double* err, const double* y0,
                    const double* y1, const double* atol_v, const double* rtol_v,
                    double atol, double rtol, double* norm, void* stream);

/* adapt_step: updates (norm_prev, norm_prev2, dt) in place. */
int bode_adapt_step(int64_t n, const double* norm, int32_t error_order,
                    const bode_controller* ctrl, double* norm_prev,
                    double* norm_prev2, double* dt, uint8_t* accept,
                    double* dt_next, void* stream);

/* initial_step: dt (NaN where f0 is non-finite) and f0. */
int bode_initial_step(const bode_dynamics* dyn, int64_t n, int64_t d,
                      const double* t0, const double* y0, int32_t order,
                      const double* atol_v, const double* rtol_v, double atol,
                      double rtol, const double* direction, double* dt,
                      double* f0, void* stream);

/* ---- run-time programs: the reference's plugin surface on the device ----
 * The reference accepts any ButcherTableau (tableau.py:17-83) and any NumPy
 * callable f(t, y) (stepper.py:19-20).  libbode compiles a solver
 * specialisation for such a pair at run time (NVRTC, sm_100a): `source`
 * is CUDA C++ that, inside namespace bode, defines `template <class O>
 * struct UserDyn` (a functor with D, load(), operator(); or an alias of a
 * registered one) and, for method == BODE_METHOD_CUSTOM, specialises
 * TabShape<3> / Tab<3> with the tableau's coefficients.  The library
 * appends the kernel instantiations the `kernels` mask asks for.  Compile
 * errors return BODE_EINVAL with the NVRTC log in bode_last_error().
 * Programs are cached on disk by content ($BODE_JIT_CACHE, default
 * ~/.cache/bode_jit).  A program is bound to the device current at
 * creation. */
#define BODE_PROGRAM_SOLVE 1 /* init pass + persistent kernel (both modes) */
#define BODE_PROGRAM_STEP 2  /* BatchSolver stepping (bode_step_begin/once) */
#define BODE_PROGRAM_UNITS 4 /* rk_step / interpolate / initial_step */
#define BODE_PROGRAM_JOINT 8 /* solve_joint (args->joint) */
typedef struct bode_program_desc {
  int32_t method;   /* BODE_METHOD_* (CUSTOM: the source specialises Tab<3>) */
  int32_t kernels;  /* BODE_PROGRAM_* mask */
  int64_t d;        /* state width = UserDyn<O>::D */
  int32_t n_params; /* per-instance parameter columns of BODE_DYN_PROGRAM */
  /* tableau metadata (CUSTOM only; must match the source) */
  int32_t stages, order, error_order, fsal;
  int32_t _pad;
} bode_program_desc;
typedef struct bode_program bode_program;
int bode_program_create(const char* source, const bode_program_desc* desc, bode_program** out);
/* Compile only (no device needed): BODE_OK if the specialisation builds,
 * BODE_EINVAL with the NVRTC log otherwise. */
int bode_program_check(const char* source, const bode_program_desc* desc);
void bode_program_destroy(bode_program* prog);


/* BatchSolver (solver.py:141-349): the stepping API, one launch per loop
 * iteration, on device state.  args describe the batch exactly as for
 * bode_solve (program required, BODE_PROGRAM_STEP); its outputs double as
 * state (final_dt = ControllerState.dt, n_emitted = t_eval cursor,
 * n_steps, n_accepted, status, ys, trace).  The caller initialises
 * t = t_start, y = y0, norm_prev = norm_prev2 = 1, fsal_valid = 1,
 * n_steps = n_accepted = 0. */
typedef struct bode_step_state {
  double* t;            /* (n) */
  double* y;            /* (n, d) */
  double* f0;           /* (n, d) FSAL cache */
  double* norm_prev;    /* (n) ControllerState.norm_prev */
  double* norm_prev2;   /* (n) ControllerState.norm_prev2 */
  double* te_next;      /* (n) scratch */
  uint8_t* fsal_valid;  /* (n) */
  int32_t* flags;       /* (2) device: [0] any instance still running,
                           [1] an FSAL refresh evaluation happened */
} bode_step_state;
/* BatchSolver.__init__ (solver.py:148-206): f0, dt0 / initial_step,
 * INFINITE_DYNAMICS, points at t_start. */
int bode_step_begin(const bode_solve_args* args, const bode_step_state* s);
/* One step_once iteration (solver.py:208-282); flags are zeroed first. */
int bode_step_once(const bode_solve_args* args, const bode_step_state* s);

/* Unit ops for any tableau / dynamics (Stepper.step, stepper.py:54-110;
 * Stepper.interpolate, :112-139; initial_step, controller.py:145-197):
 * the tableau from device memory (bode_tableau), the dynamics from a
 * program compiled with BODE_PROGRAM_UNITS (its method is not used). */
int bode_program_rk_step(const bode_program* prog, const bode_tableau* tab,
                         const bode_dynamics* dyn, int64_t n, int64_t d, const double* t,
                         const double* dt, const double* y, const double* f0, double* y_next,
                         double* err, double* k, void* stream);
int bode_interpolate_tab(const bode_tableau* tab, int64_t n, int64_t d, const double* k,
                         const double* y0, const double* dt, const double* theta, double* out,
                         void* stream);
int bode_program_initial_step(const bode_program* prog, const bode_dynamics* dyn, int64_t n,
                              int64_t d, const double* t0, const double* y0, int32_t order,
                              const double* atol_v, const double* rtol_v, double atol,
                              double rtol, const double* direction, double* dt, double* f0,
                              void* stream);

/* One batch sharded across the GPUs of one process:
 * per_dev[k] is a complete bode_solve_args for shard k -- its buffers,
 * workspace and stream on one device (found from y0), a built-in method,
 * the same method and max_steps on every shard, max_iterations_out and
 * refresh_map_out set.  The shard solves run concurrently; then the
 * batch-global n_f_evals (solver.py:184,224,239) is combined across the
 * shards -- a MAX all-reduce over NCCL when comms != NULL (comms[k] = the
 * ncclComm_t of shard k in a communicator of exactly these ndev devices;
 * NCCL is loaded at run time), else one kernel on shard 0's device reading
 * the other shards by peer access -- and written to every shard's
 * n_f_evals (max_iterations_out / refresh_map_out then hold the global
 * values too).  Asynchronous on the shards' streams; per-instance outputs
 * stay on their shard's device.  At most 16 shards. */
int bode_solve_multi(const bode_solve_args* per_dev, int32_t ndev, void* const* comms);

/* Multi-GPU shard plan (the reference has one process and
 * no partition -- a shard is bitwise equal to its rows of the full batch,
 * tests/test_solver.py:140-168).  With cost (device, n): instances dealt to
 * `world` shards in decreasing cost in a snake pattern over the longest-first
 * order; perm (device, n) = shard 0's instance indices, then shard 1's, ...,
 * each shard longest-first (its queue order).  cost == NULL: contiguous
 * blocks, perm = identity.  shard_sizes (HOST, world) is filled before the
 * call returns (it depends on n and world only).  Asynchronous on stream.
 * Instances of equal cost bucket are ranked in arrival order, so two calls
 * may deal them differently: a multi-rank caller computes the plan on one
 * rank and broadcasts perm (the Python facade does). */
size_t bode_partition_workspace_size(int64_t n);
int bode_partition(const double* cost, int64_t n, int32_t world, int64_t* perm,
                   int64_t* shard_sizes, void* ws, size_t ws_bytes, void* stream);

/* Measurement utility (not on the solve path): launches blocks x 256
 * threads each running 8 independent chains of `iters` DFMAs, so a timed
 * launch gives the FP64 roofline denominator (2 flops per DFMA). */
int bode_probe_fp64(int64_t iters, int32_t blocks, double* out, void* stream);

/* Measurement utility: `blocks` CTAs (one per SM) each issue reps x 8
 * tcgen05.mma kind::tf32 M=128 N=256 K=8 back to back; a timed launch gives
 * the TF32 tensor roofline denominator (2*128*256*8 flops per MMA). */
int bode_probe_tf32(int32_t reps, int32_t blocks, void* stream);

#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif
#endif /* BODE_H_ */
