// bode_abi.cu -- the extern "C" boundary (include/bode.h).
//
// Translates bode_solve_args into kernel parameters, validates what the
// reference validates (returning BODE_EINVAL where batchode raises
// ValueError), and sequences, asynchronously on the caller's stream:
//   workspace reset -> [LPT queue order] -> init pass -> persistent solver
//   -> n_f_evals finalisation.
// bode_solve_host adds the host<->device copies and, optionally, a chunked
// pipeline that overlaps chunk k's solve with the neighbouring chunks' copies.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "bode_adjoint.cuh"
#include "bode_dispatch.cuh"
#include "bode_hostio.cuh"
#include "bode_joint.cuh"
#include "bode_mlp.cuh"
#include "bode_program_host.cuh"
#include "bode_sched.cuh"
#include "bode_units.cuh"

using namespace bode;

int bode::set_error(int code, const std::string& msg);

namespace {
thread_local std::string g_err;
thread_local int64_t g_launches;  // kernels launched by the current call

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorNotSupported)
    return fail(BODE_EUNSUPPORTED, std::string(where) + ": unsupported dynamics/width combination");
  if (e == cudaErrorInvalidValue)
    return fail(BODE_EINVAL, std::string(where) + ": state width does not match the dynamics");
  if (e == cudaErrorInvalidConfiguration)
    return fail(BODE_EINVAL, std::string(where) + ": threads_per_block must be a multiple of 32, <= 128");
  return fail(BODE_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// tableau metadata: built-in methods, or a CUSTOM tableau's from its program
int stages_of(const bode_solve_args* a) {
  if (a->method == BODE_METHOD_CUSTOM) return program_desc(a->program).stages;
  return a->method == BODE_METHOD_HEUN ? 2 : 7;
}
int error_order_of(const bode_solve_args* a) {
  if (a->method == BODE_METHOD_CUSTOM) return program_desc(a->program).error_order;
  return a->method == BODE_METHOD_HEUN ? 1 : 4;
}
int fsal_of(const bode_solve_args* a) {
  if (a->method == BODE_METHOD_CUSTOM) return program_desc(a->program).fsal;
  return a->method == BODE_METHOD_HEUN ? 0 : 1;
}

// per-instance parameter columns: the registered functors' masked slots,
// or a program's n_params
int inst_cols(const bode_dynamics& d, const bode_program* prog) {
  if (d.kind == BODE_DYN_PROGRAM) return prog ? program_desc(prog).n_params : 0;
  return __builtin_popcount(d.inst_mask);
}

DynParams make_dyn(const bode_dynamics& d, const bode_program* prog = nullptr) {
  DynParams p;
  p.kind = d.kind;
  p.inst_mask = d.inst_mask;
  p.n_inst = inst_cols(d, prog);
  p.inst = d.inst_params;
  for (int k = 0; k < 8; k++) p.shared[k] = d.shared_params[k];
  return p;
}

CtrlParams make_ctrl(const bode_controller& c, int error_order) {
  // exponents exactly as controller.py:221-226 forms them: (-beta)/k
  const double k = (double)(error_order + 1);
  CtrlParams p;
  p.e1 = (-c.beta1) / k;
  p.e2 = (-c.beta2) / k;
  p.e3 = (-c.beta3) / k;
  p.safety = c.safety;
  p.fmin = c.factor_min;
  p.fmax = c.factor_max;
  p.hist = c.update_history_on_reject;
  auto special = [](double e) { return e == 0.0 || e == 1.0 || e == -1.0 || e == 2.0 || e == 0.5; };
  p.plain_pi = std::isfinite(p.e1) && std::isfinite(p.e2) && !special(p.e1) &&
               (p.e2 == 0.0 || !special(p.e2)) && p.e3 == 0.0;
  return p;
}

bool valid_kind(int k) {
  return (k >= BODE_DYN_VDP && k <= BODE_DYN_DAMPED) || k == BODE_DYN_MLP || k == BODE_DYN_PROGRAM;
}

int validate(const bode_solve_args* a) {
  if (!a) return fail(BODE_EINVAL, "null args");
  if (a->abi_version != BODE_ABI_VERSION) return fail(BODE_EINVAL, "abi_version mismatch");
  if (a->reserved_mlp != 0) return fail(BODE_EINVAL, "reserved_mlp must be 0");
  if (a->n < 1 || a->d < 1)
    return fail(BODE_EINVAL, "need at least one instance and one state component");
  if (a->method < BODE_METHOD_DOPRI5 || a->method > BODE_METHOD_CUSTOM)
    return fail(BODE_EINVAL, "unknown method");
  if ((a->method == BODE_METHOD_CUSTOM || a->dyn.kind == BODE_DYN_PROGRAM) && !a->program)
    return fail(BODE_EINVAL, "a custom tableau / program dynamics needs args->program");
  if (a->program) {
    const bode_program_desc& pd = program_desc(a->program);
    if (pd.method != a->method) return fail(BODE_EINVAL, "program compiled for another method");
    if (pd.d != a->d) return fail(BODE_EINVAL, "program compiled for another state width");
    if (a->dyn.kind == BODE_DYN_MLP) return fail(BODE_EUNSUPPORTED, "programs: analytic dynamics only");
    if (a->traj) return fail(BODE_EUNSUPPORTED, "programs: no trajectory recording");
  }
  if (a->mode != BODE_MODE_EXACT && a->mode != BODE_MODE_FAST) return fail(BODE_EINVAL, "unknown mode");
  if (!valid_kind(a->dyn.kind)) return fail(BODE_EINVAL, "unknown dynamics");
  if (a->max_steps < 1) return fail(BODE_EINVAL, "max_steps must be at least 1");
  if (a->max_steps > 2147483645)  // (per-instance step counters are 32-bit)
    return fail(BODE_EINVAL, "max_steps must be below 2^31 - 2");
  if (!a->y0 || !a->t_start || !a->t_end) return fail(BODE_EINVAL, "y0/t_start/t_end required");
  if (!a->n_emitted || !a->n_steps || !a->n_accepted || !a->final_dt || !a->status || !a->n_f_evals)
    return fail(BODE_EINVAL, "output statistics buffers required");
  if ((a->t_eval_offsets || a->t_eval_len > 0) && !a->t_eval)
    return fail(BODE_EINVAL, "t_eval values required");
  if (a->dt0_mode == BODE_DT0_ARRAY && !a->dt0_v) return fail(BODE_EINVAL, "dt0 array required");
  if (a->dt0_mode < 0 || a->dt0_mode > 2) return fail(BODE_EINVAL, "unknown dt0 mode");
  if (!a->atol_v && a->atol < 0) return fail(BODE_EINVAL, "tolerances must be nonnegative");
  if (!a->rtol_v && a->rtol < 0) return fail(BODE_EINVAL, "tolerances must be nonnegative");
  const bode_controller& c = a->ctrl;
  if (!(c.safety > 0.0 && c.safety <= 1.0)) return fail(BODE_EINVAL, "safety must be in (0, 1]");
  if (!(0.0 < c.factor_min && c.factor_min < 1.0 && 1.0 < c.factor_max))
    return fail(BODE_EINVAL, "need 0 < factor_min < 1 < factor_max");
  if (inst_cols(a->dyn, a->program) && !a->dyn.inst_params)
    return fail(BODE_EINVAL, "per-instance params missing");
  if (a->dyn.kind == BODE_DYN_MLP &&
      (!a->dyn.W1 || !a->dyn.b1 || !a->dyn.W2 || !a->dyn.b2 || a->dyn.hidden < 1))
    return fail(BODE_EINVAL, "MLP weights required");
  // one MLP path: the fused tcgen05 integrator's 64-wide tile (narrower
  // networks are zero-padded by the caller -- the Python facade does it)
  if (a->dyn.kind == BODE_DYN_MLP && (a->d != 64 || a->dyn.hidden % 32 || a->dyn.hidden > 256))
    return fail(BODE_EUNSUPPORTED,
                "MLP dynamics: d == 64 and hidden a multiple of 32 up to 256 (zero-pad narrower networks)");
  if (a->pipeline_chunks < 0) return fail(BODE_EINVAL, "pipeline_chunks must be >= 0");
  if (a->traj && !a->traj_offsets) return fail(BODE_EINVAL, "traj needs traj_offsets");
  if (a->traj && a->joint)
    return fail(BODE_EUNSUPPORTED, "trajectory recording: independent solve only");
  if (a->joint) {  // solver.py:391-403
    if (a->t_eval_offsets) return fail(BODE_EINVAL, "joint mode requires identical evaluation points");
    if (a->atol_v || a->rtol_v) return fail(BODE_EINVAL, "joint mode supports scalar tolerances only");
    if (a->dt0_mode == BODE_DT0_ARRAY) return fail(BODE_EINVAL, "joint mode takes a scalar dt0");
    if (a->dyn.kind == BODE_DYN_MLP) return fail(BODE_EUNSUPPORTED, "joint mode: analytic dynamics only");
  }
  return BODE_OK;
}

// Workspace: [header | iteration bitmap | f0 (n x d) | te_next (n) | LPT scratch x slots | MLP scratch]
// Header: queue counter of slot 0 at +0, max n_steps at +8, queue counter of
// slot 1 at +16.  Pipelined host solves run consecutive chunks on two
// streams (slots 0/1), so a chunk's solve can fill the SMs the previous
// chunk's tail leaves idle; each slot has its own queue and LPT scratch, and
// f0 rows are indexed by absolute instance.
struct Layout {
  size_t f0, tn, rec, lpt, lpt_slot, mlp, total;
};

// resume records (bode_solver.cuh) for the persistent analytic kernels
bool use_records(const bode_solve_args* a) { return a->dyn.kind != BODE_DYN_MLP && !a->joint; }

Layout layout(const bode_solve_args* a, int64_t n_chunk, int slots) {
  Layout L;
  L.f0 = Workspace::f0_offset(a->max_steps);
  L.tn = L.f0 + ((8 * (size_t)a->n * (size_t)a->d + 255) & ~(size_t)255);
  L.rec = L.tn + ((8 * (size_t)a->n + 255) & ~(size_t)255);
  const size_t rec_bytes =
      use_records(a) ? 8 * (size_t)a->n * rec_stride(a->d, inst_cols(a->dyn, a->program)) : 0;
  L.lpt = L.rec + ((rec_bytes + 255) & ~(size_t)255);
  L.lpt_slot = a->cost_hint && !a->order ? ((lpt_workspace_bytes(n_chunk) + 255) & ~(size_t)255) : 0;
  L.mlp = L.lpt + L.lpt_slot * slots;
  L.total = L.mlp + (a->dyn.kind == BODE_DYN_MLP ? mlp_workspace_bytes(a) : 0);
  if (a->joint) L.total = L.f0 + joint_workspace_bytes(a->n, a->d, stages_of(a));
  return L;
}

int64_t chunk_max(int64_t n, int chunks) { return chunks > 1 ? (n + chunks - 1) / chunks : n; }

int reset_workspace(const bode_solve_args* a, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(a->workspace, 0,
                                  Workspace::kHeader + Workspace::bitmap_bytes(a->max_steps), st);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "workspace reset");
}

// Solve rows [lo, hi) of the batch described by `a` (device pointers).  The
// iteration bitmap and max n_steps accumulate across chunks, so n_f_evals
// stays batch-global; the queue counter is reset per chunk.
int run_chunk(const bode_solve_args* a, int64_t lo, int64_t hi, const Layout& L, cudaStream_t st,
              int slot = 0) {
  const int64_t n = hi - lo, d = a->d;
  const int n_inst = inst_cols(a->dyn, a->program);
  char* ws = (char*)a->workspace;
  const size_t qoff = slot ? 16 : 0;
  cudaError_t e = cudaMemsetAsync(ws + qoff, 0, 8, st);  // queue counter
  if (e != cudaSuccess) return cuda_fail(e, "queue reset");

  SolveParams P;
  memset(&P, 0, sizeof(P));
  P.n = n;
  P.dyn = make_dyn(a->dyn, a->program);
  if (P.dyn.inst) P.dyn.inst += lo * n_inst;
  P.ctrl = make_ctrl(a->ctrl, error_order_of(a));
  P.y0 = a->y0 + lo * d;
  P.t_start = a->t_start + lo;
  P.t_end = a->t_end + lo;
  P.t_eval = a->t_eval;
  if (a->t_eval_offsets) {  // absolute row indices into t_eval / ys
    P.t_eval_offsets = a->t_eval_offsets + lo;
    P.ys = a->ys;
  } else {
    P.t_eval_len = a->t_eval_len;
    P.ys = a->ys ? a->ys + lo * a->t_eval_len * d : nullptr;
  }
  P.atol_v = a->atol_v ? a->atol_v + lo : nullptr;
  P.rtol_v = a->rtol_v ? a->rtol_v + lo : nullptr;
  P.atol = a->atol;
  P.rtol = a->rtol;
  P.max_steps = a->max_steps;
  P.dt0_mode = a->dt0_mode;
  P.dt0 = a->dt0;
  P.dt0_v = a->dt0_v ? a->dt0_v + lo : nullptr;
  P.n_emitted = a->n_emitted + lo;
  P.n_steps = a->n_steps + lo;
  P.n_accepted = a->n_accepted + lo;
  P.final_dt = a->final_dt + lo;
  P.status = a->status + lo;
  P.trace_cap = a->trace_cap;
  P.trace_t = a->trace_t ? a->trace_t + lo * a->trace_cap : nullptr;
  P.trace_dt = a->trace_dt ? a->trace_dt + lo * a->trace_cap : nullptr;
  P.trace_accept = a->trace_accept ? a->trace_accept + lo * a->trace_cap : nullptr;
  P.traj = a->traj;
  P.traj_offsets = a->traj_offsets ? a->traj_offsets + lo : nullptr;
  P.queue = (unsigned long long*)(ws + qoff);
  P.max_n = (unsigned long long*)(ws + 8);
  P.refresh = (uint32_t*)(ws + Workspace::kHeader);
  const size_t words = Workspace::bitmap_words(a->max_steps);
  P.smem_words = words * 4 <= 32 * 1024 ? (int32_t)words : 0;  // per-block shared bitmap
  P.f0 = (double*)(ws + L.f0) + lo * d;
  P.te_next = (double*)(ws + L.tn) + lo;
  if (use_records(a)) {
    P.rec_stride = rec_stride(d, n_inst);
    P.rec = (double*)(ws + L.rec) + lo * P.rec_stride;
  }
  P.ev_start = a->prof_event_start;
  P.ev_stop = a->prof_event_stop;
  if (a->order) {
    if (lo != 0 || hi != a->n) return fail(BODE_EINVAL, "an explicit order cannot be chunked");
    P.order = a->order;
  } else if (a->cost_hint) {
    int64_t* order = nullptr;
    e = lpt_order(a->cost_hint + lo, n, ws + L.lpt + slot * L.lpt_slot, &order, st);
    g_launches += 3;
    if (e != cudaSuccess) return cuda_fail(e, "LPT order");
    P.order = order;
  }
  if (P.rec && P.order) {  // record positions (the te_next buffer is unused with records)
    int64_t* inv = reinterpret_cast<int64_t*>(P.te_next);
    if ((e = inverse_order(P.order, n, inv, st)) != cudaSuccess) return cuda_fail(e, "record order");
    P.rec_pos = inv;
    g_launches += 1;
  }
  if (a->joint) {
    g_launches += 1;
    e = joint_solve(a->method, a->mode, a->dyn.kind, d, P, ws + L.f0, a->n_f_evals, st,
                    a->program, stages_of(a));
    if (e == cudaErrorNotSupported && a->program)
      return fail(BODE_EINVAL, "program was not compiled with BODE_PROGRAM_JOINT");
    return e == cudaSuccess ? BODE_OK : cuda_fail(e, "joint solve");
  }
  if (a->dyn.kind == BODE_DYN_MLP) {
    e = mlp_solve(a, P, ws + L.mlp, st, &g_launches);
    return e == cudaSuccess ? BODE_OK : cuda_fail(e, "mlp solve");
  }
  if (a->program) {
    e = program_solve(a->program, a->mode, P, a->threads_per_block, a->blocks, st);
    g_launches += 2;
    if (e == cudaErrorNotSupported)
      return fail(BODE_EINVAL, "program was not compiled with BODE_PROGRAM_SOLVE");
    return e == cudaSuccess ? BODE_OK : cuda_fail(e, "program solve launch");
  }
  switch (a->method) {
    case BODE_METHOD_DOPRI5: e = solve_dopri5(a->mode, a->dyn.kind, d, P, a->threads_per_block, a->blocks, st); break;
    case BODE_METHOD_TSIT5: e = solve_tsit5(a->mode, a->dyn.kind, d, P, a->threads_per_block, a->blocks, st); break;
    default: e = solve_heun(a->mode, a->dyn.kind, d, P, a->threads_per_block, a->blocks, st); break;
  }
  g_launches += 2;  // init pass + persistent integrator
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "solve launch");
}

int finalize(const bode_solve_args* a, cudaStream_t st) {
  if (a->joint) return BODE_OK;  // the joint kernel counts its own n_f_evals
  char* ws = (char*)a->workspace;
  g_launches += 1;
  bode_finalize_kernel<<<1, 256, 0, st>>>((unsigned long long*)(ws + 8),
                                          (uint32_t*)(ws + Workspace::kHeader),
                                          stages_of(a), fsal_of(a), a->n_f_evals,
                                          a->max_iterations_out, a->refresh_map_out,
                                          a->max_steps + 2);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "finalize launch");
}

// keep freed device memory in the stream-ordered pool across calls instead
// of returning it to the driver at every synchronisation
void retain_pool() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

// per-device streams/events of bode_solve_host, created on first use
struct HostStreams {
  cudaStream_t cin, cout, st2;
  cudaEvent_t ev_in[64], ev_done[65], ev_out[65], ready;
};
HostStreams& host_streams() {
  static std::mutex m;
  static HostStreams* per_dev[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(m);
  if (!per_dev[dev]) {
    HostStreams* h = new HostStreams;
    cudaStreamCreateWithFlags(&h->cin, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&h->cout, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking);
    for (int k = 0; k < 65; k++) {
      if (k < 64) cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&h->ev_done[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&h->ev_out[k], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&h->ready, cudaEventDisableTiming);
    per_dev[dev] = h;
  }
  return *per_dev[dev];
}

}  // namespace

int bode::set_error(int code, const std::string& msg) { return fail(code, msg); }

extern "C" {

int bode_abi_version(void) { return BODE_ABI_VERSION; }

size_t bode_sizeof_args(void) { return sizeof(bode_solve_args); }

const char* bode_last_error(void) { return g_err.c_str(); }

size_t bode_workspace_size(const bode_solve_args* a) {
  if (validate(a) != BODE_OK) return 0;
  return layout(a, a->n, 1).total;
}

int bode_solve(const bode_solve_args* a) {
  int rc = validate(a);
  if (rc != BODE_OK) return rc;
  g_launches = 0;
  const Layout L = layout(a, a->n, 1);
  if (!a->workspace || a->workspace_bytes < L.total)
    return fail(BODE_EINVAL, "workspace too small (see bode_workspace_size)");
  cudaStream_t st = (cudaStream_t)a->stream;
  if ((rc = reset_workspace(a, st)) != BODE_OK) return rc;
  if ((rc = run_chunk(a, 0, a->n, L, st)) != BODE_OK) return rc;
  rc = finalize(a, st);
  if (a->launch_count_out) *a->launch_count_out = g_launches;
  return rc;
}

size_t bode_adjoint_workspace_size(const bode_solve_args* a) {
  if (validate(a) != BODE_OK) return 0;
  return adjoint_workspace_bytes(a->n, a->d, a->dyn.kind, a->dyn.hidden);
}

int bode_solve_adjoint(const bode_solve_args* a, const bode_adjoint_args* g) {
  int rc = validate(a);
  if (rc != BODE_OK) return rc;
  if (!g) return fail(BODE_EINVAL, "null adjoint args");
  if (a->joint) return fail(BODE_EUNSUPPORTED, "gradients: independent solve only");
  if (a->program) return fail(BODE_EUNSUPPORTED, "gradients: built-in methods and dynamics only");

  if (!g->traj || !g->traj_offsets || !g->n_emitted || !g->grad_y0)
    return fail(BODE_EINVAL, "adjoint needs traj, traj_offsets, n_emitted and grad_y0");
  if (a->dyn.kind == BODE_DYN_MLP && !g->traj_stages)
    return fail(BODE_EINVAL, "MLP gradients: the forward must record traj_stages");
  if ((a->t_eval_offsets || a->t_eval_len > 0) && !g->grad_ys)
    return fail(BODE_EINVAL, "adjoint needs grad_ys");
  if (!g->workspace ||
      g->workspace_bytes < adjoint_workspace_bytes(a->n, a->d, a->dyn.kind, a->dyn.hidden))
    return fail(BODE_EINVAL, "workspace too small (see bode_adjoint_workspace_size)");
  AdjParams A;
  memset(&A, 0, sizeof(A));
  A.n = a->n;
  A.dyn = make_dyn(a->dyn);
  A.t_eval = a->t_eval;
  A.t_eval_offsets = a->t_eval_offsets;
  A.t_eval_len = a->t_eval_offsets ? 0 : a->t_eval_len;
  A.traj = g->traj;
  A.traj_offsets = g->traj_offsets;
  A.n_emitted = g->n_emitted;
  A.grad_ys = g->grad_ys;
  A.grad_y0 = g->grad_y0;
  A.grad_params = g->grad_params;
  if (a->dyn.kind == BODE_DYN_MLP) {
    A.H = a->dyn.hidden;
    A.W1 = a->dyn.W1;
    A.b1 = a->dyn.b1;
    A.W2 = a->dyn.W2;
    A.b2 = a->dyn.b2;
    A.gW1 = g->grad_W1;
    A.gb1 = g->grad_b1;
    A.gW2 = g->grad_W2;
    A.gb2 = g->grad_b2;
    A.traj_stages = g->traj_stages;
  }
  int64_t launches = 0;
  cudaError_t e = adjoint_launch(a->method, a->d, A, g->workspace, (cudaStream_t)a->stream,
                                 &launches);
  if (g->launch_count_out) *g->launch_count_out = launches;
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "adjoint launch");
}

int bode_solve_host(const bode_solve_args* h) {
  int rc = validate(h);
  if (rc != BODE_OK) return rc;
  if (h->traj) return fail(BODE_EUNSUPPORTED, "trajectory recording: device buffers (bode_solve) only");
  g_launches = 0;
  retain_pool();
  const int64_t n = h->n, d = h->d;
  const bool csr = h->t_eval_offsets != nullptr;
  const int64_t n_te = csr ? h->t_eval_offsets[n] : h->t_eval_len;
  const int64_t ys_rows = csr ? n_te : n * h->t_eval_len;
  const int n_inst = inst_cols(h->dyn, h->program);
  int chunks = h->pipeline_chunks > 1 ? h->pipeline_chunks : 1;
  if (h->order || h->trace_cap > 0 || h->dyn.kind == BODE_DYN_MLP || h->joint) chunks = 1;
  if (chunks > n) chunks = (int)n;
  if (chunks > 64) chunks = 64;
  // largest chunk (a middle one when the first/last are smaller); sized for
  // the smallest edge fraction BODE_EDGE_FRAC may request (0.1)
  const int64_t cmax = chunks >= 3 ? (int64_t)((double)n / ((chunks - 2) + 0.2)) + 2 : chunk_max(n, chunks);

  // one device block for every array; per-instance arrays move in chunk
  // slices so chunk k can start as soon as its own rows landed.  Pinned
  // host arrays are DMA'd directly, pageable ones through the pinned arena.
  struct Arr {
    const void* hsrc;   // host input (or null)
    void* hdst;         // host output (or null)
    size_t row_bytes;   // bytes per instance row (0: whole array)
    size_t bytes;       // total bytes
    size_t off;         // device offset
    const void** in_field;
    void** out_field;
    bool pinned;
    size_t stage;       // arena offset (pageable arrays)
  };
  bode_solve_args a = *h;
  std::vector<Arr> arrs;
  size_t total = 0, stage_total = 0;
  size_t stage_max = (size_t)2 << 30;  // larger pageable payloads use driver staging
  if (const char* e = std::getenv("BODE_STAGING_MAX")) stage_max = (size_t)std::atoll(e);
  auto place = [&](size_t bytes) {
    const size_t off = total;
    total += (bytes + 255) & ~(size_t)255;
    return off;
  };
  auto add = [&](const void* hs, void* hd, size_t row_bytes, size_t bytes, const void** fi,
                 void** fo) {
    Arr x{hs, hd, row_bytes, bytes, place(bytes), fi, fo, false, 0};
    x.pinned = hostio::is_pinned(hs ? hs : hd);
    if (!x.pinned && stage_total + bytes <= stage_max) {
      x.stage = stage_total;
      stage_total += (bytes + 4095) & ~(size_t)4095;
    } else if (!x.pinned) {
      x.stage = SIZE_MAX;  // direct pageable copy
    }
    arrs.push_back(x);
  };
  auto in = [&](const void** field, size_t row_bytes, size_t bytes) {
    if (*field && bytes) add(*field, nullptr, row_bytes, bytes, field, nullptr);
  };
  auto out = [&](void** field, size_t row_bytes, size_t bytes) {
    if (*field && bytes) add(nullptr, *field, row_bytes, bytes, nullptr, field);
  };
  in((const void**)&a.y0, 8 * d, 8 * n * d);
  in((const void**)&a.t_start, 8, 8 * n);
  in((const void**)&a.t_end, 8, 8 * n);
  in((const void**)&a.t_eval, 0, 8 * n_te);
  in((const void**)&a.t_eval_offsets, 0, csr ? 8 * (n + 1) : 0);
  in((const void**)&a.atol_v, 8, 8 * n);
  in((const void**)&a.rtol_v, 8, 8 * n);
  in((const void**)&a.dt0_v, 8, a.dt0_mode == BODE_DT0_ARRAY ? 8 * n : 0);
  in((const void**)&a.order, 0, 8 * n);
  in((const void**)&a.cost_hint, 8, 8 * n);
  in((const void**)&a.dyn.inst_params, 8 * n_inst, 8 * n * n_inst);
  if (h->dyn.kind == BODE_DYN_MLP) {
    const int64_t H = h->dyn.hidden;
    in((const void**)&a.dyn.W1, 0, 4 * H * d);
    in((const void**)&a.dyn.b1, 0, 4 * H);
    in((const void**)&a.dyn.W2, 0, 4 * d * H);
    in((const void**)&a.dyn.b2, 0, 4 * d);
  }
  const size_t n_in = arrs.size();
  // ys rows follow the instance order, so they can be fetched per chunk
  out((void**)&a.ys, 0, 8 * ys_rows * d);
  out((void**)&a.n_emitted, 8, 8 * n);
  out((void**)&a.n_steps, 8, 8 * n);
  out((void**)&a.n_accepted, 8, 8 * n);
  out((void**)&a.final_dt, 8, 8 * n);
  out((void**)&a.status, 8, 8 * n);
  out((void**)&a.trace_t, 8 * h->trace_cap, 8 * n * h->trace_cap);
  out((void**)&a.trace_dt, 8 * h->trace_cap, 8 * n * h->trace_cap);
  out((void**)&a.trace_accept, h->trace_cap, n * h->trace_cap);
  out((void**)&a.max_iterations_out, 0, 8);
  out((void**)&a.refresh_map_out, 0, (size_t)h->max_steps + 2);
  out((void**)&a.n_f_evals, 0, 8);
  const Layout L = layout(h, cmax, chunks > 1 ? 2 : 1);
  const size_t ws_off = place(L.total);

  hostio::Arena& ar = hostio::arena();
  std::lock_guard<std::mutex> arena_lock(ar.m);  // one staged host solve at a time
  cudaError_t e = ar.reserve(stage_total);
  if (e != cudaSuccess) return cuda_fail(e, "pinned staging arena");
  char* stage = ar.p;

  cudaStream_t st = (cudaStream_t)h->stream;
  char* dev = nullptr;
  e = cudaMallocAsync((void**)&dev, total, st);
  if (e != cudaSuccess) return cuda_fail(e, "device allocation");
  for (auto& x : arrs) {
    if (x.in_field) *x.in_field = dev + x.off;
    if (x.out_field) *x.out_field = dev + x.off;
  }
  a.workspace = dev + ws_off;
  a.workspace_bytes = L.total;
  // uploads on `cin`, downloads on `cout`, solves on the caller's stream
  // copy streams and the second chunk stream are created once per device and
  // reused (the arena lock serialises host solves); events likewise
  HostStreams& hs = host_streams();
  cudaStream_t cin = hs.cin, cout = hs.cout, st2 = chunks > 1 ? hs.st2 : st;
  cudaEvent_t* ev_in = hs.ev_in;
  cudaEvent_t* ev_done = hs.ev_done;
  cudaEvent_t* ev_out = hs.ev_out;
  {
    cudaEvent_t ready = hs.ready;  // the allocation is visible to the copy streams
    cudaEventRecord(ready, st);
    cudaStreamWaitEvent(cin, ready, 0);
    cudaStreamWaitEvent(cout, ready, 0);
    if (st2 != st) cudaStreamWaitEvent(st2, ready, 0);
  }
  // chunk boundaries: the first and last chunks are `edge` of a middle
  // chunk (half; BODE_EDGE_FRAC overrides it -- on C2, 3 chunks: 4.23 ms e2e
  // at 0.5 and 0.3, 4.90 at 0.15), so the first solve starts (and the last
  // download ends) sooner
  double edge = 0.5;
  if (const char* ev = std::getenv("BODE_EDGE_FRAC")) edge = std::atof(ev);
  if (!(edge >= 0.1 && edge <= 1.0)) edge = 0.5;
  int64_t bnd[65];
  bnd[0] = 0;
  for (int k = 1; k <= chunks; k++) {
    const double units = chunks >= 3 ? (chunks - 2) + 2.0 * edge : (double)chunks;
    const double done = chunks >= 3 ? (k == chunks ? units : edge + (k - 1)) : (double)k;
    bnd[k] = k == chunks ? n : (int64_t)((double)n * done / units);
  }
  auto rows = [&](int k, int64_t& lo, int64_t& hi) {
    lo = bnd[k];
    hi = bnd[k + 1];
  };
  // byte range [o, o+b) of array x that belongs to chunk k; k == chunks
  // means "the whole-array outputs written by the finaliser"
  auto slice = [&](const Arr& x, int k, size_t& o, size_t& b) -> bool {
    int64_t lo, hi;
    if (x.row_bytes) {
      if (k == chunks) return false;
      rows(k, lo, hi);
      o = (size_t)lo * x.row_bytes;
      b = (size_t)(hi - lo) * x.row_bytes;
    } else if (x.out_field == (void**)&a.ys ||
               (csr && x.in_field == (const void**)&a.t_eval)) {  // CSR rows of this chunk
      if (k == chunks) return false;
      rows(k, lo, hi);
      const int64_t r0 = csr ? h->t_eval_offsets[lo] : lo * h->t_eval_len;
      const int64_t r1 = csr ? h->t_eval_offsets[hi] : hi * h->t_eval_len;
      const size_t w = x.in_field ? 8 : 8 * (size_t)d;
      o = (size_t)r0 * w;
      b = (size_t)(r1 - r0) * w;
    } else if (x.in_field == (const void**)&a.t_eval_offsets) {  // offsets [lo, hi]
      if (k == chunks) return false;
      rows(k, lo, hi);
      o = (size_t)lo * 8;
      b = (size_t)(hi - lo + 1) * 8;
    } else {  // whole arrays: inputs with chunk 0, outputs after the finaliser
      if (k != (x.in_field ? 0 : chunks)) return false;
      o = 0;
      b = x.bytes;
    }
    return b > 0;
  };
  auto copy_in = [&](int k) -> cudaError_t {
    for (size_t j = 0; j < n_in; j++) {
      const Arr& x = arrs[j];
      size_t o, b;
      if (!slice(x, k, o, b)) continue;
      const char* src = (const char*)x.hsrc + o;
      if (!x.pinned && x.stage != SIZE_MAX) {  // pageable: fill the arena on the host team
        hostio::par_copy(stage + x.stage + o, src, b);
        src = stage + x.stage + o;
      }
      cudaError_t r = cudaMemcpyAsync(dev + x.off + o, src, b, cudaMemcpyHostToDevice, cin);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  };
  auto copy_out = [&](int k) -> cudaError_t {
    for (size_t j = n_in; j < arrs.size(); j++) {
      const Arr& x = arrs[j];
      size_t o, b;
      if (!slice(x, k, o, b)) continue;
      char* dst = (!x.pinned && x.stage != SIZE_MAX) ? stage + x.stage + o : (char*)x.hdst + o;
      cudaError_t r = cudaMemcpyAsync(dst, dev + x.off + o, b, cudaMemcpyDeviceToHost, cout);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  };
  auto drain = [&](int k) {  // arena -> pageable user outputs of chunk k
    for (size_t j = n_in; j < arrs.size(); j++) {
      const Arr& x = arrs[j];
      size_t o, b;
      if (x.pinned || x.stage == SIZE_MAX || !slice(x, k, o, b)) continue;
      hostio::par_copy((char*)x.hdst + o, stage + x.stage + o, b);
    }
  };

  rc = reset_workspace(&a, st);
  if (st2 != st) {  // the reset is visible to the second chunk stream
    cudaEventRecord(ev_done[chunks], st);
    cudaStreamWaitEvent(st2, ev_done[chunks], 0);
  }
  for (int k = 0; k < chunks && rc == BODE_OK && e == cudaSuccess; k++) {
    // while the host stages chunk k, chunk k-1 is already solving
    if ((e = copy_in(k)) != cudaSuccess) break;
    cudaStream_t sk = (k & 1) ? st2 : st;
    cudaEventRecord(ev_in[k], cin);
    cudaStreamWaitEvent(sk, ev_in[k], 0);
    int64_t lo, hi;
    rows(k, lo, hi);
    if ((rc = run_chunk(&a, lo, hi, L, sk, k & 1)) != BODE_OK) break;
    cudaEventRecord(ev_done[k], sk);
    cudaStreamWaitEvent(cout, ev_done[k], 0);
    if ((e = copy_out(k)) != cudaSuccess) break;
    cudaEventRecord(ev_out[k], cout);
  }
  if (st2 != st && rc == BODE_OK && e == cudaSuccess) {  // join: last chunk on st2
    const int last_odd = (chunks - 1) & 1 ? chunks - 1 : chunks - 2;
    cudaStreamWaitEvent(st, ev_done[last_odd], 0);
  }
  if (rc == BODE_OK && e == cudaSuccess) rc = finalize(&a, st);
  if (rc == BODE_OK && e == cudaSuccess) {
    cudaEventRecord(ev_done[chunks], st);
    cudaStreamWaitEvent(cout, ev_done[chunks], 0);
    e = copy_out(chunks);
    cudaEventRecord(ev_out[chunks], cout);
  }
  const bool ok = rc == BODE_OK && e == cudaSuccess;
  // drain pageable outputs chunk by chunk while later chunks still solve
  for (int k = 0; ok && k <= chunks; k++) {
    if (cudaEventSynchronize(ev_out[k]) != cudaSuccess) break;
    drain(k);
  }
  cudaStreamSynchronize(cin);
  cudaStreamSynchronize(cout);
  cudaFreeAsync(dev, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  if (st2 != st) cudaStreamSynchronize(st2);
  if (rc != BODE_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "host<->device copy");
  if (e2 != cudaSuccess) return cuda_fail(e2, "solve");
  if (h->launch_count_out) *h->launch_count_out = g_launches;
  return BODE_OK;
}

int bode_rk_step(int32_t method, int32_t mode, const bode_dynamics* dyn, int64_t n, int64_t d,
                 const double* t, const double* dt, const double* y, const double* f0,
                 double* y_next, double* err, double* k, void* stream) {
  if (!dyn || n < 1 || d < 1) return fail(BODE_EINVAL, "bad rk_step arguments");
  if (mode != BODE_MODE_EXACT) return fail(BODE_EUNSUPPORTED, "unit ops run in exact mode only");
  if (dyn->kind == BODE_DYN_MLP) return fail(BODE_EUNSUPPORTED, "use bode_solve for MLP dynamics");
  cudaError_t e = unit_rk_step(method, make_dyn(*dyn), n, d, t, dt, y, f0, y_next, err, k,
                               (cudaStream_t)stream);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "rk_step");
}

int bode_interpolate(int32_t method, int32_t mode, int64_t n, int64_t d, const double* k,
                     const double* y0, const double* dt, const double* theta, double* out,
                     void* stream) {
  if (n < 1 || d < 1) return fail(BODE_EINVAL, "bad interpolate arguments");
  if (mode != BODE_MODE_EXACT) return fail(BODE_EUNSUPPORTED, "unit ops run in exact mode only");
  cudaError_t e = unit_interpolate(method, n, d, k, y0, dt, theta, out, (cudaStream_t)stream);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "interpolate");
}

int bode_error_norm(int64_t n, int64_t d, const double* err, const double* y0, const double* y1,
                    const double* atol_v, const double* rtol_v, double atol, double rtol,
                    double* norm, void* stream) {
  if (n < 1 || d < 1) return fail(BODE_EINVAL, "bad error_norm arguments");
  cudaStream_t st = (cudaStream_t)stream;
  double* scratch = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&scratch, sizeof(double) * n * d, st);
  if (e != cudaSuccess) return cuda_fail(e, "error_norm scratch");
  e = unit_error_norm(n, d, err, y0, y1, atol_v, rtol_v, atol, rtol, norm, scratch, st);
  cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "error_norm");
}

int bode_adapt_step(int64_t n, const double* norm, int32_t error_order,
                    const bode_controller* ctrl, double* norm_prev, double* norm_prev2,
                    double* dt, uint8_t* accept, double* dt_next, void* stream) {
  if (!ctrl || n < 1) return fail(BODE_EINVAL, "bad adapt_step arguments");
  cudaError_t e = unit_adapt_step(n, norm, make_ctrl(*ctrl, error_order), norm_prev, norm_prev2,
                                  dt, accept, dt_next, (cudaStream_t)stream);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "adapt_step");
}

int bode_initial_step(const bode_dynamics* dyn, int64_t n, int64_t d, const double* t0,
                      const double* y0, int32_t order, const double* atol_v,
                      const double* rtol_v, double atol, double rtol, const double* direction,
                      double* dt, double* f0, void* stream) {
  if (!dyn || n < 1 || d < 1) return fail(BODE_EINVAL, "bad initial_step arguments");
  if (dyn->kind == BODE_DYN_MLP) return fail(BODE_EUNSUPPORTED, "use bode_solve for MLP dynamics");
  cudaError_t e = unit_initial_step(make_dyn(*dyn), n, d, t0, y0, order, atol_v, rtol_v, atol,
                                    rtol, direction, dt, f0, (cudaStream_t)stream);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "initial_step");
}

}  // extern "C"

// ------------------------------------------------------------ partition --
extern "C" size_t bode_partition_workspace_size(int64_t n) {
  return n < 1 ? 0 : lpt_workspace_bytes(n);
}

extern "C" int bode_partition(const double* cost, int64_t n, int32_t world, int64_t* perm,
                              int64_t* shard_sizes, void* ws, size_t ws_bytes, void* stream) {
  if (n < 1) return fail(BODE_EINVAL, "bode_partition: need at least one instance");
  if (world < 1 || world > 4096) return fail(BODE_EINVAL, "bode_partition: world must be in [1, 4096]");
  if (!perm || !shard_sizes) return fail(BODE_EINVAL, "bode_partition: null output");
  if (cost && (!ws || ws_bytes < bode_partition_workspace_size(n)))
    return fail(BODE_EINVAL, "bode_partition: workspace too small");
  compute_shard_sizes(n, world, cost != nullptr, shard_sizes);
  const cudaError_t e = shard_partition(cost, n, world, perm, ws, (cudaStream_t)stream);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "bode_partition");
}

// ------------------------------------------------- stepping API (programs) --
namespace {
int step_params(const bode_solve_args* a, const bode_step_state* s, SolveParams& P) {
  int rc = validate(a);
  if (rc != BODE_OK) return rc;
  if (!a->program) return fail(BODE_EINVAL, "the stepping API runs a program (args->program)");
  if (!s || !s->t || !s->y || !s->f0 || !s->norm_prev || !s->norm_prev2 || !s->te_next ||
      !s->fsal_valid || !s->flags)
    return fail(BODE_EINVAL, "bode_step_state: every buffer is required");
  if (a->order || a->cost_hint) return fail(BODE_EINVAL, "stepping: natural order only");
  memset(&P, 0, sizeof(P));
  P.n = a->n;
  P.dyn = make_dyn(a->dyn, a->program);
  P.ctrl = make_ctrl(a->ctrl, error_order_of(a));
  P.y0 = a->y0;
  P.t_start = a->t_start;
  P.t_end = a->t_end;
  P.t_eval = a->t_eval;
  P.t_eval_offsets = a->t_eval_offsets;
  P.t_eval_len = a->t_eval_offsets ? 0 : a->t_eval_len;
  P.ys = a->ys;
  P.atol_v = a->atol_v;
  P.rtol_v = a->rtol_v;
  P.atol = a->atol;
  P.rtol = a->rtol;
  P.max_steps = a->max_steps;
  P.dt0_mode = a->dt0_mode;
  P.dt0 = a->dt0;
  P.dt0_v = a->dt0_v;
  P.n_emitted = a->n_emitted;
  P.n_steps = a->n_steps;
  P.n_accepted = a->n_accepted;
  P.final_dt = a->final_dt;
  P.status = a->status;
  P.trace_t = a->trace_t;
  P.trace_dt = a->trace_dt;
  P.trace_accept = a->trace_accept;
  P.trace_cap = a->trace_cap;
  P.f0 = s->f0;
  P.te_next = s->te_next;
  return BODE_OK;
}
}  // namespace

extern "C" int bode_step_begin(const bode_solve_args* a, const bode_step_state* s) {
  SolveParams P;
  int rc = step_params(a, s, P);
  if (rc != BODE_OK) return rc;
  const cudaError_t e = program_init(a->program, a->mode, P, (cudaStream_t)a->stream);
  if (e == cudaErrorNotSupported)
    return fail(BODE_EINVAL, "program was not compiled with BODE_PROGRAM_STEP");
  if (a->launch_count_out) *a->launch_count_out = 1;
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "bode_step_begin");
}

extern "C" int bode_step_once(const bode_solve_args* a, const bode_step_state* s) {
  SolveParams P;
  int rc = step_params(a, s, P);
  if (rc != BODE_OK) return rc;
  cudaStream_t st = (cudaStream_t)a->stream;
  cudaError_t e = cudaMemsetAsync(s->flags, 0, 8, st);
  if (e != cudaSuccess) return cuda_fail(e, "bode_step_once");
  StepState S{s->t, s->y, s->norm_prev, s->norm_prev2, s->fsal_valid, s->flags};
  e = program_step(a->program, a->mode, P, S, st);
  if (e == cudaErrorNotSupported)
    return fail(BODE_EINVAL, "program was not compiled with BODE_PROGRAM_STEP");
  if (a->launch_count_out) *a->launch_count_out = 1;
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "bode_step_once");
}

// ------------------------------------------------------- program unit ops --
extern "C" int bode_program_rk_step(const bode_program* prog, const bode_tableau* tab,
                                    const bode_dynamics* dyn, int64_t n, int64_t d,
                                    const double* t, const double* dt, const double* y,
                                    const double* f0, double* y_next, double* err, double* k,
                                    void* stream) {
  if (!prog || !tab || !dyn || n < 1 || d != program_desc(prog).d || !t || !dt || !y || !y_next ||
      !err || !k)
    return fail(BODE_EINVAL, "bode_program_rk_step: invalid arguments");
  const cudaError_t e = program_rk_step(prog, tab, make_dyn(*dyn, prog), n, t, dt, y, f0, y_next,
                                        err, k, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported) return fail(BODE_EINVAL, "program was not compiled with BODE_PROGRAM_UNITS");
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "bode_program_rk_step");
}

extern "C" int bode_interpolate_tab(const bode_tableau* tab, int64_t n, int64_t d,
                                    const double* k, const double* y0, const double* dt,
                                    const double* theta, double* out, void* stream) {
  if (!tab || n < 1 || d < 1 || !k || !y0 || !dt || !theta || !out)
    return fail(BODE_EINVAL, "bode_interpolate_tab: invalid arguments");
  const cudaError_t e = unit_interpolate_tab(tab, n, d, k, y0, dt, theta, out, (cudaStream_t)stream);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "bode_interpolate_tab");
}

extern "C" int bode_program_initial_step(const bode_program* prog, const bode_dynamics* dyn,
                                         int64_t n, int64_t d, const double* t0, const double* y0,
                                         int32_t order, const double* atol_v,
                                         const double* rtol_v, double atol, double rtol,
                                         const double* direction, double* dt, double* f0,
                                         void* stream) {
  if (!prog || !dyn || n < 1 || d != program_desc(prog).d || !t0 || !y0 || !direction || !dt || !f0)
    return fail(BODE_EINVAL, "bode_program_initial_step: invalid arguments");
  const cudaError_t e = program_initial_step(prog, make_dyn(*dyn, prog), n, t0, y0, order, atol_v,
                                             rtol_v, atol, rtol, direction, dt, f0,
                                             (cudaStream_t)stream);
  if (e == cudaErrorNotSupported) return fail(BODE_EINVAL, "program was not compiled with BODE_PROGRAM_UNITS");
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "bode_program_initial_step");
}

extern "C" int bode_eval_dynamics(const bode_dynamics* dyn, int64_t n, int64_t d, const double* t,
                                  const double* y, double* out, void* stream) {
  if (!dyn || n < 1 || d < 1 || !t || !y || !out)
    return fail(BODE_EINVAL, "bode_eval_dynamics: invalid arguments");
  if (dyn->kind == BODE_DYN_MLP || dyn->kind == BODE_DYN_PROGRAM || !valid_kind(dyn->kind))
    return fail(BODE_EUNSUPPORTED, "bode_eval_dynamics: registered analytic functors only");
  const cudaError_t e = unit_eval_dynamics(make_dyn(*dyn), n, d, t, y, out, (cudaStream_t)stream);
  return e == cudaSuccess ? BODE_OK : cuda_fail(e, "bode_eval_dynamics");
}
