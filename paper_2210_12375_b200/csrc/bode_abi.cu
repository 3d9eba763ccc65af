// bode_abi.cu -- the extern "C" boundary (include/bode.h).
//
// Translates bode_solve_args into kernel parameters, validates what the
// reference validates (returning BODE_EINVAL where batchode raises
// ValueError), and sequences: workspace reset -> persistent solver ->
// n_f_evals finalisation, all asynchronous on the caller's stream.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "bode_dispatch.cuh"
#include "bode_mlp.cuh"
#include "bode_units.cuh"

using namespace bode;

namespace {
thread_local std::string g_err;

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

int stages_of(int method) { return method == BODE_METHOD_HEUN ? 2 : 7; }
int error_order_of(int method) { return method == BODE_METHOD_HEUN ? 1 : 4; }
int fsal_of(int method) { return method == BODE_METHOD_HEUN ? 0 : 1; }

DynParams make_dyn(const bode_dynamics& d) {
  DynParams p;
  p.kind = d.kind;
  p.inst_mask = d.inst_mask;
  p.n_inst = __builtin_popcount(d.inst_mask);
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
  return p;
}

bool valid_kind(int k) {
  return (k >= BODE_DYN_VDP && k <= BODE_DYN_DAMPED) || k == BODE_DYN_MLP;
}

int validate(const bode_solve_args* a) {
  if (!a) return fail(BODE_EINVAL, "null args");
  if (a->abi_version != BODE_ABI_VERSION) return fail(BODE_EINVAL, "abi_version mismatch");
  if (a->n < 1 || a->d < 1)
    return fail(BODE_EINVAL, "need at least one instance and one state component");
  if (a->method < BODE_METHOD_DOPRI5 || a->method > BODE_METHOD_HEUN)
    return fail(BODE_EINVAL, "unknown method");
  if (a->mode != BODE_MODE_EXACT && a->mode != BODE_MODE_FAST) return fail(BODE_EINVAL, "unknown mode");
  if (!valid_kind(a->dyn.kind)) return fail(BODE_EINVAL, "unknown dynamics");
  if (a->max_steps < 1) return fail(BODE_EINVAL, "max_steps must be at least 1");
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
  if (a->dyn.inst_mask && !a->dyn.inst_params) return fail(BODE_EINVAL, "per-instance params missing");
  if (a->dyn.kind == BODE_DYN_MLP &&
      (!a->dyn.W1 || !a->dyn.b1 || !a->dyn.W2 || !a->dyn.b2 || a->dyn.hidden < 1))
    return fail(BODE_EINVAL, "MLP weights required");
  return BODE_OK;
}

size_t ws_bytes(const bode_solve_args* a) {
  size_t b = Workspace::bytes(a->max_steps, a->n, a->d);
  if (a->dyn.kind == BODE_DYN_MLP) b += mlp_workspace_bytes(a);
  return b;
}

}  // namespace

extern "C" {

int bode_abi_version(void) { return BODE_ABI_VERSION; }

size_t bode_sizeof_args(void) { return sizeof(bode_solve_args); }

const char* bode_last_error(void) { return g_err.c_str(); }

size_t bode_workspace_size(const bode_solve_args* a) {
  if (validate(a) != BODE_OK) return 0;
  return ws_bytes(a);
}

int bode_solve(const bode_solve_args* a) {
  int rc = validate(a);
  if (rc != BODE_OK) return rc;
  const size_t need = ws_bytes(a);
  if (!a->workspace || a->workspace_bytes < need)
    return fail(BODE_EINVAL, "workspace too small (see bode_workspace_size)");
  cudaStream_t st = (cudaStream_t)a->stream;
  const size_t words = Workspace::bitmap_words(a->max_steps);
  cudaError_t e = cudaMemsetAsync(a->workspace, 0,
                                  Workspace::kHeader + Workspace::bitmap_bytes(a->max_steps), st);
  if (e != cudaSuccess) return cuda_fail(e, "workspace reset");

  SolveParams P;
  memset(&P, 0, sizeof(P));
  P.n = a->n;
  P.dyn = make_dyn(a->dyn);
  P.ctrl = make_ctrl(a->ctrl, error_order_of(a->method));
  P.y0 = a->y0;
  P.t_start = a->t_start;
  P.t_end = a->t_end;
  P.t_eval = a->t_eval;
  P.t_eval_offsets = a->t_eval_offsets;
  P.t_eval_len = a->t_eval_offsets ? 0 : a->t_eval_len;
  P.atol_v = a->atol_v;
  P.rtol_v = a->rtol_v;
  P.atol = a->atol;
  P.rtol = a->rtol;
  P.max_steps = a->max_steps;
  P.dt0_mode = a->dt0_mode;
  P.dt0 = a->dt0;
  P.dt0_v = a->dt0_v;
  P.order = a->order;
  P.ys = a->ys;
  P.n_emitted = a->n_emitted;
  P.n_steps = a->n_steps;
  P.n_accepted = a->n_accepted;
  P.final_dt = a->final_dt;
  P.status = a->status;
  P.trace_t = a->trace_t;
  P.trace_dt = a->trace_dt;
  P.trace_accept = a->trace_accept;
  P.trace_cap = a->trace_cap;
  char* ws = (char*)a->workspace;
  P.queue = (unsigned long long*)ws;
  P.max_n = (unsigned long long*)(ws + 8);
  P.refresh = (uint32_t*)(ws + Workspace::kHeader);
  P.f0 = (double*)(ws + Workspace::f0_offset(a->max_steps));
  // per-block shared bitmap when it fits comfortably (<= 32 KB)
  P.smem_words = words * 4 <= 32 * 1024 ? (int32_t)words : 0;

  if (a->dyn.kind == BODE_DYN_MLP) {
    e = mlp_solve(a, P, ws + Workspace::bytes(a->max_steps, a->n, a->d), st);
    if (e != cudaSuccess) return cuda_fail(e, "mlp solve");
  } else {
    switch (a->method) {
      case BODE_METHOD_DOPRI5: e = solve_dopri5(a->mode, a->dyn.kind, a->d, P, a->threads_per_block, a->blocks, st); break;
      case BODE_METHOD_TSIT5: e = solve_tsit5(a->mode, a->dyn.kind, a->d, P, a->threads_per_block, a->blocks, st); break;
      default: e = solve_heun(a->mode, a->dyn.kind, a->d, P, a->threads_per_block, a->blocks, st); break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "solve launch");
  }
  bode_finalize_kernel<<<1, 256, 0, st>>>(P.max_n, P.refresh, stages_of(a->method),
                                          fsal_of(a->method), a->n_f_evals);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "finalize launch");
  return BODE_OK;
}

int bode_solve_host(const bode_solve_args* h) {
  int rc = validate(h);
  if (rc != BODE_OK) return rc;
  const int64_t n = h->n, d = h->d;
  const int64_t n_te = h->t_eval_offsets ? h->t_eval_offsets[n] : h->t_eval_len;
  const int64_t ys_rows = h->t_eval_offsets ? n_te : n * h->t_eval_len;
  const int n_inst = __builtin_popcount(h->dyn.inst_mask);

  struct Blk {
    const void* src;
    void* dst_host;
    size_t bytes;
    size_t off;
  };
  std::vector<Blk> ins, outs;
  size_t total = 0;
  auto add = [&](std::vector<Blk>& v, const void* src, void* dsth, size_t bytes) -> size_t {
    const size_t off = total;
    v.push_back({src, dsth, bytes, off});
    total += (bytes + 255) & ~(size_t)255;
    return off;
  };
  bode_solve_args a = *h;
  std::vector<std::pair<const void**, size_t>> in_ptrs;
  auto in = [&](const void** field, size_t bytes) {
    if (*field && bytes) in_ptrs.push_back({field, add(ins, *field, nullptr, bytes)});
  };
  in((const void**)&a.y0, sizeof(double) * n * d);
  in((const void**)&a.t_start, sizeof(double) * n);
  in((const void**)&a.t_end, sizeof(double) * n);
  in((const void**)&a.t_eval, sizeof(double) * n_te);
  in((const void**)&a.t_eval_offsets, h->t_eval_offsets ? sizeof(int64_t) * (n + 1) : 0);
  in((const void**)&a.atol_v, sizeof(double) * n);
  in((const void**)&a.rtol_v, sizeof(double) * n);
  in((const void**)&a.dt0_v, a.dt0_mode == BODE_DT0_ARRAY ? sizeof(double) * n : 0);
  in((const void**)&a.order, sizeof(int64_t) * n);
  in((const void**)&a.dyn.inst_params, sizeof(double) * n * n_inst);
  if (h->dyn.kind == BODE_DYN_MLP) {
    const int64_t H = h->dyn.hidden;
    in((const void**)&a.dyn.W1, sizeof(float) * H * d);
    in((const void**)&a.dyn.b1, sizeof(float) * H);
    in((const void**)&a.dyn.W2, sizeof(float) * d * H);
    in((const void**)&a.dyn.b2, sizeof(float) * d);
  }
  std::vector<std::pair<void**, size_t>> out_ptrs;
  auto out = [&](void** field, size_t bytes) {
    if (*field && bytes) out_ptrs.push_back({field, add(outs, nullptr, *field, bytes)});
  };
  out((void**)&a.ys, sizeof(double) * ys_rows * d);
  out((void**)&a.n_emitted, sizeof(int64_t) * n);
  out((void**)&a.n_steps, sizeof(int64_t) * n);
  out((void**)&a.n_accepted, sizeof(int64_t) * n);
  out((void**)&a.final_dt, sizeof(double) * n);
  out((void**)&a.status, sizeof(int32_t) * n);
  out((void**)&a.n_f_evals, sizeof(int64_t));
  out((void**)&a.trace_t, sizeof(double) * n * h->trace_cap);
  out((void**)&a.trace_dt, sizeof(double) * n * h->trace_cap);
  out((void**)&a.trace_accept, sizeof(uint8_t) * n * h->trace_cap);
  const size_t ws_off = total;
  const size_t wsb = ws_bytes(h);
  total += wsb;

  cudaStream_t st = (cudaStream_t)h->stream;
  char* dev = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dev, total, st);
  if (e != cudaSuccess) return cuda_fail(e, "device allocation");
  for (auto& p : in_ptrs) {
    const Blk* b = nullptr;
    for (auto& x : ins)
      if (x.off == p.second) b = &x;
    e = cudaMemcpyAsync(dev + b->off, b->src, b->bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) break;
    *p.first = dev + b->off;
  }
  for (auto& p : out_ptrs) *p.first = dev + p.second;
  a.workspace = dev + ws_off;
  a.workspace_bytes = wsb;
  if (e == cudaSuccess) {
    rc = bode_solve(&a);
    if (rc == BODE_OK) {
      for (auto& b : outs) {
        e = cudaMemcpyAsync(b.dst_host, dev + b.off, b.bytes, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) break;
      }
    }
  }
  cudaFreeAsync(dev, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  if (rc != BODE_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "host<->device copy");
  if (e2 != cudaSuccess) return cuda_fail(e2, "solve");
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
