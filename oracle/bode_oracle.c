/*
 * bode_oracle.c -- CPU restatement of the reference solve path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the parity tests, the
 * smoke test and bench.py's cpu_baseline / --impl reference leg use.  It is
 * never linked into, loaded by, or called from the product path
 * (paper_2210_12375_b200/), which fails loudly without its CUDA library.
 *
 * It restates batchode (the reference at /root/reference/pkg/src/batchode)
 * as one scalar state machine per instance -- exactly what one GPU lane
 * executes -- with every floating-point operation in the reference's NumPy
 * order and rounding (no FMA contraction: build with -ffp-contract=off).
 * Batch independence (reference tests/test_solver.py:140-168) makes the
 * per-instance restatement equal to the lockstep batched loop; the
 * batch-global n_f_evals is rebuilt from per-iteration refresh flags
 * (SURVEY.md §8(a) A8).  Parity is pinned against golden vectors produced
 * by running the reference itself (tests/golden/make_golden.py), with NumPy
 * pinned to libm pow (NPY_DISABLE_CPU_FEATURES, SURVEY.md finding 1).
 *
 * Function-by-function anchors (reference file:line):
 *   np_pairwise_sum   numpy add.reduce order used by np.mean (controller.py:141)
 *   error_norm        controller.py:120-142
 *   initial_step      controller.py:145-197
 *   adapt             controller.py:200-238 (+ NORM_FLOOR :26)
 *   rk_step           stepper.py:54-110
 *   interpolate       stepper.py:112-139
 *   solve_one         solver.py:148-206 (init), 208-282 (step_once), 284-322 (_emit)
 *   oracle_solve      solver.py:324-349 (run/solution), 352-369 (solve)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/bode.h"
#include "../paper_2210_12375_b200/csrc/tableau_coeffs.h"

#define NORM_FLOOR 1e-10
#define MAXS 7

typedef struct {
  int S, order, error_order, fsal, ninterp;
  double a[MAXS][MAXS], b[MAXS], berr[MAXS], c[MAXS], interp[MAXS][4];
} tab_t;

static void load_tab(int method, tab_t* t) {
  memset(t, 0, sizeof(*t));
#define FILL(NAME, UP)                                                   \
  t->S = BODE_##UP##_STAGES;                                             \
  t->order = BODE_##UP##_ORDER;                                          \
  t->error_order = BODE_##UP##_ERROR_ORDER;                              \
  t->fsal = BODE_##UP##_FSAL;                                            \
  t->ninterp = BODE_##UP##_NINTERP;                                      \
  for (int i = 0; i < t->S; i++) {                                       \
    t->b[i] = bode_##NAME##_b(i);                                        \
    t->berr[i] = bode_##NAME##_berr(i);                                  \
    t->c[i] = bode_##NAME##_c(i);                                        \
    for (int j = 0; j < t->S; j++) t->a[i][j] = bode_##NAME##_a(i, j);   \
    for (int j = 0; j < t->ninterp; j++) t->interp[i][j] = bode_##NAME##_interp(i, j); \
  }
  if (method == BODE_METHOD_DOPRI5) {
    FILL(dopri5, DOPRI5)
  } else if (method == BODE_METHOD_TSIT5) {
    FILL(tsit5, TSIT5)
  } else {
    FILL(heun, HEUN)
  }
#undef FILL
}

/* ---------------------------------------------------------- numpy ops -- */
/* np.maximum / np.minimum propagate NaN (unlike fmax/fmin) */
static inline double np_max(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}
static inline double np_min(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a <= b ? a : b;
}

/* numpy pairwise_sum (loops_utils.h.src), seeded with 0.0, block 128 */
static double np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
  }
}

/* array ** python-float as numpy evaluates it (fast_scalar_power paths) */
static inline double np_scalar_pow(double x, double e) {
  if (e == 0.0) return 1.0;
  if (e == 1.0) return x;
  if (e == -1.0) return 1.0 / x;
  if (e == 2.0) return x * x;
  if (e == 0.5) return sqrt(x);
  return pow(x, e);
}

/* ------------------------------------------------------------ dynamics -- */
typedef struct {
  int kind;
  double p[8];
  const bode_dynamics* dyn;
  int64_t d;
  float* scratch; /* MLP: H + d floats */
} dynf_t;

static void dyn_params(const bode_dynamics* dyn, int64_t i, double p[8]) {
  int ninst = __builtin_popcount(dyn->inst_mask);
  int r = 0;
  for (int k = 0; k < 8; k++) {
    if ((dyn->inst_mask >> k) & 1u) {
      p[k] = dyn->inst_params[i * ninst + r];
      r++;
    } else {
      p[k] = dyn->shared_params[k];
    }
  }
}

static void dyn_eval(dynf_t* F, double t, const double* y, double* out) {
  const int64_t d = F->d;
  const double* p = F->p;
  switch (F->kind) {
    case BODE_DYN_VDP: { /* problems.py:45-48 */
      double x = y[0], v = y[1];
      out[0] = v;
      out[1] = ((p[0] * (1.0 - x * x)) * v) - x;
      break;
    }
    case BODE_DYN_LORENZ: {
      double x = y[0], yy = y[1], z = y[2];
      out[0] = p[0] * (yy - x);
      out[1] = (x * (p[1] - z)) - yy;
      out[2] = (x * yy) - (p[2] * z);
      break;
    }
    case BODE_DYN_ZERO:
      for (int64_t j = 0; j < d; j++) out[j] = 0.0;
      break;
    case BODE_DYN_CONST:
      for (int64_t j = 0; j < d; j++) out[j] = p[0];
      break;
    case BODE_DYN_LINEAR:
      for (int64_t j = 0; j < d; j++) out[j] = p[0] * y[j];
      break;
    case BODE_DYN_LINEAR_COS: {
      double g = p[1] * cos(p[2] * t);
      for (int64_t j = 0; j < d; j++) out[j] = (p[0] * y[j]) + g;
      break;
    }
    case BODE_DYN_LINEAR_SIN: {
      double g = p[1] * sin(p[2] * t);
      for (int64_t j = 0; j < d; j++) out[j] = (p[0] * y[j]) + g;
      break;
    }
    case BODE_DYN_RELAX_COS: {
      double g = cos(p[1] * t);
      for (int64_t j = 0; j < d; j++) out[j] = p[0] * (y[j] - g);
      break;
    }
    case BODE_DYN_SQUARE:
      for (int64_t j = 0; j < d; j++) out[j] = (y[j] > p[0]) ? INFINITY : y[j] * y[j];
      break;
    case BODE_DYN_LOGISTIC:
      for (int64_t j = 0; j < d; j++) out[j] = y[j] * (1.0 - y[j]);
      break;
    case BODE_DYN_SIN_PLUS_T:
      for (int64_t j = 0; j < d; j++) out[j] = sin(y[j]) + t;
      break;
    case BODE_DYN_HARMONIC:
      out[0] = y[1];
      out[1] = -y[0];
      break;
    case BODE_DYN_DAMPED:
      out[0] = y[1];
      out[1] = (-y[0]) - ((0.1 * y[1]) * fabs(y[1]));
      break;
    case BODE_DYN_MLP: { /* fp32 MLP, fp64 state */
      const bode_dynamics* D = F->dyn;
      const int64_t H = D->hidden;
      float* yf = F->scratch;
      float* h = F->scratch + d;
      for (int64_t k = 0; k < d; k++) yf[k] = (float)y[k];
      for (int64_t j = 0; j < H; j++) {
        float acc = 0.0f;
        for (int64_t k = 0; k < d; k++) acc += yf[k] * D->W1[j * d + k];
        h[j] = tanhf(acc + D->b1[j]);
      }
      for (int64_t k = 0; k < d; k++) {
        float acc = 0.0f;
        for (int64_t j = 0; j < H; j++) acc += h[j] * D->W2[k * H + j];
        out[k] = (double)(acc + D->b2[k]);
      }
      break;
    }
    default:
      for (int64_t j = 0; j < d; j++) out[j] = NAN;
  }
}

static int all_finite(const double* v, int64_t d) {
  for (int64_t j = 0; j < d; j++)
    if (!isfinite(v[j])) return 0;
  return 1;
}

/* ---------------------------------------------------- controller.py ---- */
/* error_norm, controller.py:120-142 */
static double error_norm(const double* e, const double* y0, const double* y1, int64_t d,
                         double atol, double rtol, double* sq) {
  for (int64_t j = 0; j < d; j++) {
    double scale = atol + rtol * np_max(fabs(y0[j]), fabs(y1[j]));
    double r = e[j] / scale;
    sq[j] = r * r;
  }
  double norm = sqrt(np_pairwise_sum(sq, d) / (double)d);
  return isfinite(norm) ? norm : INFINITY;
}

/* initial_step, controller.py:145-197; returns dt, fills f0 */
static double initial_step(dynf_t* F, double t0, const double* y0, int order, double atol,
                           double rtol, double direction, double* f0, double* scr) {
  const int64_t d = F->d;
  double* sq = scr;
  double* y1 = scr + d;
  double* f1 = scr + 2 * d;
  dyn_eval(F, t0, y0, f0);
  int bad = !all_finite(f0, d);
  for (int64_t j = 0; j < d; j++) {
    double scale = atol + rtol * fabs(y0[j]);
    double q = y0[j] / scale;
    sq[j] = q * q;
  }
  double d0 = sqrt(np_pairwise_sum(sq, d) / (double)d);
  for (int64_t j = 0; j < d; j++) {
    double scale = atol + rtol * fabs(y0[j]);
    double q = f0[j] / scale;
    sq[j] = q * q;
  }
  double d1 = sqrt(np_pairwise_sum(sq, d) / (double)d);
  int degenerate = (d0 < 1e-5) || (d1 < 1e-5) || !isfinite(d1);
  double h0 = degenerate ? 1e-6 : (0.01 * d0) / d1;
  double hd = h0 * direction;
  for (int64_t j = 0; j < d; j++) y1[j] = y0[j] + hd * f0[j];
  dyn_eval(F, t0 + hd, y1, f1);
  for (int64_t j = 0; j < d; j++) {
    double scale = atol + rtol * fabs(y0[j]);
    double q = (f1[j] - f0[j]) / scale;
    sq[j] = q * q;
  }
  double d2 = sqrt(np_pairwise_sum(sq, d) / (double)d) / h0;
  double dmax = np_max(d1, d2);
  int small = (dmax <= 1e-15) || !isfinite(dmax);
  double h1 = small ? np_max(1e-6, h0 * 1e-3)
                    : np_scalar_pow(0.01 / dmax, 1.0 / (double)(order + 1));
  double dt = np_min(100.0 * h0, h1) * direction;
  return bad ? NAN : dt;
}

typedef struct {
  double e1, e2, e3, safety, fmin, fmax;
  int hist;
} ctrl_t;

static void make_ctrl(const bode_controller* c, int error_order, ctrl_t* k) {
  int kk = error_order + 1;
  k->e1 = (-c->beta1) / (double)kk;
  k->e2 = (-c->beta2) / (double)kk;
  k->e3 = (-c->beta3) / (double)kk;
  k->safety = c->safety;
  k->fmin = c->factor_min;
  k->fmax = c->factor_max;
  k->hist = c->update_history_on_reject;
}

/* adapt_step, controller.py:200-238: returns accept; updates n1/n2, *dt */
static int adapt(const ctrl_t* c, double norm, double* n1, double* n2, double* dt) {
  int accept = norm <= 1.0;
  double a = np_max(norm, NORM_FLOOR);
  double b = np_max(*n1, NORM_FLOOR);
  double g = np_max(*n2, NORM_FLOOR);
  double factor = ((c->safety * np_scalar_pow(a, c->e1)) * np_scalar_pow(b, c->e2)) *
                  np_scalar_pow(g, c->e3);
  if (!isfinite(factor)) factor = c->fmin;
  factor = np_min(np_max(factor, c->fmin), c->fmax);
  *dt = *dt * factor;
  if (c->hist || accept) {
    *n2 = *n1;
    *n1 = np_max(norm, NORM_FLOOR);
  }
  return accept;
}

/* ------------------------------------------------------- stepper.py ---- */
/* Stepper.step, stepper.py:54-110.  k: S*d, k[0] must hold f0 if fsal. */
static void rk_step(const tab_t* T, dynf_t* F, double t, double dt, const double* y,
                    double* k, double* acc, double* ys, double* y_next, double* err) {
  const int64_t d = F->d;
  if (!T->fsal) dyn_eval(F, t, y, k);
  for (int i = 1; i < T->S; i++) {
    for (int64_t c = 0; c < d; c++) {
      double s = T->a[i][0] * k[c];
      for (int j = 1; j < i; j++) s = s + T->a[i][j] * k[j * d + c];
      acc[c] = s;
      ys[c] = dt * s + y[c];
    }
    dyn_eval(F, t + T->c[i] * dt, ys, k + i * d);
  }
  for (int64_t c = 0; c < d; c++) {
    double s = T->b[0] * k[c];
    for (int i = 1; i < T->S; i++) s = s + T->b[i] * k[i * d + c];
    y_next[c] = y[c] + dt * s;
    double e = T->berr[0] * k[c];
    for (int i = 1; i < T->S; i++) e = e + T->berr[i] * k[i * d + c];
    err[c] = dt * e;
  }
}

/* Stepper.interpolate, stepper.py:112-139 (Horner, separate roundings) */
static void interpolate(const tab_t* T, int64_t d, const double* k, const double* y0,
                        double dt, double theta, double* out) {
  double w[MAXS];
  const int m = T->ninterp;
  for (int i = 0; i < T->S; i++) {
    double v = T->interp[i][m - 1];
    for (int j = m - 2; j >= 0; j--) {
      v = v * theta;
      v = v + T->interp[i][j];
    }
    w[i] = v * theta;
  }
  for (int64_t c = 0; c < d; c++) {
    double s = w[0] * k[c];
    for (int i = 1; i < T->S; i++) s = s + w[i] * k[i * d + c];
    out[c] = y0[c] + dt * s;
  }
}

/* ----------------------------------------------------------- solve ---- */
typedef struct {
  const bode_solve_args* A;
  tab_t T;
  ctrl_t C;
  int64_t lo, hi;
  uint8_t* refresh; /* (max_steps + 2) flags: iteration j needs a refresh */
  int64_t max_n;
} job_t;

static void solve_one(job_t* J, int64_t i, double* buf, float* fscr) {
  const bode_solve_args* A = J->A;
  const tab_t* T = &J->T;
  const int64_t d = A->d;
  double* y = buf;
  double* f0 = y + d;
  double* k = f0 + d;          /* S*d */
  double* acc = k + MAXS * d;  /* d */
  double* ys = acc + d;        /* d */
  double* y_next = ys + d;     /* d */
  double* err = y_next + d;    /* d */
  double* y_old = err + d;     /* d */
  double* out = y_old + d;     /* d */
  double* scr = out + d;       /* 3d */

  dynf_t F;
  F.kind = A->dyn.kind;
  F.dyn = &A->dyn;
  F.d = d;
  F.scratch = fscr;
  dyn_params(&A->dyn, i, F.p);

  const double atol = A->atol_v ? A->atol_v[i] : A->atol;
  const double rtol = A->rtol_v ? A->rtol_v[i] : A->rtol;
  double t = A->t_start[i];
  const double t_end = A->t_end[i];
  const double direction = (t_end - t) > 0 ? 1.0 : -1.0; /* np.sign, t_end != t_start */
  for (int64_t c = 0; c < d; c++) y[c] = A->y0[i * d + c];

  const double* te;
  int64_t m;
  double* ysi;
  if (A->t_eval_offsets) {
    te = A->t_eval + A->t_eval_offsets[i];
    m = A->t_eval_offsets[i + 1] - A->t_eval_offsets[i];
    ysi = A->ys ? A->ys + A->t_eval_offsets[i] * d : NULL;
  } else {
    te = A->t_eval;
    m = A->t_eval_len;
    ysi = A->ys ? A->ys + i * m * d : NULL;
  }

  double dt;
  if (A->dt0_mode == BODE_DT0_HEURISTIC) {
    dt = initial_step(&F, t, y, T->order, atol, rtol, direction, f0, scr);
  } else {
    dt = A->dt0_mode == BODE_DT0_SCALAR ? A->dt0 : A->dt0_v[i];
    dyn_eval(&F, t, y, f0);
    if (!all_finite(f0, d)) dt = NAN;
  }
  int status = BODE_RUNNING;
  if (!isfinite(dt)) {
    status = BODE_INFINITE_DYNAMICS;
    dt = 0.0;
  }
  int64_t cursor = 0;
  while (cursor < m && te[cursor] == t) { /* solver.py:201-205 */
    if (ysi)
      for (int64_t c = 0; c < d; c++) ysi[cursor * d + c] = y[c];
    cursor++;
  }
  double n1 = 1.0, n2 = 1.0;
  int64_t nsteps = 0, nacc = 0;
  const int64_t cap = A->trace_cap;

  while (status == BODE_RUNNING) {
    const int64_t j = nsteps;
    const double remaining = t_end - t;
    const int truncated = fabs(dt) >= fabs(remaining);
    const double dt_used = truncated ? remaining : dt;
    if (T->fsal)
      for (int64_t c = 0; c < d; c++) k[c] = f0[c];
    rk_step(T, &F, t, dt_used, y, k, acc, ys, y_next, err);
    const double norm = error_norm(err, y, y_next, d, atol, rtol, scr);
    double dtn = dt_used;
    const int accept = adapt(&J->C, norm, &n1, &n2, &dtn);
    nsteps++;
    if (cap > 0 && j < cap) {
      if (A->trace_t) A->trace_t[i * cap + j] = t;
      if (A->trace_dt) A->trace_dt[i * cap + j] = dt_used;
      if (A->trace_accept) A->trace_accept[i * cap + j] = (uint8_t)accept;
    }
    if (accept) {
      nacc++;
      const double t_old = t;
      for (int64_t c = 0; c < d; c++) {
        y_old[c] = y[c];
        y[c] = y_next[c];
      }
      t = truncated ? t_end : t_old + dt_used;
      if (T->fsal)
        for (int64_t c = 0; c < d; c++) f0[c] = k[(T->S - 1) * d + c];
      if (cursor < m && dt_used != 0.0) { /* _emit, solver.py:301-322 */
        while (cursor < m) {
          double theta = (te[cursor] - t_old) / dt_used;
          if (!(theta <= 1.0)) break;
          theta = np_max(theta, 0.0);
          if (ysi) interpolate(T, d, k, y_old, dt_used, theta, ysi + cursor * d);
          cursor++;
        }
      }
      if (truncated) status = BODE_SUCCESS;
    }
    dt = dtn;
    if (status == BODE_RUNNING && t + dt == t) status = BODE_STEP_UNDERFLOW;
    if (status == BODE_RUNNING && nsteps >= A->max_steps) status = BODE_MAX_STEPS_EXCEEDED;
    if (!accept && status == BODE_RUNNING) J->refresh[j + 1] = 1;
  }
  if (nsteps > J->max_n) J->max_n = nsteps;
  if (A->n_emitted) A->n_emitted[i] = cursor;
  if (A->n_steps) A->n_steps[i] = nsteps;
  if (A->n_accepted) A->n_accepted[i] = nacc;
  if (A->final_dt) A->final_dt[i] = dt;
  if (A->status) A->status[i] = status;
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  const int64_t d = J->A->d;
  double* buf = (double*)malloc(sizeof(double) * (size_t)((MAXS + 12) * d + 16));
  float* fscr = (float*)malloc(sizeof(float) * (size_t)(d + J->A->dyn.hidden + 16));
  for (int64_t i = J->lo; i < J->hi; i++) solve_one(J, i, buf, fscr);
  free(buf);
  free(fscr);
  return NULL;
}

/* Whole-batch solve on HOST buffers, instances split over nthreads. */
int oracle_solve(const bode_solve_args* A, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > A->n) nthreads = (int)(A->n > 0 ? A->n : 1);
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  tab_t T;
  load_tab(A->method, &T);
  ctrl_t C;
  make_ctrl(&A->ctrl, T.error_order, &C);
  for (int w = 0; w < nthreads; w++) {
    jobs[w].A = A;
    jobs[w].T = T;
    jobs[w].C = C;
    jobs[w].lo = A->n * w / nthreads;
    jobs[w].hi = A->n * (w + 1) / nthreads;
    jobs[w].refresh = (uint8_t*)calloc((size_t)A->max_steps + 2, 1);
    jobs[w].max_n = 0;
  }
  for (int w = 1; w < nthreads; w++) pthread_create(&th[w], NULL, worker, &jobs[w]);
  worker(&jobs[0]);
  for (int w = 1; w < nthreads; w++) pthread_join(th[w], NULL);
  int64_t max_n = 0, refreshes = 0;
  for (int w = 0; w < nthreads; w++)
    if (jobs[w].max_n > max_n) max_n = jobs[w].max_n;
  for (int64_t j = 1; j < max_n; j++) {
    int any = 0;
    for (int w = 0; w < nthreads; w++) any |= jobs[w].refresh[j];
    refreshes += any;
  }
  if (A->n_f_evals)
    A->n_f_evals[0] = T.fsal ? 1 + (int64_t)(T.S - 1) * max_n + refreshes
                             : 1 + (int64_t)T.S * max_n;
  if (A->max_iterations_out) A->max_iterations_out[0] = max_n;
  if (A->refresh_map_out)
    for (int64_t j = 0; j < A->max_steps + 2; j++) {
      uint8_t any = 0;
      for (int w = 0; w < nthreads; w++) any |= jobs[w].refresh[j];
      A->refresh_map_out[j] = any;
    }
  for (int w = 0; w < nthreads; w++) free(jobs[w].refresh);
  free(jobs);
  free(th);
  return 0;
}

/* --------------------------------------------- unit ops (host arrays) -- */
int oracle_rk_step(int method, const bode_dynamics* dyn, int64_t n, int64_t d,
                   const double* t, const double* dt, const double* y, const double* f0,
                   double* y_next, double* err, double* k) {
  tab_t T;
  load_tab(method, &T);
  double* kk = (double*)malloc(sizeof(double) * (size_t)(MAXS * d));
  double* acc = (double*)malloc(sizeof(double) * (size_t)(3 * d));
  float* fscr = (float*)malloc(sizeof(float) * (size_t)(d + dyn->hidden + 16));
  for (int64_t i = 0; i < n; i++) {
    dynf_t F = {dyn->kind, {0}, dyn, d, fscr};
    dyn_params(dyn, i, F.p);
    if (T.fsal)
      for (int64_t c = 0; c < d; c++) kk[c] = f0[i * d + c];
    rk_step(&T, &F, t[i], dt[i], y + i * d, kk, acc, acc + d, y_next + i * d, err + i * d);
    for (int s = 0; s < T.S; s++)
      for (int64_t c = 0; c < d; c++) k[(s * n + i) * d + c] = kk[s * d + c];
  }
  free(kk);
  free(acc);
  free(fscr);
  return 0;
}

int oracle_interpolate(int method, int64_t n, int64_t d, const double* k, const double* y0,
                       const double* dt, const double* theta, double* out) {
  tab_t T;
  load_tab(method, &T);
  double* kk = (double*)malloc(sizeof(double) * (size_t)(MAXS * d));
  for (int64_t i = 0; i < n; i++) {
    for (int s = 0; s < T.S; s++)
      for (int64_t c = 0; c < d; c++) kk[s * d + c] = k[(s * n + i) * d + c];
    interpolate(&T, d, kk, y0 + i * d, dt[i], theta[i], out + i * d);
  }
  free(kk);
  return 0;
}

int oracle_error_norm(int64_t n, int64_t d, const double* err, const double* y0,
                      const double* y1, const double* atol_v, const double* rtol_v,
                      double atol, double rtol, double* norm) {
  double* sq = (double*)malloc(sizeof(double) * (size_t)d);
  for (int64_t i = 0; i < n; i++)
    norm[i] = error_norm(err + i * d, y0 + i * d, y1 + i * d, d, atol_v ? atol_v[i] : atol,
                         rtol_v ? rtol_v[i] : rtol, sq);
  free(sq);
  return 0;
}

int oracle_adapt_step(int64_t n, const double* norm, int error_order,
                      const bode_controller* ctrl, double* n1, double* n2, double* dt,
                      uint8_t* accept, double* dt_next) {
  ctrl_t C;
  make_ctrl(ctrl, error_order, &C);
  for (int64_t i = 0; i < n; i++) {
    double x = dt[i];
    accept[i] = (uint8_t)adapt(&C, norm[i], &n1[i], &n2[i], &x);
    dt[i] = x;
    dt_next[i] = x;
  }
  return 0;
}

int oracle_initial_step(const bode_dynamics* dyn, int64_t n, int64_t d, const double* t0,
                        const double* y0, int order, const double* atol_v,
                        const double* rtol_v, double atol, double rtol,
                        const double* direction, double* dt, double* f0) {
  double* scr = (double*)malloc(sizeof(double) * (size_t)(3 * d));
  float* fscr = (float*)malloc(sizeof(float) * (size_t)(d + dyn->hidden + 16));
  for (int64_t i = 0; i < n; i++) {
    dynf_t F = {dyn->kind, {0}, dyn, d, fscr};
    dyn_params(dyn, i, F.p);
    dt[i] = initial_step(&F, t0[i], y0 + i * d, order, atol_v ? atol_v[i] : atol,
                         rtol_v ? rtol_v[i] : rtol, direction[i], f0 + i * d, scr);
  }
  free(scr);
  free(fscr);
  return 0;
}
