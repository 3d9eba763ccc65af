"""ctypes front end of the C oracle (``bode_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU legs as the checker / CPU baseline, never by the
product package.  Parity status: PINNED -- ``tests/test_oracle_golden.py``
checks this oracle bit for bit against golden vectors produced by running
the reference (``tests/golden/make_golden.py``).

The argument struct is declared here independently of the product's
``_abi.py`` (a layout test checks both against ``include/bode.h``).
"""

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

RUNNING, SUCCESS, MAX_STEPS_EXCEEDED, STEP_UNDERFLOW, INFINITE_DYNAMICS = range(5)
METHODS = {"dopri5": 0, "tsit5": 1, "heun": 2}
DYN = {"vdp": 1, "lorenz": 2, "zero": 3, "const": 4, "linear": 5, "linear_cos": 6,
       "linear_sin": 7, "relax_cos": 8, "square": 9, "logistic": 10, "sin_plus_t": 11,
       "harmonic": 12, "damped": 13, "mlp": 20}
# named parameter slots per dynamics (include/bode.h)
SLOTS = {"vdp": ("mu",), "lorenz": ("sigma", "rho", "beta"), "const": ("c",),
         "linear": ("lam",), "linear_cos": ("lam", "amp", "omega"),
         "linear_sin": ("lam", "amp", "omega"), "relax_cos": ("lam", "omega"),
         "square": ("thr",)}


class Dyn(C.Structure):
    _fields_ = [("kind", C.c_int32), ("inst_mask", C.c_uint32),
                ("inst_params", C.c_void_p), ("shared_params", C.c_double * 8),
                ("W1", C.c_void_p), ("b1", C.c_void_p), ("W2", C.c_void_p),
                ("b2", C.c_void_p), ("hidden", C.c_int64)]


class Ctrl(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("beta3", C.c_double),
                ("safety", C.c_double), ("factor_min", C.c_double),
                ("factor_max", C.c_double), ("update_history_on_reject", C.c_int32),
                ("_pad", C.c_int32)]


class Args(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("method", C.c_int32), ("mode", C.c_int32),
                ("dt0_mode", C.c_int32), ("n", C.c_int64), ("d", C.c_int64),
                ("dyn", Dyn), ("ctrl", Ctrl),
                ("y0", C.c_void_p), ("t_start", C.c_void_p), ("t_end", C.c_void_p),
                ("t_eval", C.c_void_p), ("t_eval_offsets", C.c_void_p),
                ("t_eval_len", C.c_int64), ("atol_v", C.c_void_p), ("rtol_v", C.c_void_p),
                ("atol", C.c_double), ("rtol", C.c_double), ("max_steps", C.c_int64),
                ("dt0", C.c_double), ("dt0_v", C.c_void_p), ("order", C.c_void_p),
                ("ys", C.c_void_p), ("n_emitted", C.c_void_p), ("n_steps", C.c_void_p),
                ("n_accepted", C.c_void_p), ("final_dt", C.c_void_p),
                ("status", C.c_void_p), ("n_f_evals", C.c_void_p),
                ("trace_t", C.c_void_p), ("trace_dt", C.c_void_p),
                ("trace_accept", C.c_void_p), ("trace_cap", C.c_int64),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("stream", C.c_void_p), ("threads_per_block", C.c_int32),
                ("blocks", C.c_int32), ("cost_hint", C.c_void_p),
                ("pipeline_chunks", C.c_int32), ("_pad2", C.c_int32),
                ("max_iterations_out", C.c_void_p), ("refresh_map_out", C.c_void_p),
                ("reserved_mlp", C.c_int32), ("_pad3", C.c_int32),
                ("prof_event_start", C.c_void_p), ("prof_event_stop", C.c_void_p),
                ("launch_count_out", C.c_void_p),
                ("traj", C.c_void_p), ("traj_offsets", C.c_void_p),
                ("program", C.c_void_p), ("traj_stages", C.c_void_p)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.oracle_solve.argtypes = [C.POINTER(Args), C.c_int]
        P, I64, I, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
        sig = {
            "oracle_rk_step": [I, P, I64, I64, P, P, P, P, P, P, P],
            "oracle_interpolate": [I, I64, I64, P, P, P, P, P],
            "oracle_error_norm": [I64, I64, P, P, P, P, P, D, D, P],
            "oracle_adapt_step": [I64, P, I, P, P, P, P, P, P],
            "oracle_initial_step": [P, I64, I64, P, P, I, P, P, D, D, P, P, P],
        }
        for name, args in sig.items():
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def make_dyn(name, inst=None, shared=(), mlp=None, keep=None):
    """Registry spec -> Dyn struct.  ``inst`` (n, p) fills the first p slots
    per instance; ``shared`` fills the remaining slots in order."""
    d = Dyn()
    d.kind = DYN[name]
    nslots = len(SLOTS.get(name, ()))
    ninst = 0 if inst is None else inst.shape[1]
    vals = list(shared)
    sp = [0.0] * 8
    for k in range(ninst, nslots):
        sp[k] = float(vals[k - ninst]) if k - ninst < len(vals) else 0.0
    d.shared_params = (C.c_double * 8)(*sp)
    if ninst:
        ip = np.ascontiguousarray(inst, dtype=np.float64)
        keep.append(ip)
        d.inst_params = ip.ctypes.data
        d.inst_mask = (1 << ninst) - 1
    if name == "mlp":
        W1, b1, W2, b2 = [np.ascontiguousarray(x, dtype=np.float32) for x in mlp]
        keep.extend([W1, b1, W2, b2])
        d.W1, d.b1, d.W2, d.b2 = W1.ctypes.data, b1.ctypes.data, W2.ctypes.data, b2.ctypes.data
        d.hidden = W1.shape[0]
    return d


def solve(y0, t_start, t_end, t_eval, dyn, method="dopri5", atol=1e-6, rtol=1e-6,
          ctrl=None, max_steps=10_000, dt0=None, trace=False, nthreads=None,
          with_ys=True, with_refresh=False):
    """Solve on the CPU oracle.  ``t_eval`` is a list of arrays (ragged) or a
    single 1-D array shared by all instances.  Returns a dict shaped like
    the golden fixtures."""
    keep = []
    y0 = _f64(np.atleast_2d(y0))
    n, d = y0.shape
    ts = _f64(np.broadcast_to(t_start, (n,)))
    tn = _f64(np.broadcast_to(t_end, (n,)))
    a = Args()
    a.abi_version = 4
    a.method = METHODS[method]
    a.n, a.d = n, d
    a.dyn = make_dyn(dyn["name"], dyn.get("inst"), dyn.get("shared", ()), dyn.get("mlp"), keep)
    ctrl = ctrl or dict(betas=(1.0, 0.0, 0.0), safety=0.9, factor_min=0.2,
                        factor_max=10.0, hist=True)
    c = Ctrl()
    c.beta1, c.beta2, c.beta3 = ctrl["betas"]
    c.safety, c.factor_min, c.factor_max = ctrl["safety"], ctrl["factor_min"], ctrl["factor_max"]
    c.update_history_on_reject = int(ctrl["hist"])
    a.ctrl = c
    a.y0, a.t_start, a.t_end = _p(y0), _p(ts), _p(tn)
    if isinstance(t_eval, np.ndarray) and t_eval.ndim == 1:
        te_vals = _f64(t_eval)
        te_offs = None
        a.t_eval_len = te_vals.shape[0]
        n_rows = n * te_vals.shape[0]
    else:
        if t_eval is None:
            t_eval = [np.empty(0)] * n
        lens = np.array([len(x) for x in t_eval], dtype=np.int64)
        te_offs = np.zeros(n + 1, dtype=np.int64)
        te_offs[1:] = np.cumsum(lens)
        te_vals = _f64(np.concatenate([np.asarray(x, float) for x in t_eval])
                       if te_offs[-1] else np.zeros(1))
        n_rows = int(te_offs[-1])
    a.t_eval, a.t_eval_offsets = _p(te_vals), _p(te_offs)
    atol_v = _f64(atol) if np.ndim(atol) else None
    rtol_v = _f64(rtol) if np.ndim(rtol) else None
    a.atol_v, a.rtol_v = _p(atol_v), _p(rtol_v)
    a.atol = 0.0 if atol_v is not None else float(atol)
    a.rtol = 0.0 if rtol_v is not None else float(rtol)
    a.max_steps = max_steps
    dt0_v = None
    if dt0 is None:
        a.dt0_mode = 0
    elif np.ndim(dt0) == 0:
        a.dt0_mode, a.dt0 = 1, float(dt0)
    else:
        dt0_v = _f64(dt0)
        a.dt0_mode, a.dt0_v = 2, _p(dt0_v)
    out = dict(
        ys=np.full((max(n_rows, 1), d), np.nan) if with_ys else None,
        n_emitted=np.zeros(n, np.int64), n_steps=np.zeros(n, np.int64),
        n_accepted=np.zeros(n, np.int64), final_dt=np.zeros(n),
        status=np.zeros(n, np.int64), n_f_evals=np.zeros(1, np.int64))
    a.ys = _p(out["ys"])
    a.n_emitted, a.n_steps, a.n_accepted = _p(out["n_emitted"]), _p(out["n_steps"]), _p(out["n_accepted"])
    a.final_dt, a.status, a.n_f_evals = _p(out["final_dt"]), _p(out["status"]), _p(out["n_f_evals"])
    cap = 0
    if trace:
        cap = max_steps
        out["trace_t"] = np.zeros((n, cap))
        out["trace_dt"] = np.zeros((n, cap))
        out["trace_accept"] = np.zeros((n, cap), np.uint8)
        a.trace_t, a.trace_dt, a.trace_accept = (_p(out["trace_t"]), _p(out["trace_dt"]),
                                                 _p(out["trace_accept"]))
    a.trace_cap = cap
    if with_refresh:
        out["max_iterations"] = np.zeros(1, np.int64)
        out["refresh_map"] = np.zeros(max_steps + 2, np.uint8)
        a.max_iterations_out = _p(out["max_iterations"])
        a.refresh_map_out = _p(out["refresh_map"])
    nthreads = nthreads or min(os.cpu_count() or 1, 64)
    lib().oracle_solve(C.byref(a), int(nthreads))
    if with_ys:
        out["ys"] = out["ys"][:n_rows]
    out["te_offs"] = te_offs
    return out


# ---------------------------------------------------------- unit ops ----
def rk_step(method, dyn, t, dt, y, f0):
    keep = []
    y = _f64(np.atleast_2d(y))
    n, d = y.shape
    D = make_dyn(dyn["name"], dyn.get("inst"), dyn.get("shared", ()), dyn.get("mlp"), keep)
    S = 2 if method == "heun" else 7
    t, dt, f0 = _f64(t), _f64(dt), _f64(f0)
    yn, err, k = np.zeros((n, d)), np.zeros((n, d)), np.zeros((S, n, d))
    lib().oracle_rk_step(METHODS[method], C.addressof(D), C.c_int64(n), C.c_int64(d),
                         _p(t), _p(dt), _p(y), _p(f0), _p(yn), _p(err), _p(k))
    return yn, err, k


def interpolate(method, k, y0, dt, theta):
    k, y0, dt, theta = _f64(k), _f64(y0), _f64(dt), _f64(theta)
    n, d = y0.shape
    out = np.zeros((n, d))
    lib().oracle_interpolate(METHODS[method], C.c_int64(n), C.c_int64(d), _p(k), _p(y0),
                             _p(dt), _p(theta), _p(out))
    return out


def error_norm(err, y0, y1, atol, rtol):
    err, y0, y1 = _f64(err), _f64(y0), _f64(y1)
    n, d = err.shape
    av = _f64(atol) if np.ndim(atol) else None
    rv = _f64(rtol) if np.ndim(rtol) else None
    out = np.zeros(n)
    lib().oracle_error_norm(C.c_int64(n), C.c_int64(d), _p(err), _p(y0), _p(y1), _p(av),
                            _p(rv), C.c_double(0.0 if av is not None else atol),
                            C.c_double(0.0 if rv is not None else rtol), _p(out))
    return out


def adapt_step(norm, error_order, betas, n1, n2, dt, safety=0.9, fmin=0.2, fmax=10.0,
               hist=True):
    c = Ctrl()
    c.beta1, c.beta2, c.beta3 = betas
    c.safety, c.factor_min, c.factor_max = safety, fmin, fmax
    c.update_history_on_reject = int(hist)
    norm = _f64(norm)
    n = norm.shape[0]
    acc = np.zeros(n, np.uint8)
    dtn = np.zeros(n)
    lib().oracle_adapt_step(C.c_int64(n), _p(norm), C.c_int(error_order), C.addressof(c),
                            _p(n1), _p(n2), _p(dt), _p(acc), _p(dtn))
    return acc.astype(bool), dtn


def initial_step(dyn, t0, y0, order, atol, rtol, direction):
    keep = []
    y0 = _f64(np.atleast_2d(y0))
    n, d = y0.shape
    D = make_dyn(dyn["name"], dyn.get("inst"), dyn.get("shared", ()), dyn.get("mlp"), keep)
    t0, direction = _f64(t0), _f64(direction)
    av = _f64(atol) if np.ndim(atol) else None
    rv = _f64(rtol) if np.ndim(rtol) else None
    dt, f0 = np.zeros(n), np.zeros((n, d))
    lib().oracle_initial_step(C.addressof(D), C.c_int64(n), C.c_int64(d), _p(t0), _p(y0),
                              C.c_int(order), _p(av), _p(rv),
                              C.c_double(0.0 if av is not None else atol),
                              C.c_double(0.0 if rv is not None else rtol), _p(direction),
                              _p(dt), _p(f0))
    return dt, f0
