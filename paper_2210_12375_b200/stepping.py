"""The reference's stepping API on the device: ``BatchSolver`` and ``Stepper``.

``BatchSolver`` (reference ``pkg/src/batchode/solver.py:141-349``) drives the
batched loop one iteration at a time: ``step_once`` advances every running
instance by one attempted step and returns whether any instance is still
running, ``run`` iterates to completion, ``solution`` packages the result.
Here the per-instance state (t, y, FSAL cache, controller history and dt,
counters, t_eval cursor, status, ys, traces) lives in device memory; each
``step_once`` is ONE launch of ``bode_step_kernel`` (csrc/bode_stepper.cuh),
which runs the very Lane::step of the persistent solver, so a step_once
loop takes exactly the decisions ``solve`` takes (exact mode).  The
kernels come from a run-time program
(program.py) for the solver's (tableau, dynamics) pair -- any tableau and
any traceable NumPy callable.

``Stepper`` (stepper.py:40-139) is one embedded RK trial step on the full
batch plus dense output: the unit kernels with the tableau's coefficients
read from device memory (any ButcherTableau, no recompilation per
coefficient set).

Host-side attributes (``t``, ``y``, ``status``, ``ctrl``, ``n_steps``, ...)
are read from the device on access, as NumPy arrays, like the reference's.
"""

import numpy as np

from . import _abi
from .controller import PidCoefficients, Tolerances, integral_controller
from .dynamics import DeviceDynamics, as_device_dynamics, build_struct
from .program import STEP, UNITS, get_program
from .solver import DEFAULT_MAX_STEPS, IvpBatch, Solution, SolveStats, SolveStatus
from .tableau import ButcherTableau, dopri5, fsal_of, is_custom, method_of, stages_of
from .units import ControllerState, StepResult

__all__ = ["BatchSolver", "Stepper", "StepResult", "ControllerState", "rk_step", "interpolate"]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _abi.BodeLibraryError("the stepping API needs a CUDA device (no CPU fallback)")
    return torch


def tableau_struct(tab) -> "_abi.Tableau_":
    s = _abi.Tableau_()
    S = int(tab.stages)
    w = np.asarray(tab.interp_coeffs, dtype=np.float64)
    if S > _abi.TAB_MAX_STAGES or w.shape[1] > _abi.TAB_MAX_INTERP:
        raise NotImplementedError("device tableaus: at most 16 stages and 8 interpolant terms")
    s.stages, s.n_interp, s.fsal = S, w.shape[1], int(bool(tab.fsal))
    a = np.zeros((_abi.TAB_MAX_STAGES, _abi.TAB_MAX_STAGES))
    a[:S, :S] = np.asarray(tab.a, dtype=np.float64)
    s.a[:] = a.reshape(-1).tolist()
    for name in ("b", "b_err", "c"):
        v = np.zeros(_abi.TAB_MAX_STAGES)
        v[:S] = np.asarray(getattr(tab, name), dtype=np.float64)
        getattr(s, name)[:] = v.tolist()
    wi = np.zeros((_abi.TAB_MAX_STAGES, _abi.TAB_MAX_INTERP))
    wi[:S, :w.shape[1]] = w
    s.interp[:] = wi.reshape(-1).tolist()
    return s


def _tableau_dev(tab):
    torch = _torch()
    s = tableau_struct(tab)
    raw = np.frombuffer(bytes(s), dtype=np.uint8).copy()
    return torch.from_numpy(raw).to("cuda")


class Stepper:
    """Trial steps and dense output for one solve (stepper.py:40-139)."""

    def __init__(self, tableau: ButcherTableau, batch_size: int, n_features: int):
        self.tableau = tableau
        self.batch_size, self.n_features = batch_size, n_features

    def step(self, f, t, dt, y, f0) -> StepResult:
        """One embedded RK trial step on the full batch (stepper.py:54-110):
        stages in ascending order, every term of every sum included, non-finite
        stage values propagating into the error estimate."""
        torch = _torch()
        lib = _abi.load()
        tab = self.tableau
        y = np.atleast_2d(np.asarray(y, dtype=float))
        n, d = y.shape
        dyn = as_device_dynamics(f, n, d)
        S, fsal = int(tab.stages), bool(tab.fsal)
        prog = get_program("dopri5", dyn, d, UNITS)  # dynamics only; the tableau is data
        keep = []
        dev = lambda a: (keep.append(torch.tensor(np.asarray(a, dtype=np.float64))  # noqa: E731
                                     .to("cuda")), keep[-1].data_ptr())[1]
        ds = build_struct(dyn, n, keep, device_arrays=dev)
        tt = dev(np.broadcast_to(np.asarray(t if t is not None else 0.0, dtype=float), (n,)))
        dtt = dev(np.broadcast_to(np.asarray(dt, dtype=float), (n,)))
        yy = dev(y)
        ff = dev(np.broadcast_to(np.asarray(f0, dtype=float), (n, d))) if (fsal and f0 is not None) \
            else None
        if fsal and ff is None:
            raise ValueError("an FSAL tableau needs f0 = f(t, y)")
        tabd = _tableau_dev(tab)
        yn = torch.empty((n, d), dtype=torch.float64, device="cuda")
        err = torch.empty_like(yn)
        k = torch.empty((S, n, d), dtype=torch.float64, device="cuda")
        _abi.check(lib.bode_program_rk_step(prog.handle, tabd.data_ptr(), _abi.C.addressof(ds), n,
                                            d, tt, dtt, yy, ff, yn.data_ptr(), err.data_ptr(),
                                            k.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream))
        kk = k.cpu().numpy()
        return StepResult(y_next=yn.cpu().numpy(), error_estimate=err.cpu().numpy(),
                          stage_derivs=kk, f_next=kk[S - 1] if fsal else None,
                          n_evals=S - 1 if fsal else S)

    def interpolate(self, step: StepResult, y0, dt, theta) -> np.ndarray:
        """Dense output y(t + theta*dt) (stepper.py:112-139); theta outside
        [0, 1] raises ValueError as in the reference (:126-127)."""
        torch = _torch()
        lib = _abi.load()
        theta = np.asarray(theta, dtype=float)
        if np.any((theta < 0.0) | (theta > 1.0)):
            raise ValueError("theta must lie in [0, 1]")
        y0 = np.atleast_2d(np.asarray(y0, dtype=float))
        n, d = y0.shape
        to = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")  # noqa: E731
        k, yy = to(step.stage_derivs), to(y0)
        dtt, th = to(np.broadcast_to(dt, (n,))), to(np.broadcast_to(theta, (n,)))
        tabd = _tableau_dev(self.tableau)
        out = torch.empty((n, d), dtype=torch.float64, device="cuda")
        _abi.check(lib.bode_interpolate_tab(tabd.data_ptr(), n, d, k.data_ptr(), yy.data_ptr(),
                                            dtt.data_ptr(), th.data_ptr(), out.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream))
        return out.cpu().numpy()


def rk_step(f, tableau: ButcherTableau, t, dt, y, f0) -> StepResult:
    """One-off trial step (stepper.py:142-152)."""
    n, d = np.atleast_2d(y).shape
    return Stepper(tableau, n, d).step(f, t, dt, y, f0)


def interpolate(step: StepResult, tableau: ButcherTableau, y0, dt, theta) -> np.ndarray:
    """Dense output without an explicit stepper (stepper.py:155-165)."""
    n, d = np.atleast_2d(y0).shape
    return Stepper(tableau, n, d).interpolate(step, y0, dt, theta)


class BatchSolver:
    """The batched integration loop, one instance per batch row
    (solver.py:141-349), on device state."""

    def __init__(self, problem: IvpBatch, f, tableau: ButcherTableau | None = None,
                 tol: Tolerances | None = None, controller: PidCoefficients | None = None,
                 max_steps: int = DEFAULT_MAX_STEPS, dt0=None, record_trace: bool = False,
                 *, mode: str = "exact"):
        if max_steps < 1:
            raise ValueError("max_steps must be at least 1")
        torch = _torch()
        self.problem = problem
        self.tableau = tableau if tableau is not None else dopri5()
        self.tol = tol if tol is not None else Tolerances()
        self.controller = controller if controller is not None else integral_controller()
        self.max_steps = max_steps
        self.record_trace = record_trace
        self.mode = mode
        self.direction = problem.direction
        n, d = problem.batch_size, problem.n_features
        self._n, self._d = n, d
        self._method = method_of(self.tableau)
        self._S, self._fsal = stages_of(self._method), fsal_of(self._method)
        self._f = f
        dev = torch.device("cuda", torch.cuda.current_device())
        f64 = dict(dtype=torch.float64, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        self._keep = []

        def up(x, dtype=np.float64):
            t_ = torch.as_tensor(np.ascontiguousarray(x, dtype=dtype)).to(dev)
            self._keep.append(t_)
            return t_

        a = self._args = _abi.SolveArgs()
        a.abi_version = _abi.ABI_VERSION
        a.mode = _abi.MODE[mode]
        a.n, a.d = n, d
        self._y0 = up(problem.y0)
        self._ts = up(problem.t_start)
        self._tn = up(problem.t_end)
        a.y0, a.t_start, a.t_end = self._y0.data_ptr(), self._ts.data_ptr(), self._tn.data_ptr()
        te = problem.te_values
        if te.size:
            tev = up(te)
            a.t_eval = tev.data_ptr()
            if problem.te_shared:
                a.t_eval_len = te.size
                rows = n * te.size
            else:
                offs = up(problem.te_offsets, np.int64)
                a.t_eval_offsets = offs.data_ptr()
                rows = int(problem.te_offsets[-1])
        else:
            rows = 0
        self._rows = rows
        from .solver import _controller_struct, _tol_arrays
        (av, a.atol), (rv, a.rtol) = _tol_arrays(self.tol, n)
        if av is not None:
            a.atol_v = up(av).data_ptr()
        if rv is not None:
            a.rtol_v = up(rv).data_ptr()
        a.ctrl = _controller_struct(self.controller)
        a.max_steps = int(max_steps)
        if dt0 is None:
            a.dt0_mode = _abi.DT0_HEURISTIC
        elif np.ndim(dt0) == 0:
            a.dt0_mode, a.dt0 = _abi.DT0_SCALAR, float(dt0)
        else:
            a.dt0_mode = _abi.DT0_ARRAY
            a.dt0_v = up(np.broadcast_to(np.asarray(dt0, dtype=float), (n,))).data_ptr()
        # outputs (they double as loop state)
        self._ys_dev = torch.zeros((max(rows, 1), d), **f64)
        self._n_emitted = torch.zeros(n, **i64)
        self._n_steps = torch.zeros(n, **i64)
        self._n_acc = torch.zeros(n, **i64)
        self._final_dt = torch.zeros(n, **f64)
        self._status = torch.zeros(n, **i64)
        self._nfe_dev = torch.zeros(1, **i64)
        a.ys = self._ys_dev.data_ptr() if rows else None
        a.n_emitted, a.n_steps = self._n_emitted.data_ptr(), self._n_steps.data_ptr()
        a.n_accepted, a.final_dt = self._n_acc.data_ptr(), self._final_dt.data_ptr()
        a.status, a.n_f_evals = self._status.data_ptr(), self._nfe_dev.data_ptr()
        if record_trace:
            cap = int(max_steps)
            self._tr_t = torch.zeros((n, cap), **f64)
            self._tr_dt = torch.zeros((n, cap), **f64)
            self._tr_acc = torch.zeros((n, cap), dtype=torch.uint8, device=dev)
            a.trace_t, a.trace_dt = self._tr_t.data_ptr(), self._tr_dt.data_ptr()
            a.trace_accept, a.trace_cap = self._tr_acc.data_ptr(), cap
        # loop state
        self._t = self._ts.clone()
        self._y = self._y0.clone()
        self._f0 = torch.zeros((n, d), **f64)
        self._n1 = torch.ones(n, **f64)
        self._n2 = torch.ones(n, **f64)
        self._te_next = torch.zeros(n, **f64)
        self._fsal_valid = torch.ones(n, dtype=torch.uint8, device=dev)
        self._flags = torch.zeros(2, dtype=torch.int32, device=dev)
        self._flags_h = torch.zeros(2, dtype=torch.int32).pin_memory()
        s = self._state = _abi.StepState()
        s.t, s.y, s.f0 = self._t.data_ptr(), self._y.data_ptr(), self._f0.data_ptr()
        s.norm_prev, s.norm_prev2 = self._n1.data_ptr(), self._n2.data_ptr()
        s.te_next, s.fsal_valid = self._te_next.data_ptr(), self._fsal_valid.data_ptr()
        s.flags = self._flags.data_ptr()
        self._bind_dynamics(STEP)
        lib = _abi.load()
        _abi.check(lib.bode_step_begin(_abi.C.byref(a), _abi.C.byref(s)))
        self.n_f_evals = 1  # the FSAL seed (solver.py:184)
        self._iterations = 0
        self._running = bool((self._status == SolveStatus.RUNNING).any().item())

    # ------------------------------------------------------------ dynamics --
    @property
    def f(self):
        return self._f

    @f.setter
    def f(self, f):  # re-bound lazily: a finished solver never evaluates f (solver.py:215)
        self._f = f
        self._dyn_bound = None

    def _bind_dynamics(self, kernels):
        torch = _torch()
        dyn = as_device_dynamics(self._f, self._n, self._d)
        prog = get_program(self._method, dyn, self._d, kernels)
        a = self._args
        a.method = _abi.METHOD_CUSTOM if is_custom(self._method) else _abi.METHOD[self._method]
        a.program = prog.handle
        keep = []
        dev = lambda x: (keep.append(torch.as_tensor(np.ascontiguousarray(x)).to("cuda")),  # noqa: E731
                         keep[-1].data_ptr())[1]
        a.dyn = build_struct(dyn, self._n, keep, device_arrays=dev)
        self._dyn_bound = (prog, keep)

    # -------------------------------------------------------------- loop ----
    def step_once(self) -> bool:
        """One loop iteration (solver.py:208-282); False once every instance
        terminated (and then nothing is evaluated)."""
        if not self._running:
            return False
        torch = _torch()
        if self._dyn_bound is None:
            self._bind_dynamics(STEP)
        lib = _abi.load()
        _abi.check(lib.bode_step_once(_abi.C.byref(self._args), _abi.C.byref(self._state)))
        self._flags_h.copy_(self._flags, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        flags = self._flags_h.tolist()
        self.n_f_evals += (self._S - 1 if self._fsal else self._S) + (1 if flags[1] else 0)
        self._iterations += 1
        self._running = bool(flags[0])
        return self._running

    def run(self) -> Solution:
        """Iterate :meth:`step_once` to completion and package the result
        (solver.py:324-330).  (``solve`` runs the same loop as one
        persistent-kernel launch.)"""
        while self.step_once():
            pass
        return self.solution()

    # ------------------------------------------------------- host views ----
    def _np(self, t):
        return t.cpu().numpy()

    @property
    def t(self):
        return self._np(self._t)

    @property
    def y(self):
        return self._np(self._y)

    @property
    def f0(self):
        return self._np(self._f0)

    @property
    def fsal_valid(self):
        return self._np(self._fsal_valid).astype(bool)

    @property
    def status(self):
        return self._np(self._status)

    @property
    def n_steps(self):
        return self._np(self._n_steps)

    @property
    def n_accepted(self):
        return self._np(self._n_acc)

    @property
    def _cursor(self):
        return self._np(self._n_emitted)

    @property
    def ctrl(self) -> ControllerState:
        return ControllerState(self._np(self._n1), self._np(self._n2), self._np(self._final_dt))

    @property
    def stepper(self) -> Stepper:
        return Stepper(self.tableau, self._n, self._d)

    def _ys_rows(self):
        d = self._d
        ys = self._np(self._ys_dev)[:self._rows].reshape(-1, d)
        ne = self.n_emitted_np()
        if self.problem.te_shared:
            m = self.problem.te_values.size
            return [ys[i * m:i * m + ne[i]] for i in range(self._n)]
        o = self.problem.te_offsets
        return [ys[o[i]:o[i] + ne[i]] for i in range(self._n)]

    def n_emitted_np(self):
        return self._np(self._n_emitted)

    def _trace(self, buf, cast=None):
        ns = self.n_steps
        v = self._np(buf)
        out = [list(v[i, :ns[i]]) for i in range(self._n)]
        if cast is not None:
            out = [[cast(x) for x in row] for row in out]
        return out

    @property
    def _trace_t(self):
        return self._trace(self._tr_t, float)

    @property
    def _trace_dt(self):
        return self._trace(self._tr_dt, float)

    @property
    def _trace_accept(self):
        return self._trace(self._tr_acc, bool)

    def solution(self) -> Solution:
        n, d = self._n, self._d
        ne = self.n_emitted_np()
        extra = {}
        if self.record_trace:
            ns = self.n_steps
            tt, tdt, tac = self._np(self._tr_t), self._np(self._tr_dt), self._np(self._tr_acc)
            extra["trace_t"] = [tt[i, :ns[i]].copy() for i in range(n)]
            extra["trace_dt"] = [tdt[i, :ns[i]].copy() for i in range(n)]
            extra["trace_accept"] = [tac[i, :ns[i]].astype(bool) for i in range(n)]
        stats = SolveStats(n_steps=self.n_steps, n_accepted=self.n_accepted,
                           n_f_evals=np.full(n, self.n_f_evals, dtype=np.int64),
                           final_dt=self._np(self._final_dt), extra=extra)
        ys = self._np(self._ys_dev)[:self._rows]
        if self.problem.te_shared or self.problem.te_values.size == 0:
            offs, shared = None, self.problem.te_values.size
        else:
            offs, shared = self.problem.te_offsets, 0
        return Solution(ys, offs, shared, ne, stats, self.status, d)


# ``solver._ys`` in the reference is a list (per instance) of emitted rows
BatchSolver._ys = property(lambda self: self._ys_list_rows())


def _ys_list_rows(self):
    return [list(rows) for rows in self._ys_rows()]


BatchSolver._ys_list_rows = _ys_list_rows
