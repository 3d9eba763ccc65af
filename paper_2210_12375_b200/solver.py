"""Batched independent ODE solve: the reference-facing entry points.

Mirrors ``batchode.solver`` (reference ``pkg/src/batchode/solver.py``):
``SolveStatus`` (:45-50), ``IvpBatch`` (:53-101, same validation and
ValueErrors), ``SolveStats`` (:104-119), ``Solution`` (:122-138) and
``solve`` (:352-369, same signature and defaults).  The loop itself
(``BatchSolver`` :141-349) is the persistent sm_100a kernel behind
``bode_solve`` -- one C-ABI call per solve, no per-step launches.

Two call styles:
  * ``solve(problem, f, ...)``: NumPy in, NumPy out, exactly like the
    reference.  It goes through ``bode_solve_host`` (host buffers, copies
    inside the call) -- the end-to-end path.
  * ``solve_device(...)``: torch CUDA tensors in/out, asynchronous on the
    current stream, no host sync -- the device-resident path.
"""

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .controller import PidCoefficients, Tolerances, integral_controller
from .dynamics import MLP_TILE, DeviceDynamics, as_device_dynamics, build_struct, mlp_pad
from .tableau import is_custom, method_of

__all__ = ["DEFAULT_MAX_STEPS", "SolveStatus", "IvpBatch", "SolveStats", "Solution",
           "solve", "solve_joint", "solve_device", "adjoint_device", "pinned", "host_empty"]

DEFAULT_MAX_STEPS = 10_000
# MLP path: fused persistent tcgen05 kernel (auto when d == 64), lockstep
# per-stage tcgen05 3xTF32 kernels, or lockstep CUDA-core fp32


# host arrays in [PIN_MIN_BYTES, PIN_MAX_BYTES] are page-locked (DMA at ~50
# GB/s instead of a driver-staged pageable copy at 13-19 GB/s, measured on
# the B200 box); below the minimum the pinned-allocator call costs more than
# the copy it saves
PIN_MIN_BYTES = 1 << 20
PIN_MAX_BYTES = 16 << 30
# resident lanes of the persistent kernel (148 SMs x 5 blocks x 128): the
# share of work one lane gets, used to decide whether chunking pays
_LANES = 148 * 5 * 128


def host_empty(shape, dtype=np.float64) -> np.ndarray:
    """Uninitialised host array for solver outputs; page-locked when a CUDA
    device is present and the array is at most ``PIN_MAX_BYTES``.  Pinned
    blocks come from torch's caching host allocator, so repeated solves reuse
    the pinning instead of paying for it (the NumPy array keeps the block
    alive and returns it to the cache when collected)."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    if PIN_MIN_BYTES <= nbytes <= PIN_MAX_BYTES:
        try:
            import torch
            if torch.cuda.is_available():
                t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
                return t.numpy().view(dtype).reshape(shape)
        except ImportError:
            pass
    return np.empty(shape, dtype)


def pinned(x, dtype=None) -> np.ndarray:
    """Copy of ``x`` in page-locked host memory (see :func:`host_empty`):
    inputs staged this way are copied to the device by DMA directly."""
    x = np.asarray(x, dtype=dtype)
    out = host_empty(x.shape, x.dtype)
    out[...] = x
    return out


class SolveStatus(enum.IntEnum):
    RUNNING = 0
    SUCCESS = 1
    MAX_STEPS_EXCEEDED = 2
    STEP_UNDERFLOW = 3
    INFINITE_DYNAMICS = 4


class IvpBatch:
    """A batch of independent initial value problems (solver.py:53-101).

    ``t_eval`` is, as in the reference, a list of per-instance sorted arrays
    (ragged, possibly empty).  For large batches it may also be given as a
    2-D array (n, m) -- every instance m points -- or a 1-D array shared by
    all instances; these are validated vectorised and passed to the device
    without building per-instance lists.
    """

    def __init__(self, y0, t_start, t_end, t_eval):
        self.y0 = np.atleast_2d(np.asarray(y0, dtype=float))
        self.t_start = np.asarray(t_start, dtype=float)
        self.t_end = np.asarray(t_end, dtype=float)
        n, d = self.y0.shape
        if n < 1 or d < 1:
            raise ValueError("need at least one instance and one state component")
        if self.t_start.shape != (n,) or self.t_end.shape != (n,):
            raise ValueError("t_start/t_end must have one entry per instance")
        if np.any(self.t_end == self.t_start):
            raise ValueError("t_end must differ from t_start for every instance")
        direction = np.sign(self.t_end - self.t_start)
        span = np.abs(self.t_end - self.t_start)
        self._te_list = None
        if isinstance(t_eval, np.ndarray) and t_eval.ndim == 1 and t_eval.dtype != object:
            te = np.asarray(t_eval, dtype=float)  # shared by every instance
            self.te_values, self.te_offsets, self.te_shared = te, None, True
            if te.size:
                pos = (te[None, :] - self.t_start[:, None]) * direction[:, None]
                self._check_dense(pos, span)
        elif isinstance(t_eval, np.ndarray) and t_eval.ndim == 2:
            te = np.ascontiguousarray(t_eval, dtype=float)
            if te.shape[0] != n:
                raise ValueError("t_eval must have one (possibly empty) array per instance")
            m = te.shape[1]
            self.te_values = te.reshape(-1)
            self.te_offsets = host_empty(n + 1, np.int64)
            np.multiply(np.arange(n + 1, dtype=np.int64), m, out=self.te_offsets)
            self.te_shared = False
            if m:
                pos = (te - self.t_start[:, None]) * direction[:, None]
                self._check_dense(pos, span)
        else:
            if len(t_eval) != n:
                raise ValueError("t_eval must have one (possibly empty) array per instance")
            lst = [np.asarray(te, dtype=float) for te in t_eval]
            for i, te in enumerate(lst):
                if te.size == 0:
                    continue
                pos = (te - self.t_start[i]) * direction[i]
                if np.any(np.diff(pos) < 0):
                    raise ValueError(f"t_eval of instance {i} is not sorted in integration direction")
                if pos[0] < 0 or pos[-1] > span[i]:
                    raise ValueError(f"t_eval of instance {i} leaves the integration interval")
            self._te_list = lst
            lens = np.fromiter((te.size for te in lst), dtype=np.int64, count=n)
            self.te_offsets = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(lens, out=self.te_offsets[1:])
            self.te_values = (np.concatenate(lst) if self.te_offsets[-1] else np.zeros(0))
            self.te_shared = False

    @staticmethod
    def _check_dense(pos, span):
        bad = np.any(np.diff(pos, axis=1) < 0, axis=1)
        if np.any(bad):
            i = int(np.flatnonzero(bad)[0])
            raise ValueError(f"t_eval of instance {i} is not sorted in integration direction")
        bad = (pos[:, 0] < 0) | (pos[:, -1] > span)
        if np.any(bad):
            i = int(np.flatnonzero(bad)[0])
            raise ValueError(f"t_eval of instance {i} leaves the integration interval")

    @property
    def t_eval(self) -> list:
        if self._te_list is None:
            n = self.batch_size
            if self.te_shared:
                self._te_list = [self.te_values] * n
            else:
                o = self.te_offsets
                self._te_list = [self.te_values[o[i]:o[i + 1]] for i in range(n)]
        return self._te_list

    @property
    def batch_size(self) -> int:
        return self.y0.shape[0]

    @property
    def n_features(self) -> int:
        return self.y0.shape[1]

    @property
    def direction(self) -> np.ndarray:
        return np.sign(self.t_end - self.t_start)

    def eval_counts(self) -> np.ndarray:
        n = self.batch_size
        if self.te_shared:
            return np.full(n, self.te_values.size, dtype=np.int64)
        return np.diff(self.te_offsets)


@dataclass
class SolveStats:
    """Per-instance statistics (solver.py:104-119); n_f_evals is batch-global."""

    n_steps: np.ndarray
    n_accepted: np.ndarray
    n_f_evals: np.ndarray
    final_dt: np.ndarray
    extra: dict = field(default_factory=dict)


class Solution:
    """Outputs at the requested times plus statistics and statuses
    (solver.py:122-138).  ``ys[i]`` holds only the points instance i
    reached; the ragged list is materialised lazily from the flat buffer."""

    def __init__(self, ys_flat, offsets, shared_len, n_emitted, stats, status, d):
        self.ys_flat = ys_flat
        self.offsets = offsets
        self.shared_len = shared_len
        self.n_emitted = n_emitted
        self.stats = stats
        self.status = status
        self.d = d
        self._ys = None

    @property
    def ys(self) -> list:
        if self._ys is None:
            n, d = self.status.shape[0], self.d
            if self.offsets is None:
                m = self.shared_len
                dense = self.ys_flat.reshape(n, m, d) if m else np.zeros((n, 0, d))
                self._ys = [dense[i, :self.n_emitted[i]] for i in range(n)]
            else:
                o = self.offsets
                flat = self.ys_flat.reshape(-1, d)
                self._ys = [flat[o[i]:o[i] + self.n_emitted[i]] for i in range(n)]
        return self._ys

    @property
    def ok(self) -> bool:
        return bool(np.all(self.status == SolveStatus.SUCCESS))


def _controller_struct(controller: PidCoefficients):
    c = _abi.Controller_()
    c.beta1, c.beta2, c.beta3 = controller.beta1, controller.beta2, controller.beta3
    c.safety, c.factor_min, c.factor_max = controller.safety, controller.factor_min, controller.factor_max
    c.update_history_on_reject = int(bool(controller.update_history_on_reject))
    return c


def _bind_method(a, method, dyn, d: int, keep: list, kernels: int = 1):
    """Set args.method (+ args.program for a custom tableau, traced dynamics
    or a registered elementwise functor wider than the compiled-in widths:
    a run-time specialisation of the same kernels, program.py)."""
    need = is_custom(method) or dyn.kind == "program"
    if not need and dyn.kind != "mlp":
        try:
            dyn.check_width(d)
        except NotImplementedError:
            need = True
    else:
        dyn.check_width(d)
    a.method = _abi.METHOD_CUSTOM if is_custom(method) else _abi.METHOD[method]
    if need:
        from .program import get_program
        prog = get_program(method, dyn, d, kernels)
        keep.append(prog)
        a.program = prog.handle
    return need


def _tol_arrays(tol: Tolerances, n: int):
    out = []
    for v in (tol.atol, tol.rtol):
        if np.ndim(v) == 0:
            out.append((None, float(v)))
        else:
            a = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
            if a.shape[0] != n:
                raise ValueError("per-instance tolerances need one entry per instance")
            out.append((a, 0.0))
    return out


def solve(problem: IvpBatch, f, tableau=None, tol: Tolerances | None = None,
          controller: PidCoefficients | None = None, max_steps: int = DEFAULT_MAX_STEPS,
          dt0=None, record_trace: bool = False, *, mode: str = "exact", order=None,
          cost_hint=None, pipeline_chunks="auto", with_refresh_map: bool = False,
          device_ys: bool = False, _joint: bool = False) -> Solution:
    """Integrate every instance independently with adaptive steps on the GPU
    (reference ``solve``, solver.py:352-369), host arrays in and out.
    ``device_ys=True``: the same solve, but ``Solution.ys_flat`` (and the
    ``ys`` rows) stay on the GPU as a torch tensor -- only the inputs go up
    and the statistics / statuses come back (for callers that consume the
    dense output on the device; torchode's semantics)."""
    if max_steps < 1:
        raise ValueError("max_steps must be at least 1")
    if device_ys:
        if _joint or record_trace or with_refresh_map:
            raise ValueError("device_ys: independent solve without trace / refresh map")
        return _solve_device_ys(problem, f, tableau, tol, controller, max_steps, dt0, mode,
                                order, cost_hint)
    lib = _abi.load()
    n, d = problem.batch_size, problem.n_features
    dyn = as_device_dynamics(f, n, d)
    method = method_of(tableau)
    tol = tol if tol is not None else Tolerances()
    if dyn.kind == "mlp" and (pad := mlp_pad(dyn)) is not None:
        return _solve_mlp_padded(problem, pad, tableau, tol, controller, max_steps, dt0,
                                 record_trace, mode=mode, order=order, cost_hint=cost_hint,
                                 pipeline_chunks=pipeline_chunks,
                                 with_refresh_map=with_refresh_map)
    controller = controller if controller is not None else integral_controller()
    keep = []
    a = _abi.SolveArgs()
    a.abi_version = _abi.ABI_VERSION
    _bind_method(a, method, dyn, d, keep, kernels=8 if _joint else 1)  # program JOINT / SOLVE
    a.mode = _abi.MODE[mode]
    a.n, a.d = n, d
    a.dyn = build_struct(dyn, n, keep)
    a.ctrl = _controller_struct(controller)
    y0 = np.ascontiguousarray(problem.y0)
    ts = np.ascontiguousarray(problem.t_start)
    tn = np.ascontiguousarray(problem.t_end)
    te = np.ascontiguousarray(problem.te_values)
    keep += [y0, ts, tn, te]
    a.y0, a.t_start, a.t_end = y0.ctypes.data, ts.ctypes.data, tn.ctypes.data
    a.t_eval = te.ctypes.data if te.size else None
    if problem.te_shared or te.size == 0:
        a.t_eval_len = te.size
        n_rows = n * te.size
        offs = None
    else:
        offs = np.ascontiguousarray(problem.te_offsets)
        keep.append(offs)
        a.t_eval_offsets = offs.ctypes.data
        n_rows = int(offs[-1])
    (av, a.atol), (rv, a.rtol) = _tol_arrays(tol, n)
    keep += [av, rv]
    a.atol_v = av.ctypes.data if av is not None else None
    a.rtol_v = rv.ctypes.data if rv is not None else None
    a.max_steps = int(max_steps)
    if dt0 is None:
        a.dt0_mode = _abi.DT0_HEURISTIC
    elif np.ndim(dt0) == 0:
        a.dt0_mode, a.dt0 = _abi.DT0_SCALAR, float(dt0)
    else:
        dv = np.ascontiguousarray(np.broadcast_to(np.asarray(dt0, dtype=np.float64), (n,)))
        keep.append(dv)
        a.dt0_mode, a.dt0_v = _abi.DT0_ARRAY, dv.ctypes.data
    if order is not None:
        order = np.ascontiguousarray(np.asarray(order, dtype=np.int64))
        keep.append(order)
        a.order = order.ctypes.data
    elif cost_hint is not None:  # LPT queue order built on the device
        ch = np.ascontiguousarray(np.broadcast_to(np.asarray(cost_hint, dtype=np.float64), (n,)))
        keep.append(ch)
        a.cost_hint = ch.ctypes.data
    if pipeline_chunks == "auto":
        # 3 chunks overlap uploads / downloads with the solve, but each chunk
        # ends with its own tail: with a heavy-tailed cost hint (one instance
        # costing more than a lane's share of a chunk) a single launch wins
        pipeline_chunks = 3 if n >= 65536 else 1
        if cost_hint is not None and pipeline_chunks > 1:
            c = np.asarray(cost_hint, dtype=np.float64).reshape(-1)
            # one strided gather, then max and mean on the contiguous copy
            smp = np.ascontiguousarray(c[::max(1, c.size // 4096)])
            if smp.max() > smp.mean() * n / (_LANES * pipeline_chunks):
                pipeline_chunks = 1
    a.pipeline_chunks = int(pipeline_chunks) if n >= 65536 else 1
    a.joint = 1 if _joint else 0
    ys = host_empty((max(n_rows, 1), d))
    n_emitted = host_empty(n, np.int64)
    n_steps = host_empty(n, np.int64)
    n_accepted = host_empty(n, np.int64)
    final_dt = host_empty(n)
    status = host_empty(n, np.int64)
    nfe = np.zeros(1, np.int64)
    a.ys = ys.ctypes.data if n_rows else None
    a.n_emitted, a.n_steps, a.n_accepted = n_emitted.ctypes.data, n_steps.ctypes.data, n_accepted.ctypes.data
    a.final_dt, a.status, a.n_f_evals = final_dt.ctypes.data, status.ctypes.data, nfe.ctypes.data
    if record_trace:
        cap = int(max_steps)
        tt, tdt, tacc = np.zeros((n, cap)), np.zeros((n, cap)), np.zeros((n, cap), np.uint8)
        a.trace_t, a.trace_dt, a.trace_accept, a.trace_cap = (tt.ctypes.data, tdt.ctypes.data,
                                                              tacc.ctypes.data, cap)
    if with_refresh_map:  # for combining n_f_evals across shards (distributed.py)
        max_it = np.zeros(1, np.int64)
        rmap = np.zeros(int(max_steps) + 2, np.uint8)
        a.max_iterations_out, a.refresh_map_out = max_it.ctypes.data, rmap.ctypes.data
    _abi.check(lib.bode_solve_host(_abi.C.byref(a)))
    extra = {}
    if with_refresh_map:
        extra["max_iterations"] = int(max_it[0])
        extra["refresh_map"] = rmap
    if record_trace and _joint:  # one trajectory, replicated (solver.py:423)
        extra["trace_t"] = [tt[0, :n_steps[0]].copy()] * n
        extra["trace_dt"] = [tdt[0, :n_steps[0]].copy()] * n
        extra["trace_accept"] = [tacc[0, :n_steps[0]].astype(bool)] * n
    elif record_trace:
        extra["trace_t"] = [tt[i, :n_steps[i]].copy() for i in range(n)]
        extra["trace_dt"] = [tdt[i, :n_steps[i]].copy() for i in range(n)]
        extra["trace_accept"] = [tacc[i, :n_steps[i]].astype(bool) for i in range(n)]
    stats = SolveStats(n_steps=n_steps, n_accepted=n_accepted,
                       n_f_evals=np.broadcast_to(nfe, (n,)), final_dt=final_dt,
                       extra=extra)
    if te.size == 0:
        offs = None
    return Solution(ys[:n_rows], offs, te.size if problem.te_shared else 0, n_emitted, stats,
                    status, d)


def _solve_device_ys(problem, f, tableau, tol, controller, max_steps, dt0, mode, order,
                     cost_hint) -> Solution:
    """solve(..., device_ys=True): host inputs uploaded, solve_device, the
    statistics downloaded, ys left on the device."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    T = lambda x: None if x is None else torch.as_tensor(np.asarray(x)).to(dev, non_blocking=True)  # noqa: E731
    n, d = problem.batch_size, problem.n_features
    tol = tol if tol is not None else Tolerances()
    tv = T(problem.te_values) if problem.te_values.size else None
    offs = None if problem.te_shared or tv is None else T(problem.te_offsets)
    tv2 = tv
    atol = tol.atol if np.ndim(tol.atol) == 0 else T(np.asarray(tol.atol, dtype=float))
    rtol = tol.rtol if np.ndim(tol.rtol) == 0 else T(np.asarray(tol.rtol, dtype=float))
    d0 = dt0 if dt0 is None or np.ndim(dt0) == 0 else T(np.asarray(dt0, dtype=float))
    out = solve_device(T(problem.y0), T(problem.t_start), T(problem.t_end), f, t_eval=tv2,
                       t_eval_offsets=offs, method=tableau if tableau is not None else "dopri5",
                       atol=atol, rtol=rtol, controller=controller, max_steps=max_steps, dt0=d0,
                       order=None if order is None else T(np.asarray(order, dtype=np.int64)),
                       cost_hint=None if cost_hint is None else T(np.asarray(cost_hint, dtype=float)),
                       mode=mode)
    h = {k: out[k].cpu().numpy() for k in ("n_emitted", "n_steps", "n_accepted", "final_dt",
                                           "status", "n_f_evals")}
    stats = SolveStats(n_steps=h["n_steps"], n_accepted=h["n_accepted"],
                       n_f_evals=np.broadcast_to(h["n_f_evals"], (n,)), final_dt=h["final_dt"],
                       extra={})
    shared = problem.te_values.size if problem.te_shared else 0
    return Solution(out["ys"].reshape(-1), None if problem.te_shared or tv is None
                    else problem.te_offsets, shared, h["n_emitted"], stats, h["status"], d)


def _pad_scale(D: int) -> float:
    """Tolerance factor making the RMS error norm over the zero-padded
    64-wide state equal the norm over the D real components."""
    return float(np.sqrt(D / MLP_TILE))


def _pad_tol(v, D: int, positive: bool = False):
    if positive and np.any(np.asarray(v.cpu() if hasattr(v, "cpu") else v) <= 0):
        raise ValueError("MLP dynamics narrower than 64 need atol > 0 (the zero-padded "
                         "components would divide 0 by 0 in the error norm)")
    return v * _pad_scale(D)


def _solve_mlp_padded(problem, pad, tableau, tol, controller, max_steps, dt0, record_trace, **kw):
    """solve() for an MLP narrower than the tensor-core tile: the same
    solve on the zero-padded 64-wide state with sqrt(D/64)-scaled
    tolerances (dynamics.mlp_pad), outputs sliced back to D."""
    import copy

    dyn64, D, _ = pad
    p64 = copy.copy(problem)
    p64.y0 = np.zeros((problem.batch_size, MLP_TILE))
    p64.y0[:, :D] = problem.y0
    tol64 = Tolerances(_pad_tol(tol.atol, D, positive=True), _pad_tol(tol.rtol, D))
    sol = solve(p64, dyn64, tableau, tol64, controller, max_steps, dt0, record_trace, **kw)
    ys = np.ascontiguousarray(sol.ys_flat.reshape(-1, MLP_TILE)[:, :D]).reshape(-1)
    return Solution(ys, sol.offsets, sol.shared_len, sol.n_emitted, sol.stats, sol.status, D)


def solve_joint(problem: IvpBatch, f, tableau=None, tol: Tolerances | None = None,
                controller: PidCoefficients | None = None, max_steps: int = DEFAULT_MAX_STEPS,
                dt0=None, record_trace: bool = False, *, mode: str = "exact") -> Solution:
    """Integrate the batch as one concatenated problem of size ``n * d``
    (reference ``solve_joint``, solver.py:372-427): one RMS error norm over
    all components, one shared step size and accept decision, statistics of
    the shared trajectory replicated per instance -- the naive-batching
    behaviour independent solving avoids.  Same validation as the reference;
    one single-CTA kernel on the GPU (csrc/bode_joint.cu)."""
    n = problem.batch_size
    if np.any(problem.t_start != problem.t_start[0]) or np.any(
            problem.t_end != problem.t_end[0]):
        raise ValueError("joint mode requires identical integration bounds")
    te0 = np.asarray(problem.t_eval[0], dtype=float)
    if not problem.te_shared:
        counts = problem.eval_counts()
        if np.any(counts != te0.size):
            raise ValueError("joint mode requires identical evaluation points")
        vals = problem.te_values.reshape(n, te0.size) if te0.size else None
        if vals is not None and np.any(vals != te0[None, :]):
            raise ValueError("joint mode requires identical evaluation points")
    if np.asarray(tol.atol if tol else 0.0).ndim > 0 or np.asarray(
            tol.rtol if tol else 0.0).ndim > 0:
        raise ValueError("joint mode supports scalar tolerances only")
    if dt0 is not None and np.ndim(dt0) > 0:  # the flat problem has one row
        dt0 = float(np.asarray(dt0, dtype=float).reshape(-1)[0])
    flat = IvpBatch(problem.y0, problem.t_start, problem.t_end, te0)
    return solve(flat, f, tableau, tol, controller, max_steps, dt0, record_trace, mode=mode,
                 _joint=True)


def solve_device(y0, t_start, t_end, f, *, t_eval=None, t_eval_offsets=None, method="dopri5",
                 atol=1e-6, rtol=1e-6, controller: PidCoefficients | None = None,
                 max_steps: int = DEFAULT_MAX_STEPS, dt0=None, order=None, cost_hint=None,
                 mode: str = "exact", record_trace: bool = False, stream=None,
                 threads_per_block: int = 0, blocks: int = 0,
                 prof_events=None, with_refresh_map: bool = False,
                 record_trajectory: bool = False, _launch: bool = True):
    """Device-resident solve on torch CUDA tensors; asynchronous (no host
    sync).  ``t_eval``: None, a 1-D tensor shared by all instances, a 2-D
    (n, m) tensor, or CSR values with ``t_eval_offsets`` (n+1).  ``atol`` /
    ``rtol`` / ``dt0``: Python floats or (n,) tensors.  Returns a dict of
    device tensors: ys, n_emitted, n_steps, n_accepted, final_dt, status,
    n_f_evals (+ trace_* when ``record_trace``).  ``record_trajectory``:
    also record every accepted step for :func:`adjoint_device` (a second,
    recording pass of the same deterministic solve, sized from the first
    pass's n_accepted -- one host sync).  ``_launch=False`` (internal,
    ``distributed.solve_multi``): build the arguments and outputs without
    launching; the returned dict's ``_args`` is then launched by the
    caller."""
    import torch

    lib = _abi.load()
    if not _launch and record_trajectory:
        raise ValueError("record_trajectory needs the launch (its sizing pass)")
    if max_steps < 1:
        raise ValueError("max_steps must be at least 1")
    method = method_of(method)
    controller = controller if controller is not None else integral_controller()
    dev = y0.device
    if dev.type != "cuda":
        raise ValueError("solve_device needs CUDA tensors")
    f64 = dict(dtype=torch.float64, device=dev)
    y0 = y0.to(**f64).contiguous()
    n, d = y0.shape
    dyn = as_device_dynamics(f, n, d)
    if dyn.kind == "mlp" and (pad := mlp_pad(dyn)) is not None:
        # the zero-padded 64-wide solve (dynamics.mlp_pad), outputs sliced to D
        dyn64, D, H = pad
        y64 = torch.zeros((n, MLP_TILE), **f64)
        y64[:, :D] = y0
        out = solve_device(y64, t_start, t_end, dyn64, t_eval=t_eval, t_eval_offsets=t_eval_offsets,
                           method=method, atol=_pad_tol(atol, D, positive=True), rtol=_pad_tol(rtol, D),
                           controller=controller, max_steps=max_steps, dt0=dt0, order=order,
                           cost_hint=cost_hint, mode=mode, record_trace=record_trace,
                           stream=stream, threads_per_block=threads_per_block, blocks=blocks,
                           prof_events=prof_events, with_refresh_map=with_refresh_map,
                           record_trajectory=record_trajectory, _launch=_launch)
        out["ys"] = out["ys"][:, :D].contiguous()
        out["_mlp_pad"] = (D, H)
        return out
    t_start = torch.as_tensor(t_start, **f64).expand(n).contiguous()
    t_end = torch.as_tensor(t_end, **f64).expand(n).contiguous()
    keep = [y0, t_start, t_end]

    def dptr(x):
        t = torch.as_tensor(x, device=dev).contiguous()
        keep.append(t)
        return t.data_ptr()

    a = _abi.SolveArgs()
    a.abi_version = _abi.ABI_VERSION
    _bind_method(a, method, dyn, d, keep)
    a.mode = _abi.MODE[mode]
    a.n, a.d = n, d
    a.dyn = build_struct(dyn, n, keep, device_arrays=dptr)
    a.ctrl = _controller_struct(controller)
    a.y0, a.t_start, a.t_end = y0.data_ptr(), t_start.data_ptr(), t_end.data_ptr()
    offsets = None
    if t_eval is None:
        n_rows, shared_len = 0, 0
    elif t_eval_offsets is not None:
        tv = t_eval.to(**f64).contiguous()
        offsets = t_eval_offsets.to(dtype=torch.int64, device=dev).contiguous()
        keep += [tv, offsets]
        a.t_eval, a.t_eval_offsets = tv.data_ptr(), offsets.data_ptr()
        n_rows, shared_len = tv.numel(), 0
    elif t_eval.dim() == 1:
        tv = t_eval.to(**f64).contiguous()
        keep.append(tv)
        a.t_eval, a.t_eval_len = tv.data_ptr(), tv.numel()
        n_rows, shared_len = n * tv.numel(), tv.numel()
    else:
        tv = t_eval.to(**f64).contiguous()
        m = tv.shape[1]
        offsets = torch.arange(n + 1, device=dev, dtype=torch.int64) * m
        keep += [tv, offsets]
        a.t_eval, a.t_eval_offsets = tv.data_ptr(), offsets.data_ptr()
        n_rows, shared_len = n * m, 0
    for name, v in (("atol", atol), ("rtol", rtol)):
        if isinstance(v, torch.Tensor) and v.dim() > 0:
            setattr(a, name + "_v", dptr(v.to(torch.float64)))
        else:
            setattr(a, name, float(v))
    a.max_steps = int(max_steps)
    if dt0 is None:
        a.dt0_mode = _abi.DT0_HEURISTIC
    elif isinstance(dt0, torch.Tensor) and dt0.dim() > 0:
        a.dt0_mode, a.dt0_v = _abi.DT0_ARRAY, dptr(dt0.to(torch.float64))
    else:
        a.dt0_mode, a.dt0 = _abi.DT0_SCALAR, float(dt0)
    if order is not None:
        a.order = dptr(order.to(torch.int64))
    elif cost_hint is not None:  # LPT queue order built on the device
        a.cost_hint = dptr(torch.as_tensor(cost_hint, dtype=torch.float64, device=dev).expand(n))
    out = dict(
        ys=torch.empty((max(n_rows, 1), d), **f64),
        n_emitted=torch.empty(n, dtype=torch.int64, device=dev),
        n_steps=torch.empty(n, dtype=torch.int64, device=dev),
        n_accepted=torch.empty(n, dtype=torch.int64, device=dev),
        final_dt=torch.empty(n, **f64),
        status=torch.empty(n, dtype=torch.int64, device=dev),
        n_f_evals=torch.empty(1, dtype=torch.int64, device=dev),
    )
    a.ys = out["ys"].data_ptr() if n_rows else None
    for k in ("n_emitted", "n_steps", "n_accepted", "final_dt", "status", "n_f_evals"):
        setattr(a, k, out[k].data_ptr())
    if record_trace:
        cap = int(max_steps)
        out["trace_t"] = torch.zeros((n, cap), **f64)
        out["trace_dt"] = torch.zeros((n, cap), **f64)
        out["trace_accept"] = torch.zeros((n, cap), dtype=torch.uint8, device=dev)
        a.trace_t, a.trace_dt = out["trace_t"].data_ptr(), out["trace_dt"].data_ptr()
        a.trace_accept, a.trace_cap = out["trace_accept"].data_ptr(), cap
    if with_refresh_map:  # for the cross-shard n_f_evals (distributed.global_f_evals_device)
        out["max_iterations"] = torch.zeros(1, dtype=torch.int64, device=dev)
        out["refresh_map"] = torch.zeros(int(max_steps) + 2, dtype=torch.uint8, device=dev)
        a.max_iterations_out = out["max_iterations"].data_ptr()
        a.refresh_map_out = out["refresh_map"].data_ptr()
    a.threads_per_block, a.blocks = int(threads_per_block), int(blocks)
    if prof_events is not None:  # (torch.cuda.Event, torch.cuda.Event) around the integrator
        a.prof_event_start, a.prof_event_stop = (prof_events[0].cuda_event,
                                                 prof_events[1].cuda_event)
    wsb = lib.bode_workspace_size(_abi.C.byref(a))
    if wsb == 0:
        _abi.check(_abi.EINVAL)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    keep.append(ws)
    a.workspace, a.workspace_bytes = ws.data_ptr(), wsb
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    a.stream = st.cuda_stream
    nlaunch = _abi.C.c_int64(0)
    keep.append(nlaunch)  # a.launch_count_out must stay valid while `a` is reused
    a.launch_count_out = _abi.C.addressof(nlaunch)
    if _launch:
        _abi.check(lib.bode_solve(_abi.C.byref(a)))
    if record_trajectory:
        # the sizing reads (cumsum, row count, divergence check) run on the
        # solve's own stream, so they see the sizing solve's n_accepted even
        # when the caller passed a non-current `stream`
        with torch.cuda.stream(st):
            toff = torch.zeros(n + 1, dtype=torch.int64, device=dev)
            torch.cumsum(out["n_accepted"], 0, out=toff[1:])
            rows = int(toff[-1])
            traj = torch.empty((max(rows, 1), _abi.traj_stride(d)), **f64)
            keep += [toff, traj]
            a.traj, a.traj_offsets = traj.data_ptr(), toff.data_ptr()
            tstages = None
            ns = _abi.mlp_stage_record(a)
            if ns:  # tensor-core backward: the fp32 stage inputs of every step
                tstages = torch.zeros((max(rows, 1), ns, 64), dtype=torch.float32, device=dev)
                keep.append(tstages)
                a.traj_stages = tstages.data_ptr()
            n_acc0 = out["n_accepted"].clone()
            _abi.check(lib.bode_solve(_abi.C.byref(a)))
            if not torch.equal(n_acc0, out["n_accepted"]):  # (the rows are bounded in-kernel)
                raise _abi.BodeLibraryError("the recording solve diverged from the sizing solve")
        out["traj"], out["traj_offsets"] = traj[:rows], toff
        out["traj_stages"] = tstages
        out["_args"], out["_keep"], out["_stream"] = a, keep, st
    # keep inputs alive until the stream has consumed them
    for t in keep:
        if isinstance(t, torch.Tensor):
            t.record_stream(st)
    out["ys"] = out["ys"][:n_rows]
    out.setdefault("_args", a)
    out.setdefault("_keep", keep)
    out["launches"] = int(nlaunch.value)
    out["offsets"] = offsets
    out["shared_len"] = shared_len
    return out


def adjoint_device(fwd: dict, grad_ys):
    """Reverse-mode gradients of a recorded device solve
    (``solve_device(..., record_trajectory=True)``): returns
    ``(grad_y0 (n, d), grad_params (n, 8))`` for ``grad_ys`` = dL/dys in
    the forward ys layout.  Column k of grad_params is dL/dp_k per instance
    for parameter slot k of the dynamics (``dynamics.SLOTS`` order); for a
    parameter shared by the batch its gradient is the column sum.  For MLP
    dynamics grad_params is instead a dict of the batch-summed fp32 weight
    gradients {W1, b1, W2, b2}.  Step
    sizes and accept decisions are constants (no gradient through the
    step-size controller); see include/bode.h ``bode_solve_adjoint``."""
    import torch

    lib = _abi.load()
    if "_args" not in fwd:
        raise ValueError("the forward solve was not recorded (record_trajectory=True)")
    if "_mlp_pad" in fwd:  # the forward ran zero-padded to 64 (dynamics.mlp_pad)
        D, H = fwd["_mlp_pad"]
        g64 = torch.zeros((fwd["ys"].shape[0], MLP_TILE), dtype=torch.float64,
                          device=fwd["n_emitted"].device)
        g64[:, :D] = grad_ys.reshape(-1, D)
        inner = {k: v for k, v in fwd.items() if k not in ("_mlp_pad", "ys")}
        inner["ys"] = g64  # (only its shape is used)
        gy0, gw = adjoint_device(inner, g64)
        return gy0[:, :D].contiguous(), {"W1": gw["W1"][:H, :D].contiguous(),
                                         "b1": gw["b1"][:H].contiguous(),
                                         "W2": gw["W2"][:D, :H].contiguous(),
                                         "b2": gw["b2"][:D].contiguous()}
    a = fwd["_args"]
    n, d = int(a.n), int(a.d)
    dev = fwd["n_emitted"].device
    g = _abi.AdjointArgs()
    keep = []
    g.traj, g.traj_offsets = fwd["traj"].data_ptr(), fwd["traj_offsets"].data_ptr()
    if fwd.get("traj_stages") is not None:
        g.traj_stages = fwd["traj_stages"].data_ptr()
    g.n_emitted = fwd["n_emitted"].data_ptr()
    if fwd["ys"].numel():
        gy = grad_ys.to(dtype=torch.float64, device=dev).reshape(fwd["ys"].shape).contiguous()
        keep.append(gy)
        g.grad_ys = gy.data_ptr()
    grad_y0 = torch.empty((n, d), dtype=torch.float64, device=dev)
    g.grad_y0 = grad_y0.data_ptr()
    if a.dyn.kind != _abi.DYN["mlp"]:  # per-instance parameter-slot gradients
        grad_params = torch.empty((n, 8), dtype=torch.float64, device=dev)
        g.grad_params = grad_params.data_ptr()
    else:  # batch-summed weight gradients (fp32)
        H = int(a.dyn.hidden)
        f32 = dict(dtype=torch.float32, device=dev)
        grad_params = dict(W1=torch.empty((H, d), **f32), b1=torch.empty(H, **f32),
                           W2=torch.empty((d, H), **f32), b2=torch.empty(d, **f32))
        g.grad_W1, g.grad_b1 = grad_params["W1"].data_ptr(), grad_params["b1"].data_ptr()
        g.grad_W2, g.grad_b2 = grad_params["W2"].data_ptr(), grad_params["b2"].data_ptr()
    wsb = lib.bode_adjoint_workspace_size(_abi.C.byref(a))
    if wsb == 0:
        _abi.check(_abi.EINVAL)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    keep.append(ws)
    g.workspace, g.workspace_bytes = ws.data_ptr(), wsb
    nlaunch = _abi.C.c_int64(0)
    g.launch_count_out = _abi.C.addressof(nlaunch)
    # the adjoint runs on the caller's current stream (where grad_y0 and the
    # weight gradients were allocated), after the forward's stream
    st = torch.cuda.current_stream(dev)
    st.wait_stream(fwd["_stream"])
    a.stream = st.cuda_stream
    _abi.check(lib.bode_solve_adjoint(_abi.C.byref(a), _abi.C.byref(g)))
    for t in keep:
        t.record_stream(st)
    fwd["adjoint_launches"] = int(nlaunch.value)
    return grad_y0, grad_params
