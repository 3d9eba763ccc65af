"""The reference's solve-path building blocks as batched GPU ops.

Same names, signatures and error behaviour as the reference functions
(``pkg/src/batchode/``): ``rk_step`` / ``interpolate`` / ``StepResult``
(stepper.py:23-37,142-165), ``error_norm`` (controller.py:120-142),
``initial_step`` (controller.py:145-197), ``adapt_step`` +
``ControllerState`` (controller.py:102-117,200-238).  NumPy in, NumPy out;
each call runs one exact-arithmetic kernel (csrc/bode_units.cu) through the
C ABI.  The persistent solver fuses all of these; the standalone ops exist
so the reference's unit tests can be re-expressed against the device code.
"""

from dataclasses import dataclass

import numpy as np

from . import _abi
from .controller import NORM_FLOOR, ControllerState, PidCoefficients, Tolerances  # noqa: F401
from .dynamics import as_device_dynamics, build_struct
from .tableau import ButcherTableau, method_of

__all__ = ["StepResult", "ControllerState", "rk_step", "interpolate", "error_norm",
           "initial_step", "adapt_step"]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _abi.BodeLibraryError("the unit ops need a CUDA device (no CPU fallback)")
    return torch


def _dev(x, dtype=None):
    torch = _torch()
    a = np.array(x, dtype=dtype or np.float64, order="C", copy=True)
    return torch.from_numpy(a).to("cuda")


def _stream():
    return _torch().cuda.current_stream().cuda_stream


@dataclass
class StepResult:
    """One trial step for every instance (stepper.py:23-37)."""

    y_next: np.ndarray
    error_estimate: np.ndarray
    stage_derivs: np.ndarray
    f_next: np.ndarray | None
    n_evals: int = 0


def rk_step(f, tableau: ButcherTableau, t, dt, y, f0) -> StepResult:
    """One embedded RK trial step on the full batch (stepper.py:54-110)."""
    torch = _torch()
    lib = _abi.load()
    dyn = as_device_dynamics(f)
    method = method_of(tableau)
    y = np.atleast_2d(np.asarray(y, dtype=float))
    n, d = y.shape
    dyn.check_width(d)
    keep = []
    dptr = lambda a: (keep.append(_dev(a)), keep[-1].data_ptr())[1]  # noqa: E731
    ds = build_struct(dyn, n, keep, device_arrays=dptr)
    S = 2 if method == "heun" else 7
    tt, dtt, yy = _dev(np.broadcast_to(t, (n,))), _dev(np.broadcast_to(dt, (n,))), _dev(y)
    ff = _dev(f0 if f0 is not None else np.zeros((n, d)))
    yn = torch.empty((n, d), dtype=torch.float64, device="cuda")
    err = torch.empty_like(yn)
    k = torch.empty((S, n, d), dtype=torch.float64, device="cuda")
    _abi.check(lib.bode_rk_step(_abi.METHOD[method], _abi.MODE["exact"], _abi.C.addressof(ds),
                                n, d, tt.data_ptr(), dtt.data_ptr(), yy.data_ptr(),
                                ff.data_ptr(), yn.data_ptr(), err.data_ptr(), k.data_ptr(),
                                _stream()))
    kk = k.cpu().numpy()
    fsal = method != "heun"
    return StepResult(y_next=yn.cpu().numpy(), error_estimate=err.cpu().numpy(),
                      stage_derivs=kk, f_next=kk[S - 1] if fsal else None,
                      n_evals=S - 1 if fsal else S)


def interpolate(step: StepResult, tableau: ButcherTableau, y0, dt, theta) -> np.ndarray:
    """Dense output y(t + theta*dt) (stepper.py:112-139); theta outside
    [0, 1] is an argument error, as in the reference (:126-127)."""
    torch = _torch()
    lib = _abi.load()
    theta = np.asarray(theta, dtype=float)
    if np.any((theta < 0.0) | (theta > 1.0)):
        raise ValueError("theta must lie in [0, 1]")
    method = method_of(tableau)
    y0 = np.atleast_2d(np.asarray(y0, dtype=float))
    n, d = y0.shape
    out = torch.empty((n, d), dtype=torch.float64, device="cuda")
    k, yy, dtt, th = (_dev(step.stage_derivs), _dev(y0), _dev(np.broadcast_to(dt, (n,))),
                      _dev(np.broadcast_to(theta, (n,))))
    _abi.check(lib.bode_interpolate(_abi.METHOD[method], _abi.MODE["exact"], n, d,
                                    k.data_ptr(), yy.data_ptr(), dtt.data_ptr(), th.data_ptr(),
                                    out.data_ptr(), _stream()))
    return out.cpu().numpy()


def _tol_dev(v, n):
    if np.ndim(v) == 0:
        return None, float(v)
    return _dev(np.asarray(v, dtype=float).reshape(n)), 0.0


def error_norm(error_estimate, y0, y1, tol: Tolerances) -> np.ndarray:
    """Mixed-tolerance RMS norm per instance (controller.py:120-142)."""
    torch = _torch()
    lib = _abi.load()
    e = np.atleast_2d(np.asarray(error_estimate, dtype=float))
    n, d = e.shape
    av, a = _tol_dev(tol.atol, n)
    rv, r = _tol_dev(tol.rtol, n)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    ee, a0, a1 = _dev(e), _dev(y0), _dev(y1)
    _abi.check(lib.bode_error_norm(n, d, ee.data_ptr(), a0.data_ptr(), a1.data_ptr(),
                                   av.data_ptr() if av is not None else None,
                                   rv.data_ptr() if rv is not None else None, a, r,
                                   out.data_ptr(), _stream()))
    return out.cpu().numpy()


def initial_step(f, t0, y0, order: int, tol: Tolerances, direction=1.0):
    """Two-evaluation starting step (controller.py:145-197) -> (dt, f0)."""
    torch = _torch()
    lib = _abi.load()
    y0 = np.atleast_2d(np.asarray(y0, dtype=float))
    n, d = y0.shape
    dyn = as_device_dynamics(f, n, d)
    prog = None
    if dyn.kind == "program":
        from .program import UNITS, get_program
        prog = get_program("dopri5", dyn, d, UNITS)
    else:
        dyn.check_width(d)
    keep = []
    dptr = lambda a: (keep.append(_dev(a)), keep[-1].data_ptr())[1]  # noqa: E731
    ds = build_struct(dyn, n, keep, device_arrays=dptr)
    av, a = _tol_dev(tol.atol, n)
    rv, r = _tol_dev(tol.rtol, n)
    tt, yy = _dev(np.broadcast_to(t0, (n,))), _dev(y0)
    dr = _dev(np.broadcast_to(np.asarray(direction, dtype=float), (n,)))
    dt = torch.empty(n, dtype=torch.float64, device="cuda")
    f0 = torch.empty((n, d), dtype=torch.float64, device="cuda")
    args = (_abi.C.addressof(ds), n, d, tt.data_ptr(), yy.data_ptr(), int(order),
            av.data_ptr() if av is not None else None, rv.data_ptr() if rv is not None else None,
            a, r, dr.data_ptr(), dt.data_ptr(), f0.data_ptr(), _stream())
    if prog is not None:  # traced dynamics: the program's initial_step kernel
        _abi.check(lib.bode_program_initial_step(prog.handle, *args))
    else:
        _abi.check(lib.bode_initial_step(*args))
    return dt.cpu().numpy(), f0.cpu().numpy()


def adapt_step(state: ControllerState, norm, error_order: int, coeffs: PidCoefficients):
    """Accept decision and next step size; updates ``state`` in place
    (controller.py:200-238).  Returns (accept, dt_next)."""
    torch = _torch()
    lib = _abi.load()
    norm = np.asarray(norm, dtype=float)
    n = norm.shape[0]
    c = _abi.Controller_()
    c.beta1, c.beta2, c.beta3 = coeffs.beta1, coeffs.beta2, coeffs.beta3
    c.safety, c.factor_min, c.factor_max = coeffs.safety, coeffs.factor_min, coeffs.factor_max
    c.update_history_on_reject = int(bool(coeffs.update_history_on_reject))
    nn, p1, p2, dt = _dev(norm), _dev(state.norm_prev), _dev(state.norm_prev2), _dev(state.dt)
    acc = torch.empty(n, dtype=torch.uint8, device="cuda")
    dtn = torch.empty(n, dtype=torch.float64, device="cuda")
    _abi.check(lib.bode_adapt_step(n, nn.data_ptr(), int(error_order), _abi.C.addressof(c),
                                   p1.data_ptr(), p2.data_ptr(), dt.data_ptr(), acc.data_ptr(),
                                   dtn.data_ptr(), _stream()))
    state.norm_prev = p1.cpu().numpy()
    state.norm_prev2 = p2.cpu().numpy()
    state.dt = dt.cpu().numpy()
    return acc.cpu().numpy().astype(bool), dtn.cpu().numpy()
