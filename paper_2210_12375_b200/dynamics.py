"""Registered device dynamics (the plugin surface of the solve path).

The reference takes any NumPy callable ``f(t, y) -> (n, d)``
(``pkg/src/batchode/stepper.py:19-20``).  A persistent GPU integrator has
to evaluate ``f`` inside the kernel, so dynamics here are descriptors of
compiled-in device functors (``csrc/bode_device.cuh``) plus their
parameters; each parameter is a scalar (shared by the batch) or an (n,)
array (one value per instance, like ``VdpParams.mu``).  Arbitrary Python
callables are rejected with NotImplementedError -- there is no CPU
fallback.

Reference anchors: ``VdpParams`` / ``vdp_dynamics`` (problems.py:29-50),
``AnalyticProblem`` / ``analytic_problems`` (problems.py:146-189).  The
other functors cover the dynamics the reference's own tests pass as
lambdas (tests/test_solver.py, test_stepper.py, test_acceptance.py) and
the Lorenz / MLP systems of BASELINE.json.
"""

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _abi

__all__ = ["DeviceDynamics", "VdpParams", "vdp_dynamics", "lorenz_dynamics",
           "zero_dynamics", "constant_dynamics", "linear_dynamics",
           "forced_linear_dynamics", "relaxation_dynamics", "square_dynamics",
           "logistic_dynamics", "sin_plus_t_dynamics", "harmonic_dynamics",
           "damped_dynamics", "mlp_dynamics", "AnalyticProblem", "analytic_problems",
           "as_device_dynamics", "ProgramDynamics"]

# parameter slot order per functor (must match include/bode.h)
SLOTS = {
    "vdp": ("mu",), "lorenz": ("sigma", "rho", "beta"), "zero": (), "const": ("c",),
    "linear": ("lam",), "linear_cos": ("lam", "amp", "omega"),
    "linear_sin": ("lam", "amp", "omega"), "relax_cos": ("lam", "omega"),
    "square": ("thr",), "logistic": (), "sin_plus_t": (), "harmonic": (), "damped": (),
    "mlp": (),
}
FIXED_WIDTH = {"vdp": 2, "lorenz": 3, "harmonic": 2, "damped": 2}
MAX_ELEMENTWISE_WIDTH = 4


@dataclass(frozen=True, eq=False)
class DeviceDynamics:
    """A compiled-in device functor plus its parameters."""

    kind: str
    params: dict = field(default_factory=dict)
    mlp: tuple | None = None  # (W1 (H,D), b1 (H,), W2 (D,H), b2 (D,)) float32

    def __post_init__(self):
        if self.kind not in SLOTS:
            raise ValueError(f"unknown dynamics {self.kind!r}")
        missing = [s for s in SLOTS[self.kind] if s not in self.params]
        if missing:
            raise ValueError(f"{self.kind} dynamics missing parameters {missing}")

    def check_width(self, d: int) -> None:
        want = FIXED_WIDTH.get(self.kind)
        if want is not None and d != want:
            raise ValueError(f"{self.kind} dynamics need d={want}, got d={d}")
        if self.kind == "mlp":
            W1 = self.mlp[0]
            if W1.shape[1] != d:
                raise ValueError(f"MLP input width {W1.shape[1]} != state width {d}")
        elif want is None and d > MAX_ELEMENTWISE_WIDTH:
            raise NotImplementedError(
                f"{self.kind} dynamics are compiled for d <= {MAX_ELEMENTWISE_WIDTH}")

    def pack(self, n: int):
        """-> (shared[8], inst_mask, per-instance columns).  Columns are NumPy
        arrays, or torch tensors when the parameter was given as one (kept on
        its device for the device-resident path)."""
        shared = [0.0] * 8
        cols, mask = [], 0
        for k, name in enumerate(SLOTS[self.kind]):
            v = self.params[name]
            if _is_tensor(v):
                if v.dim() == 0:
                    shared[k] = float(v)
                    continue
                v = v.reshape(-1)
            elif np.ndim(v) == 0:
                shared[k] = float(v)
                continue
            else:
                v = np.asarray(v, dtype=np.float64).reshape(-1)
            if v.shape[0] != n:
                raise ValueError(f"parameter {name!r} must be scalar or have one entry "
                                 f"per instance ({n}), got {v.shape[0]}")
            cols.append(v)
            mask |= 1 << k
        return shared, mask, cols

    def subset(self, idx) -> "DeviceDynamics":
        """The same functor restricted to instances ``idx`` (per-instance
        parameters are sliced, shared ones kept) -- a shard of the batch."""
        params = {k: (v if np.ndim(v) == 0 else v[idx]) for k, v in self.params.items()}
        return DeviceDynamics(self.kind, params, self.mlp)

    def __call__(self, t, y):
        """f(t, y) on the batch, like the reference's dynamics callables
        (problems.py:41-50): the device functor evaluated by one kernel
        (``bode_eval_dynamics``), NumPy in / out."""
        import torch
        if self.kind == "mlp":
            raise TypeError("MLP dynamics are evaluated inside the fused tcgen05 solver only")
        if not torch.cuda.is_available():
            raise _abi.BodeLibraryError("evaluating a device functor needs a CUDA device "
                                        "(no CPU fallback)")
        y = np.atleast_2d(np.asarray(y, dtype=np.float64))
        n, d = y.shape
        self.check_width(d)
        tt = np.broadcast_to(np.asarray(0.0 if t is None else t, dtype=np.float64), (n,))
        keep = []
        dev = lambda a: (keep.append(torch.as_tensor(np.ascontiguousarray(a)).to("cuda")),  # noqa: E731
                         keep[-1].data_ptr())[1]
        ds = build_struct(self, n, keep, device_arrays=dev)
        out = torch.empty((n, d), dtype=torch.float64, device="cuda")
        lib = _abi.load()
        _abi.check(lib.bode_eval_dynamics(_abi.C.addressof(ds), n, d, dev(tt), dev(y),
                                          out.data_ptr(), torch.cuda.current_stream().cuda_stream))
        return out.cpu().numpy()


def _is_tensor(v) -> bool:
    return type(v).__module__.startswith("torch") and hasattr(v, "dim")


class ProgramDynamics:
    """A NumPy dynamics callable traced into a device functor (trace.py) and
    compiled into a run-time program with the solver templates
    (program.py): the reference's plugin surface (stepper.py:19-20) for any
    callable the tracer can follow.  ``params`` holds the (n, P) per-instance
    values the callable closes over (None when there are none)."""

    kind = "program"

    def __init__(self, traced, params, d, source_fn=None):
        self.traced, self.params, self.d = traced, params, d
        self.n_params = 0 if params is None else int(params.shape[1])
        self.source_fn = source_fn

    def check_width(self, d: int) -> None:
        if d != self.d:
            raise ValueError(f"dynamics traced for d={self.d}, got d={d}")

    def subset(self, idx) -> "ProgramDynamics":
        p = None if self.params is None else self.params[idx]
        return ProgramDynamics(self.traced, p, self.d, self.source_fn)

    def __call__(self, t, y):
        raise TypeError("traced dynamics are evaluated inside the B200 solver")


def as_device_dynamics(f, n: int | None = None, d: int | None = None):
    """Registered functors pass through; a NumPy callable f(t, y) is traced
    for a batch of n instances of width d (trace.py) -- raising
    NotImplementedError when it cannot run on the device (no CPU fallback)."""
    if isinstance(f, (DeviceDynamics, ProgramDynamics)):
        return f
    if callable(f) and n is not None and d is not None:
        from .trace import trace_dynamics
        tf = trace_dynamics(f, int(n), int(d))
        return ProgramDynamics(tf, tf.params, int(d), f)
    raise NotImplementedError(
        "this Python callable cannot run inside the sm_100a solver; pass a registered device "
        "functor from paper_2210_12375_b200.dynamics or a traceable NumPy callable "
        "(no CPU fallback)")


@dataclass(frozen=True)
class VdpParams:
    """Van der Pol damping strength, scalar or per instance (problems.py:29-38)."""

    mu: float | np.ndarray = 2.0

    def __post_init__(self):
        mu = self.mu
        if _is_tensor(mu):
            bad = bool((~mu.isfinite()).any() or (mu < 0).any())
        else:
            mu = np.asarray(mu)
            bad = bool(np.any(~np.isfinite(mu)) or np.any(mu < 0))
        if bad:
            raise ValueError("mu must be finite and nonnegative")


def vdp_dynamics(params: VdpParams) -> DeviceDynamics:
    """(x, v) -> (v, mu*(1-x*x)*v - x)   (problems.py:41-50)."""
    return DeviceDynamics("vdp", {"mu": params.mu})


def lorenz_dynamics(sigma=10.0, rho=28.0, beta=8.0 / 3.0) -> DeviceDynamics:
    """(sigma*(y-x), x*(rho-z)-y, x*y-beta*z)."""
    return DeviceDynamics("lorenz", {"sigma": sigma, "rho": rho, "beta": beta})


def zero_dynamics() -> DeviceDynamics:
    return DeviceDynamics("zero")


def constant_dynamics(c=1.0) -> DeviceDynamics:
    return DeviceDynamics("const", {"c": c})


def linear_dynamics(lam=1.0) -> DeviceDynamics:
    """lam * y (lam scalar or per instance)."""
    return DeviceDynamics("linear", {"lam": lam})


def forced_linear_dynamics(lam, amp=1.0, omega=1.0, forcing="cos") -> DeviceDynamics:
    """lam*y + amp*cos(omega*t)  (or sin)."""
    if forcing not in ("cos", "sin"):
        raise ValueError("forcing must be 'cos' or 'sin'")
    return DeviceDynamics("linear_" + forcing, {"lam": lam, "amp": amp, "omega": omega})


def relaxation_dynamics(lam, omega=1.0) -> DeviceDynamics:
    """lam*(y - cos(omega*t))."""
    return DeviceDynamics("relax_cos", {"lam": lam, "omega": omega})


def square_dynamics(threshold=np.inf) -> DeviceDynamics:
    """y*y, and +inf where y > threshold."""
    return DeviceDynamics("square", {"thr": threshold})


def logistic_dynamics() -> DeviceDynamics:
    return DeviceDynamics("logistic")


def sin_plus_t_dynamics() -> DeviceDynamics:
    return DeviceDynamics("sin_plus_t")


def harmonic_dynamics() -> DeviceDynamics:
    return DeviceDynamics("harmonic")


def damped_dynamics() -> DeviceDynamics:
    """(v, -x - 0.1*v*|v|)."""
    return DeviceDynamics("damped")


MLP_TILE = 64   # state width of the tensor-core tile (csrc/bode_tc.cuh kD)
MLP_HMAX = 256  # hidden width the fused kernel keeps in TMEM


def mlp_pad(dyn: DeviceDynamics):
    """The MLP zero-padded to the tensor-core tile: D -> 64, H -> a multiple
    of 32.  Returns (padded dynamics, D, H), or None when it already fits.
    Padded hidden units have zero weights and bias (tanh(0) = 0 feeds zero
    columns of W2), padded outputs have zero rows of W2 and zero bias, so
    f of a zero-padded state is the zero-padded f exactly and padded state
    components stay exactly 0.  solve / solve_device scale the tolerances by
    sqrt(D/64) so the 64-wide RMS error norm equals the D-wide one."""
    W1, b1, W2, b2 = dyn.mlp
    H, D = W1.shape
    if D > MLP_TILE or H > MLP_HMAX:
        raise NotImplementedError(f"MLP dynamics run on the 64-wide tensor-core tile: need "
                                  f"D <= {MLP_TILE} and hidden <= {MLP_HMAX}, got D={D}, H={H}")
    Hp = (H + 31) // 32 * 32
    if D == MLP_TILE and Hp == H:
        return None
    if _is_tensor(W1):
        import torch

        def z(*shape):
            return torch.zeros(shape, dtype=torch.float32, device=W1.device)
    else:
        def z(*shape):
            return np.zeros(shape, dtype=np.float32)
    W1p, b1p, W2p, b2p = z(Hp, MLP_TILE), z(Hp), z(MLP_TILE, Hp), z(MLP_TILE)
    W1p[:H, :D] = W1
    b1p[:H] = b1
    W2p[:D, :H] = W2
    b2p[:D] = b2
    return DeviceDynamics("mlp", {}, mlp=(W1p, b1p, W2p, b2p)), D, H


def mlp_dynamics(W1, b1, W2, b2) -> DeviceDynamics:
    """Neural-ODE dynamics W2 tanh(W1 y + b1) + b2 evaluated in fp32 on the
    tensor cores; the state stays fp64.  Weights as
    NumPy arrays, or CUDA tensors (for the device path; tensors that
    require grad receive gradients through torchode.AutoDiffAdjoint)."""
    if any(_is_tensor(x) for x in (W1, b1, W2, b2)):  # device tensors (may require grad)
        W1, b1, W2, b2 = (x.float().contiguous() for x in (W1, b1, W2, b2))
    else:
        W1, b1, W2, b2 = (np.ascontiguousarray(np.asarray(x, dtype=np.float32))
                          for x in (W1, b1, W2, b2))
    H, D = W1.shape
    if b1.shape != (H,) or W2.shape != (D, H) or b2.shape != (D,):
        raise ValueError("MLP weights must be W1 (H,D), b1 (H,), W2 (D,H), b2 (D,)")
    return DeviceDynamics("mlp", {}, mlp=(W1, b1, W2, b2))


@dataclass(frozen=True)
class AnalyticProblem:
    """Dynamics with a closed-form solution (problems.py:146-157)."""

    name: str
    n_features: int
    dynamics: DeviceDynamics
    exact: Callable[[np.ndarray, np.ndarray], np.ndarray]


def analytic_problems(lam: float = 1.0) -> list[AnalyticProblem]:
    """Exponential, harmonic oscillator and logistic growth (problems.py:160-189)."""

    def exp_exact(t, y0):
        return y0 * np.exp(lam * t)[:, None]

    def harmonic_exact(t, y0):
        c, s = np.cos(t), np.sin(t)
        return np.stack([y0[:, 0] * c + y0[:, 1] * s, -y0[:, 0] * s + y0[:, 1] * c], axis=1)

    def logistic_exact(t, y0):
        e = np.exp(t)[:, None]
        return y0 * e / (1.0 + y0 * (e - 1.0))

    return [
        AnalyticProblem("exponential", 1, linear_dynamics(lam), exp_exact),
        AnalyticProblem("harmonic", 2, harmonic_dynamics(), harmonic_exact),
        AnalyticProblem("logistic", 1, logistic_dynamics(), logistic_exact),
    ]


def build_struct(dyn: DeviceDynamics, n: int, keep: list, device_arrays=None):
    """Fill a ``bode_dynamics`` struct.  ``device_arrays`` maps host arrays to
    device pointers (device path); without it host pointers are used."""
    s = _abi.Dynamics_()
    s.kind = _abi.DYN[dyn.kind]
    ptr = device_arrays if device_arrays is not None else (lambda a: a.ctypes.data)
    if dyn.kind == "program":
        if dyn.params is not None:
            if dyn.params.shape[0] != n:
                raise ValueError(f"traced per-instance parameters have {dyn.params.shape[0]} "
                                 f"rows, the batch has {n}")
            inst = np.ascontiguousarray(dyn.params, dtype=np.float64)
            keep.append(inst)
            s.inst_params = ptr(inst)
        return s
    shared, mask, cols = dyn.pack(n)
    s.shared_params = (_abi.C.c_double * 8)(*shared)
    s.inst_mask = mask
    if cols:
        if device_arrays is not None and any(_is_tensor(c) for c in cols):
            import torch
            inst = torch.stack([torch.as_tensor(c, dtype=torch.float64) if not _is_tensor(c)
                                else c.to(torch.float64) for c in cols], dim=1)
        else:
            if any(_is_tensor(c) for c in cols):
                raise ValueError("device tensors given to the host solve path")
            if len(cols) == 1:  # one per-instance slot: pass the caller's array, no copy
                inst = np.ascontiguousarray(np.asarray(cols[0], dtype=np.float64).reshape(n, 1))
            else:
                inst = np.ascontiguousarray(np.stack(cols, axis=1))
        keep.append(inst)
        s.inst_params = ptr(inst)
    if dyn.kind == "mlp":
        W1, b1, W2, b2 = dyn.mlp
        keep.extend(dyn.mlp)
        s.W1, s.b1, s.W2, s.b2 = ptr(W1), ptr(b1), ptr(W2), ptr(b2)
        s.hidden = W1.shape[0]
    return s
