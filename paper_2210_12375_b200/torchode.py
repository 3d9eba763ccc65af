"""torchode-style API (arXiv 2210.12375) over the B200 solver.

The names BASELINE.json's north_star asks for -- ``ODETerm``,
``InitialValueProblem``, ``Dopri5`` / ``Tsit5`` / ``Heun``,
``IntegralController`` / ``PIDController``, ``AutoDiffAdjoint.solve`` and a
``Solution`` with ``ys``, ``status`` and per-instance ``stats`` -- mapped
onto the reference's semantics (SURVEY.md §8(b) mapping table):

  ODETerm(f)                 <- Dynamics callable         stepper.py:19-20
  InitialValueProblem        <- IvpBatch                  solver.py:53-101
  Dopri5 / Tsit5 / Heun      <- dopri5() / tsit5() / Heun-Euler pair
  IntegralController         <- integral_controller() + Tolerances
  PIDController              <- pid_controller / PidCoefficients
  AutoDiffAdjoint.solve      <- solve() / BatchSolver.run  solver.py:352,324

Everything is torch CUDA tensors and stays on the device (no host sync in
``solve``).  ``f`` must be a registered device functor
(:mod:`paper_2210_12375_b200.dynamics`); gradients through the solve are not
part of the reference and are not provided.
"""

from dataclasses import dataclass

from . import _abi  # noqa: F401  (fails loudly without the CUDA library)
from .controller import PID_PRESETS, PidCoefficients
from .dynamics import DeviceDynamics, as_device_dynamics
from .solver import DEFAULT_MAX_STEPS, SolveStatus, solve_device

__all__ = ["ODETerm", "InitialValueProblem", "Dopri5", "Tsit5", "Heun", "IntegralController",
           "PIDController", "AutoDiffAdjoint", "Solution", "Status"]

Status = SolveStatus


class ODETerm:
    """Right-hand side f(t, y).  Only registered device functors run on the
    B200 kernels; a plain Python callable raises NotImplementedError."""

    def __init__(self, f, with_args: bool = False):
        if with_args:
            raise NotImplementedError("extra dynamics arguments go into the functor's parameters")
        self.f: DeviceDynamics = as_device_dynamics(f)


@dataclass
class InitialValueProblem:
    """y0 (batch, features); t_start / t_end (batch,) or scalars; t_eval
    (batch, m) or (m,).  As in torchode, t_start / t_end default to the
    first / last evaluation time."""

    y0: "object"
    t_start: "object" = None
    t_end: "object" = None
    t_eval: "object" = None

    def __post_init__(self):
        import torch

        if self.y0.dim() != 2:
            raise ValueError("y0 must be (batch, features)")
        n = self.y0.shape[0]
        dev = self.y0.device
        if self.t_eval is not None:
            te = self.t_eval.to(device=dev, dtype=torch.float64)
            if self.t_start is None:
                self.t_start = te[..., 0] if te.dim() == 2 else te[0].expand(n)
            if self.t_end is None:
                self.t_end = te[..., -1] if te.dim() == 2 else te[-1].expand(n)
            self.t_eval = te
        if self.t_start is None or self.t_end is None:
            raise ValueError("need t_start and t_end (or t_eval)")
        self.t_start = torch.as_tensor(self.t_start, dtype=torch.float64, device=dev).expand(n)
        self.t_end = torch.as_tensor(self.t_end, dtype=torch.float64, device=dev).expand(n)
        if bool((self.t_start == self.t_end).any()):
            raise ValueError("t_end must differ from t_start for every instance")
        if self.t_eval is not None:
            te = self.t_eval if self.t_eval.dim() == 2 else self.t_eval.expand(n, -1)
            direction = torch.sign(self.t_end - self.t_start)[:, None]
            pos = (te - self.t_start[:, None]) * direction
            if te.shape[1] > 1 and bool((pos.diff(dim=1) < 0).any()):
                raise ValueError("t_eval is not sorted in integration direction")
            span = (self.t_end - self.t_start).abs()
            if te.shape[1] and bool(((pos[:, 0] < 0) | (pos[:, -1] > span)).any()):
                raise ValueError("t_eval leaves the integration interval")

    @property
    def batch_size(self) -> int:
        return self.y0.shape[0]


class _StepMethod:
    method = ""

    def __init__(self, term: ODETerm | None = None):
        self.term = term


class Dopri5(_StepMethod):
    method = "dopri5"


class Tsit5(_StepMethod):
    method = "tsit5"


class Heun(_StepMethod):
    method = "heun"


class IntegralController:
    def __init__(self, atol=1e-7, rtol=1e-7, term: ODETerm | None = None, safety=0.9,
                 factor_min=0.2, factor_max=10.0):
        self.atol, self.rtol, self.term = atol, rtol, term
        self.coeffs = PidCoefficients(1.0, 0.0, 0.0, safety, factor_min, factor_max)


class PIDController(IntegralController):
    """PID step-size control.  Either a batchode preset name (``preset=
    "PI42"``, exact reference coefficients) or torchode/diffrax gains, mapped
    as beta1 = p + i + d, beta2 = -(p + 2d), beta3 = d."""

    def __init__(self, atol=1e-7, rtol=1e-7, pcoeff=0.0, icoeff=1.0, dcoeff=0.0,
                 term: ODETerm | None = None, preset: str | None = None, safety=0.9,
                 factor_min=0.2, factor_max=10.0, update_history_on_reject=True):
        super().__init__(atol, rtol, term, safety, factor_min, factor_max)
        if preset is not None:
            if preset not in PID_PRESETS:
                raise ValueError(f"unknown PID preset {preset!r}; available: {sorted(PID_PRESETS)}")
            b1, b2, b3 = PID_PRESETS[preset]
        else:
            b1, b2, b3 = pcoeff + icoeff + dcoeff, -(pcoeff + 2.0 * dcoeff), dcoeff
        self.coeffs = PidCoefficients(b1, b2, b3, safety, factor_min, factor_max,
                                      update_history_on_reject)


@dataclass
class Solution:
    """ts (batch, m) or (m,); ys (batch, m, features), NaN where an instance
    never reached the point (failed instances; batchode's "absent" rows);
    status (batch,) SolveStatus codes; stats: n_steps / n_accepted /
    n_f_evals / final_dt (batch,) tensors plus n_emitted."""

    ts: "object"
    ys: "object"
    status: "object"
    stats: dict


class AutoDiffAdjoint:
    """Solver facade (torchode's name).  ``solve`` runs the batch through the
    persistent sm_100a integrator; it is forward only."""

    def __init__(self, step_method: _StepMethod, step_size_controller: IntegralController,
                 max_steps: int | None = None, mode: str = "exact"):
        self.step_method = step_method
        self.controller = step_size_controller
        self.max_steps = max_steps or DEFAULT_MAX_STEPS
        self.mode = mode

    def solve(self, problem: InitialValueProblem, term: ODETerm | None = None, dt0=None,
              cost_hint=None) -> Solution:
        import torch

        term = term or self.step_method.term or self.controller.term
        if term is None:
            raise ValueError("no ODETerm given")
        n = problem.batch_size
        te = problem.t_eval
        out = solve_device(problem.y0, problem.t_start, problem.t_end, term.f, t_eval=te,
                           method=self.step_method.method, atol=self.controller.atol,
                           rtol=self.controller.rtol, controller=self.controller.coeffs,
                           max_steps=self.max_steps, dt0=dt0, cost_hint=cost_hint,
                           mode=self.mode)
        d = problem.y0.shape[1]
        if te is None:
            ys = out["ys"].new_empty((n, 0, d))
        else:
            m = te.shape[-1]
            ys = out["ys"].reshape(n, m, d)
            reached = torch.arange(m, device=ys.device)[None, :] < out["n_emitted"][:, None]
            ys = torch.where(reached[:, :, None], ys, torch.full_like(ys, float("nan")))
        stats = {k: out[k] for k in ("n_steps", "n_accepted", "final_dt", "n_emitted")}
        stats["n_f_evals"] = out["n_f_evals"].expand(n)
        return Solution(ts=te, ys=ys, status=out["status"].to(torch.int64), stats=stats)
