"""bode: B200-native batched independent ODE solving (arXiv 2210.12375).

Drop-in for the reference's solve path (``batchode``; torchode-style names
in :mod:`.torchode`).  Host code is Python; the solve runs in hand-written
sm_100a kernels behind the C ABI in ``include/bode.h`` (``libbode.so``).
"""

from .controller import (NORM_FLOOR, PID_PRESETS, PidCoefficients, Tolerances,
                         integral_controller, pid_controller)
from .dynamics import (AnalyticProblem, DeviceDynamics, VdpParams, analytic_problems,
                       constant_dynamics, damped_dynamics, forced_linear_dynamics,
                       harmonic_dynamics, linear_dynamics, logistic_dynamics,
                       lorenz_dynamics, mlp_dynamics, relaxation_dynamics,
                       sin_plus_t_dynamics, square_dynamics, vdp_dynamics, zero_dynamics)
from .solver import (DEFAULT_MAX_STEPS, IvpBatch, Solution, SolveStats, SolveStatus, host_empty,
                     pinned, solve, solve_device, solve_joint, adjoint_device)
from .tableau import ButcherTableau, dopri5, heun, tsit5
from .units import ControllerState, StepResult, adapt_step, error_norm, initial_step
from .stepping import BatchSolver, Stepper, interpolate, rk_step
from .problems import vdp_batch, vdp_limit_cycle
from .trace import TraceError

__version__ = "0.1.0"

__all__ = [
    "NORM_FLOOR", "PID_PRESETS", "PidCoefficients", "Tolerances", "integral_controller",
    "pid_controller", "AnalyticProblem", "DeviceDynamics", "VdpParams", "analytic_problems",
    "constant_dynamics", "damped_dynamics", "forced_linear_dynamics", "harmonic_dynamics",
    "linear_dynamics", "logistic_dynamics", "lorenz_dynamics", "mlp_dynamics",
    "relaxation_dynamics", "sin_plus_t_dynamics", "square_dynamics", "vdp_dynamics",
    "zero_dynamics", "DEFAULT_MAX_STEPS", "IvpBatch", "Solution", "SolveStats", "SolveStatus",
    "solve", "solve_joint", "solve_device", "adjoint_device", "pinned", "host_empty", "ButcherTableau", "dopri5", "heun", "tsit5",
    # the rest of batchode's public names (pkg/src/batchode/__init__.py:3-66)
    "BatchSolver", "Stepper", "StepResult", "ControllerState", "rk_step", "interpolate",
    "error_norm", "adapt_step", "initial_step", "vdp_batch", "vdp_limit_cycle", "TraceError",
]
