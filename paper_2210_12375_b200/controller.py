"""Step-size controller configuration (host side).

Mirrors ``batchode.controller``'s configuration types and their
validation (reference ``pkg/src/batchode/controller.py``): ``NORM_FLOOR``
(:26), ``PID_PRESETS`` (:30-36), ``Tolerances`` (:39-54),
``PidCoefficients`` (:57-83), ``integral_controller`` (:86-88),
``pid_controller`` (:91-99).  The arithmetic (error norm, factor, accept)
runs on the device inside the persistent solver; ``units.py`` exposes the
same functions as standalone GPU ops.
"""

from dataclasses import dataclass

import numpy as np

__all__ = ["NORM_FLOOR", "PID_PRESETS", "Tolerances", "PidCoefficients",
           "integral_controller", "pid_controller", "ControllerState"]

NORM_FLOOR = 1e-10

PID_PRESETS: dict[str, tuple[float, float, float]] = {
    "PI42": (0.6, -0.2, 0.0),
    "PI33": (2 / 3, -1 / 3, 0.0),
    "PI34": (0.7, -0.4, 0.0),
    "H211": (1 / 6, 1 / 6, 0.0),
    "H312": (1 / 18, 1 / 9, 1 / 18),
}


@dataclass(frozen=True)
class Tolerances:
    """Absolute/relative tolerances: scalars or per-instance (n,) arrays."""

    atol: float | np.ndarray = 1e-6
    rtol: float | np.ndarray = 1e-6

    def __post_init__(self):
        if np.any(np.asarray(self.atol) < 0) or np.any(np.asarray(self.rtol) < 0):
            raise ValueError("tolerances must be nonnegative")
        if np.all(np.asarray(self.atol) == 0) and np.all(np.asarray(self.rtol) == 0):
            raise ValueError("atol and rtol must not both be zero")


@dataclass(frozen=True)
class PidCoefficients:
    """factor = safety * n^(-b1/k) * n_prev^(-b2/k) * n_prev2^(-b3/k),
    k = error_order + 1, clamped to [factor_min, factor_max]."""

    beta1: float = 1.0
    beta2: float = 0.0
    beta3: float = 0.0
    safety: float = 0.9
    factor_min: float = 0.2
    factor_max: float = 10.0
    update_history_on_reject: bool = True

    def __post_init__(self):
        if not (0.0 < self.safety <= 1.0):
            raise ValueError("safety must be in (0, 1]")
        if not (0.0 < self.factor_min < 1.0 < self.factor_max):
            raise ValueError("need 0 < factor_min < 1 < factor_max")


def integral_controller(safety: float = 0.9) -> PidCoefficients:
    return PidCoefficients(beta1=1.0, beta2=0.0, beta3=0.0, safety=safety)


def pid_controller(preset: str, **overrides) -> PidCoefficients:
    try:
        b1, b2, b3 = PID_PRESETS[preset]
    except KeyError:
        raise ValueError(
            f"unknown PID preset {preset!r}; available: {sorted(PID_PRESETS)}"
        ) from None
    return PidCoefficients(beta1=b1, beta2=b2, beta3=b3, **overrides)


@dataclass
class ControllerState:
    """Per-instance controller memory (controller.py:102-117)."""

    norm_prev: np.ndarray
    norm_prev2: np.ndarray
    dt: np.ndarray

    @classmethod
    def initial(cls, dt: np.ndarray) -> "ControllerState":
        n = dt.shape[0]
        return cls(norm_prev=np.ones(n), norm_prev2=np.ones(n), dt=np.array(dt, dtype=float))
