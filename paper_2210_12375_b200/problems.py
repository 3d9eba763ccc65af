"""Van der Pol batch builders (the reference's ``vdp_limit_cycle`` and
``vdp_batch``, problems.py:53-143) on top of the GPU solve.

Both need one tight-tolerance trajectory of a single oscillator: first to
settle onto the limit cycle and time one revolution, then to sample the
cycle at the requested phases.  Here both trajectories come from the
persistent sm_100a kernel (:func:`solve`); what is left on the host is the
section-crossing arithmetic on the sampled trajectory:

* the Poincare section is ``xdot = 0`` crossed from above; a crossing lies
  between grid samples k and k+1 with ``v_k > 0 >= v_{k+1}`` and its time
  is the secant root of v on that interval;
* crossings in the first 2% of the horizon are transients of the start
  (2, 0), which already sits on the section;
* the period is the spacing of the last two crossings and the anchor the
  grid sample that opens the last full revolution.

Same return values, caching, validation and errors as the reference.
"""

import functools
from typing import NamedTuple

import numpy as np

from .controller import Tolerances
from .dynamics import VdpParams, vdp_dynamics
from .solver import IvpBatch, SolveStatus, solve

__all__ = ["vdp_limit_cycle", "vdp_batch"]

# samples of the settling trajectory, and a step budget no VdP cycle reaches
_SETTLE_SAMPLES = 8000
_STEP_BUDGET = 5_000_000
# the section-crossing search ignores this leading share of the horizon
_TRANSIENT_SHARE = 0.02


class _Section(NamedTuple):
    sample: np.ndarray  # grid index k opening each crossing interval [k, k+1]
    time: np.ndarray    # secant-refined crossing times


def _settle_horizon(mu: float) -> float:
    """About four revolutions: the period is ~2 pi for small mu and grows
    like (3 - 2 ln 2) mu for relaxation oscillations."""
    return 4.0 * (6.3 + 1.7 * mu)


def _one_trajectory(mu: float, start, t_final: float, samples: np.ndarray, tol: float):
    """States of one oscillator at ``samples`` (GPU solve, tight tolerance)."""
    batch = IvpBatch(np.asarray(start, dtype=float).reshape(1, 2), np.zeros(1),
                     np.array([t_final]), [samples])
    out = solve(batch, vdp_dynamics(VdpParams(mu)), tol=Tolerances(tol, tol),
                max_steps=_STEP_BUDGET)
    return out.status[0] == SolveStatus.SUCCESS, out.ys[0]


def _downward_section(times: np.ndarray, xdot: np.ndarray, t_min: float) -> _Section:
    above, below = xdot[:-1], xdot[1:]
    k = np.nonzero((above > 0.0) & (below <= 0.0))[0]
    k = k[times[k] > t_min]
    frac = xdot[k] / (xdot[k] - xdot[k + 1])
    return _Section(k, times[k] + frac * (times[k + 1] - times[k]))


@functools.lru_cache(maxsize=None)
def vdp_limit_cycle(mu: float, tol: float = 1e-10) -> tuple[tuple[float, float], float]:
    """``(anchor, period)``: a state on the limit cycle and the revolution
    time, for one damping strength (reference problems.py:53-97)."""
    horizon = _settle_horizon(mu)
    grid = np.linspace(0.0, horizon, _SETTLE_SAMPLES)
    ok, states = _one_trajectory(mu, (2.0, 0.0), horizon, grid, tol)
    if not ok:
        raise RuntimeError(f"limit-cycle pre-integration failed for mu={mu}")
    sec = _downward_section(grid, states[:, 1], _TRANSIENT_SHARE * horizon)
    if len(sec.time) < 2:
        raise RuntimeError(f"not enough Poincare returns for mu={mu}")
    last, prev = sec.time[-1], sec.time[-2]
    x0, v0 = states[sec.sample[-2]]
    return (float(x0), float(v0)), float(last - prev)


def vdp_batch(n: int, mu: float, phase_spread: float = 2.0 * np.pi, n_eval: int = 0) -> IvpBatch:
    """``n`` oscillators started at evenly spaced phases covering
    ``phase_spread`` radians of the limit cycle, each integrated over one
    period, optionally with ``n_eval`` evenly spaced output times
    (reference problems.py:100-143)."""
    if n < 1:
        raise ValueError("need at least one instance")
    if not 0.0 <= phase_spread <= 2.0 * np.pi:
        raise ValueError("phase_spread must lie in [0, 2 pi]")
    anchor, period = vdp_limit_cycle(float(mu))
    if n > 1 and phase_spread != 0.0:
        # phase j of n sits j/n of the spread along the cycle, in time units
        # (the reference's rounding order, so the start states agree bitwise)
        lag = period * phase_spread * np.arange(n) / (2.0 * np.pi * n)
        ok, y0 = _one_trajectory(mu, anchor, period, lag, 1e-10)
        if not ok:
            raise RuntimeError(f"phase sampling failed for mu={mu}")
        y0 = np.array(y0)
    else:
        y0 = np.repeat(np.asarray(anchor, dtype=float)[None, :], n, axis=0)
    outputs = np.linspace(0.0, period, n_eval) if n_eval > 0 else np.empty(0)
    return IvpBatch(y0, np.zeros(n), np.full(n, period), [outputs] * n)
