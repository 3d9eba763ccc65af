"""Van der Pol batch builders on the GPU solve (reference problems.py:53-143).

``vdp_limit_cycle`` pre-integrates one instance at tight tolerance and
measures the cycle period from Poincare returns; ``vdp_batch`` spreads n
instances along that cycle.  Both are the reference's algorithms, with the
integrations done by :func:`solve` (the persistent sm_100a kernel) instead
of NumPy; the post-processing (crossing detection, interpolation) is the
reference's NumPy code path on the solver's output.
"""

import functools

import numpy as np

from .controller import Tolerances
from .dynamics import VdpParams, vdp_dynamics
from .solver import IvpBatch, SolveStatus, solve

__all__ = ["vdp_limit_cycle", "vdp_batch"]


@functools.lru_cache(maxsize=None)
def vdp_limit_cycle(mu: float, tol: float = 1e-10) -> tuple[tuple[float, float], float]:
    """A point on the limit cycle and the cycle period, for one mu
    (problems.py:53-97): ``(anchor, period)``."""
    horizon = 4.0 * (6.3 + 1.7 * mu)  # the relaxation period grows like (3 - 2 ln 2) mu
    n_grid = 8000
    grid = np.linspace(0.0, horizon, n_grid)
    problem = IvpBatch(y0=np.array([[2.0, 0.0]]), t_start=np.array([0.0]),
                       t_end=np.array([horizon]), t_eval=[grid])
    sol = solve(problem, vdp_dynamics(VdpParams(mu)), tol=Tolerances(atol=tol, rtol=tol),
                max_steps=5_000_000)
    if sol.status[0] != SolveStatus.SUCCESS:
        raise RuntimeError(f"limit-cycle pre-integration failed for mu={mu}")
    states = sol.ys[0]
    v = states[:, 1]
    # downward zero crossings of xdot, skipping the t = 0 boundary crossing
    sign_change = (v[:-1] > 0.0) & (v[1:] <= 0.0)
    idx = np.flatnonzero(sign_change)
    idx = idx[grid[idx] > horizon * 0.02]
    if idx.size < 2:
        raise RuntimeError(f"not enough Poincare returns for mu={mu}")
    t_cross = grid[idx] + (grid[idx + 1] - grid[idx]) * v[idx] / (v[idx] - v[idx + 1])
    period = float(t_cross[-1] - t_cross[-2])
    anchor_state = states[idx[-2]]
    return (float(anchor_state[0]), float(anchor_state[1])), period


def vdp_batch(n: int, mu: float, phase_spread: float = 2.0 * np.pi, n_eval: int = 0) -> IvpBatch:
    """n Van der Pol problems phase-shifted along the limit cycle, each over
    one period (problems.py:100-143)."""
    if n < 1:
        raise ValueError("need at least one instance")
    if not (0.0 <= phase_spread <= 2.0 * np.pi):
        raise ValueError("phase_spread must lie in [0, 2 pi]")
    anchor, period = vdp_limit_cycle(float(mu))
    offsets = period * phase_spread * np.arange(n) / (2.0 * np.pi * n)
    if n == 1 or phase_spread == 0.0:
        y0 = np.tile(np.asarray(anchor), (n, 1))
    else:
        sampler = IvpBatch(y0=np.array([list(anchor)]), t_start=np.array([0.0]),
                           t_end=np.array([period]), t_eval=[offsets])
        sampled = solve(sampler, vdp_dynamics(VdpParams(mu)), tol=Tolerances(1e-10, 1e-10),
                        max_steps=5_000_000)
        if sampled.status[0] != SolveStatus.SUCCESS:
            raise RuntimeError(f"phase sampling failed for mu={mu}")
        y0 = np.array(sampled.ys[0])
    t_eval = [np.linspace(0.0, period, n_eval) if n_eval > 0 else np.empty(0) for _ in range(n)]
    return IvpBatch(y0=y0, t_start=np.zeros(n), t_end=np.full(n, period), t_eval=t_eval)
