"""CPU oracle for the gradient path (``bode_solve_adjoint``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/`` as the checker, never by
the product package.

The reference has no gradients (SURVEY.md §8(f) row 1 names
"torch autograd on CPU" as the oracle to build).  This module replays a
solve's accepted steps -- the (t_old, h) sequence the pinned C oracle
records in its trace (``oracle.solve(..., trace=True)``) -- as torch fp64
operations on the CPU, in the reference's operation order:

  stage i      Stepper.step            stepper.py:83-89
  y_next       Stepper.step            stepper.py:93-101
  dense output Stepper.interpolate     stepper.py:112-139, emitted by the
               cursor rule of BatchSolver._emit (solver.py:284-322)
  points at t_start are copies of y0   solver.py:200-206

and differentiates it with torch.autograd.  The step sizes are data (the
definition of the product's gradient: discretise-then-optimise with the
step-size controller held fixed).  Parity status of this oracle:
``tests/test_adjoint_oracle.py`` checks that the replayed ys equal the
pinned C oracle's ys and that the autograd gradients equal central finite
differences of the replay.
"""

import os
import re

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
_COEFFS = os.path.join(HERE, "..", "paper_2210_12375_b200", "csrc", "tableau_coeffs.h")


def tableau(method: str) -> dict:
    """Coefficients of the generated header the C oracle also compiles
    (a (7,7) | b | b_err | c | w (7,4), checked against the reference's
    tableau.py by tests/test_oracle_golden.py)."""
    src = open(_COEFFS).read()
    key = method.upper()
    S = int(re.search(rf"#define BODE_{key}_STAGES (\d+)", src).group(1))
    NI = int(re.search(rf"#define BODE_{key}_NINTERP (\d+)", src).group(1))
    fsal = int(re.search(rf"#define BODE_{key}_FSAL (\d+)", src).group(1))
    flat = re.search(rf"#define BODE_{key}_FLAT_INIT \{{([^}}]*)\}}", src).group(1)
    v = np.array([float.fromhex(x.strip()) for x in flat.split(",")])
    return dict(S=S, NI=NI, fsal=bool(fsal), a=v[:49].reshape(7, 7)[:S, :S], b=v[49:56][:S],
                c=v[63:70][:S], w=v[70:98].reshape(7, 4)[:S, :NI])


def dynamics(name: str):
    """torch restatements of the registered functors (include/bode.h)."""
    inf = float("inf")

    def vdp(t, y, p):
        x, v = y[0], y[1]
        return torch.stack([v, p["mu"] * (1.0 - x * x) * v - x])

    def lorenz(t, y, p):
        x, yy, z = y[0], y[1], y[2]
        return torch.stack([p["sigma"] * (yy - x), x * (p["rho"] - z) - yy,
                            x * yy - p["beta"] * z])

    def harmonic(t, y, p):
        return torch.stack([y[1], -y[0]])

    def damped(t, y, p):
        return torch.stack([y[1], -y[0] - 0.1 * y[1] * torch.abs(y[1])])

    table = {
        "vdp": vdp, "lorenz": lorenz, "harmonic": harmonic, "damped": damped,
        "zero": lambda t, y, p: torch.zeros_like(y),
        "const": lambda t, y, p: p["c"] * torch.ones_like(y),
        "linear": lambda t, y, p: p["lam"] * y,
        "linear_cos": lambda t, y, p: p["lam"] * y + p["amp"] * torch.cos(p["omega"] * t),
        "linear_sin": lambda t, y, p: p["lam"] * y + p["amp"] * torch.sin(p["omega"] * t),
        "relax_cos": lambda t, y, p: p["lam"] * (y - torch.cos(p["omega"] * t)),
        "square": lambda t, y, p: torch.where(y > p["thr"], torch.full_like(y, inf), y * y),
        "logistic": lambda t, y, p: y * (1.0 - y),
        "sin_plus_t": lambda t, y, p: torch.sin(y) + t,
    }
    return table[name]


def accepted_steps(ref: dict, i: int) -> list:
    """(t_old, h) of instance i's accepted steps from an oracle trace."""
    ns = int(ref["n_steps"][i])
    acc = ref["trace_accept"][i, :ns].astype(bool)
    return list(zip(ref["trace_t"][i, :ns][acc].tolist(), ref["trace_dt"][i, :ns][acc].tolist()))


def replay(method: str, f, params: dict, y0: torch.Tensor, t0: float, steps: list,
           t_eval: np.ndarray) -> torch.Tensor:
    """ys of ONE instance (rows = emitted points) as a torch function of y0
    and params, given its accepted steps."""
    T = tableau(method)
    S, NI = T["S"], T["NI"]
    a, b, c, w = T["a"], T["b"], T["c"], T["w"]
    out = []
    cur = 0
    m = len(t_eval)
    while cur < m and t_eval[cur] == t0:
        out.append(y0)
        cur += 1
    y = y0
    for (t, h) in steps:
        k = [f(torch.tensor(t, dtype=torch.float64), y, params)]
        for i in range(1, S):
            acc = a[i, 0] * k[0]
            for j in range(1, i):
                acc = acc + a[i, j] * k[j]
            ys = h * acc + y
            k.append(f(torch.tensor(t + c[i] * h, dtype=torch.float64), ys, params))
        while cur < m:
            theta = (t_eval[cur] - t) / h
            if not theta <= 1.0:
                break
            theta = max(theta, 0.0)
            acc = None
            for i in range(S):
                v = w[i, NI - 1]
                for j in range(NI - 2, -1, -1):
                    v = v * theta + w[i, j]
                v = v * theta
                acc = v * k[i] if acc is None else acc + v * k[i]
            out.append(y + h * acc)
            cur += 1
        acc = b[0] * k[0]
        for i in range(1, S):
            acc = acc + b[i] * k[i]
        y = y + h * acc
    if not out:
        return y0.new_zeros((0, y0.shape[0]))
    return torch.stack(out)


def gradients(method: str, dyn_name: str, params: dict, y0: np.ndarray, t_start, ref: dict,
              t_eval: list, grad_ys: list):
    """dL/dy0 (n, d) and dL/dparams ({name: (n,)} per-instance contributions)
    for L = sum_i <grad_ys[i], ys_i>, by torch autograd through the replay.
    ``params``: {name: scalar or (n,) array}; ``t_eval``/``grad_ys``: per
    instance lists."""
    f = dynamics(dyn_name)
    y0 = np.atleast_2d(y0)
    n, d = y0.shape
    t0 = np.broadcast_to(np.asarray(t_start, dtype=np.float64), (n,))
    gy0 = np.zeros((n, d))
    gp = {k: np.zeros(n) for k in params}
    for i in range(n):
        yi = torch.tensor(y0[i], dtype=torch.float64, requires_grad=True)
        pi = {k: torch.tensor(float(np.broadcast_to(v, (n,))[i]), dtype=torch.float64,
                              requires_grad=True) for k, v in params.items()}
        ys = replay(method, f, pi, yi, float(t0[i]), accepted_steps(ref, i),
                    np.asarray(t_eval[i], dtype=np.float64))
        g = torch.as_tensor(np.asarray(grad_ys[i])[:ys.shape[0]], dtype=torch.float64)
        loss = (ys * g).sum()
        leaves = [yi] + list(pi.values())
        if not loss.requires_grad:
            continue
        grads = torch.autograd.grad(loss, leaves, allow_unused=True)
        gy0[i] = grads[0].numpy() if grads[0] is not None else 0.0
        for (k, _), gk in zip(pi.items(), grads[1:]):
            gp[k][i] = float(gk) if gk is not None else 0.0
    return gy0, gp


def replay_ys(method: str, dyn_name: str, params: dict, y0: np.ndarray, t_start, ref: dict,
              t_eval: list) -> list:
    """The replayed ys per instance (no gradients), for checking the replay
    against the C oracle's own ys."""
    f = dynamics(dyn_name)
    y0 = np.atleast_2d(y0)
    n = y0.shape[0]
    t0 = np.broadcast_to(np.asarray(t_start, dtype=np.float64), (n,))
    res = []
    with torch.no_grad():
        for i in range(n):
            pi = {k: torch.tensor(float(np.broadcast_to(v, (n,))[i]), dtype=torch.float64)
                  for k, v in params.items()}
            res.append(replay(method, f, pi, torch.tensor(y0[i], dtype=torch.float64),
                              float(t0[i]), accepted_steps(ref, i),
                              np.asarray(t_eval[i], dtype=np.float64)).numpy())
    return res


def mlp_dynamics(W1, b1, W2, b2):
    """f(y) = W2 tanh(W1 y + b1) + b2 in fp32 on the fp64 state (the C4
    oracle's NumPy fp32 MLP), as a torch function."""

    def f(t, y, p):
        z = p["W1"] @ y.to(torch.float32) + p["b1"]
        return (p["W2"] @ torch.tanh(z) + p["b2"]).to(torch.float64)

    return f


def gradients_mlp(method: str, weights, y0: np.ndarray, t_start, steps: list, t_eval: list,
                  grad_ys: list):
    """dL/dy0 (n, d) and the batch-summed dL/dW1, db1, dW2, db2 for
    L = sum_i <grad_ys[i], ys_i>, replaying the given accepted steps
    (``steps[i]`` = list of (t_old, h)) with the fp32 MLP."""
    f = mlp_dynamics(*weights)
    y0 = np.atleast_2d(y0)
    n, d = y0.shape
    t0 = np.broadcast_to(np.asarray(t_start, dtype=np.float64), (n,))
    p = {k: torch.tensor(np.asarray(v, dtype=np.float32), requires_grad=True)
         for k, v in zip(("W1", "b1", "W2", "b2"), weights)}
    gy0 = np.zeros((n, d))
    total = None
    for i in range(n):
        yi = torch.tensor(y0[i], dtype=torch.float64, requires_grad=True)
        ys = replay(method, f, p, yi, float(t0[i]), steps[i], np.asarray(t_eval[i], np.float64))
        g = torch.as_tensor(np.asarray(grad_ys[i])[:ys.shape[0]], dtype=torch.float64)
        loss = (ys * g).sum()
        (gyi,) = torch.autograd.grad(loss, [yi], retain_graph=True) if loss.requires_grad else (None,)
        if gyi is not None:
            gy0[i] = gyi.numpy()
        total = loss if total is None else total + loss
    gw = torch.autograd.grad(total, list(p.values()), allow_unused=True)
    return gy0, {k: (g.numpy() if g is not None else np.zeros_like(v.detach().numpy()))
                 for (k, v), g in zip(p.items(), gw)}
