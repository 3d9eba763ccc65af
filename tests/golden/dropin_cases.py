"""Drop-in parity cases: the reference's plugin surface used as the reference
uses it -- plain NumPy lambdas / closures as dynamics (stepper.py:19-20) and
a user-built ButcherTableau (tableau.py:17-83) -- shared by the golden
generator (``make_golden_dropin.py``, which runs them through the reference
``batchode``) and the GPU tests (``tests/test_gpu_dropin.py``, which run the
SAME callables through ``paper_2210_12375_b200``).  Nothing here imports the
reference or the product: a case is data plus NumPy code.
"""

import numpy as np


def bs3_data():
    """Bogacki-Shampine 3(2), FSAL, with the cubic Hermite dense output built
    from k0 and the FSAL stage (weights w_i(theta) = h01 b_i + [i=0] h10 +
    [i=3] h11; w_i(1) = b_i, so it passes ButcherTableau.validate)."""
    a = np.zeros((4, 4))
    a[1, 0] = 1 / 2
    a[2, 1] = 3 / 4
    a[3, :3] = [2 / 9, 1 / 3, 4 / 9]
    b = np.array([2 / 9, 1 / 3, 4 / 9, 0.0])
    b_hat = np.array([7 / 24, 1 / 4, 1 / 3, 1 / 8])
    c = np.array([0.0, 1 / 2, 3 / 4, 1.0])
    interp = np.array([
        [1.0, 3 * b[0] - 2.0, 1.0 - 2 * b[0]],
        [0.0, 3 * b[1], -2 * b[1]],
        [0.0, 3 * b[2], -2 * b[2]],
        [0.0, -1.0, 1.0],
    ])
    return dict(stages=4, a=a, b=b, b_err=b - b_hat, c=c, order=3, error_order=2,
                interp_coeffs=interp, fsal=True)


def ralston_data():
    """Ralston 2(1) with an Euler embedding, non-FSAL, with the linear dense
    output w_i(theta) = b_i theta (m = 1 interpolant term)."""
    a = np.zeros((2, 2))
    a[1, 0] = 2 / 3
    b = np.array([1 / 4, 3 / 4])
    return dict(stages=2, a=a, b=b, b_err=b - np.array([1.0, 0.0]), c=np.array([0.0, 2 / 3]),
                order=2, error_order=1, interp_coeffs=b[:, None].copy(), fsal=False)


# ------------------------------------------------------------- dynamics --
def make_dynamics(name, n, rng):
    """-> (f, description).  Per-instance closures are drawn from rng."""
    if name == "vdp_closure":
        mu = rng.uniform(1.0, 10.0, n)

        def f(t, y):  # problems.py:41-50 written as a user would
            x, v = y[:, 0], y[:, 1]
            return np.stack([v, mu * (1.0 - x * x) * v - x], axis=1)
        return f
    if name == "neg":
        return lambda t, y: -y
    if name == "forced_linear":
        lam = -rng.uniform(0.5, 3.0, n)
        return lambda t, y: lam[:, None] * y + np.cos(3.0 * t)[:, None]
    if name == "damped_stack":  # the reference's own test_stepper.py:165-166
        return lambda t, y: np.stack([y[:, 1], -y[:, 0] - 0.1 * y[:, 1] * np.abs(y[:, 1])],
                                     axis=1)
    if name == "where_blowup":  # test_stepper.py:72-73 + a blow-up
        return lambda t, y: np.where(y > 2.0, np.inf, y * y)
    if name == "lorenz_setitem":
        sigma, rho, beta = 10.0, 28.0, 8.0 / 3.0

        def f(t, y):
            out = np.empty_like(y)
            out[:, 0] = sigma * (y[:, 1] - y[:, 0])
            out[:, 1] = y[:, 0] * (rho - y[:, 2]) - y[:, 1]
            out[:, 2] = y[:, 0] * y[:, 1] - beta * y[:, 2]
            return out
        return f
    if name == "matrix":  # linear system y' = A y through matmul with a constant
        A = np.array([[-0.5, 2.0, 0.0], [-2.0, -0.5, 0.1], [0.0, -0.1, -1.0]])
        return lambda t, y: y @ A.T
    if name == "stiff_pair":  # test_solver.py:271-276 (per-instance rates)
        lam = np.array([-1.0, -2000.0] * (n // 2) + [-1.0] * (n % 2))
        return lambda t, y: lam[:, None] * y
    raise KeyError(name)


# --------------------------------------------------------------- cases --
def solve_cases():
    """(name, dict) full-solve cases."""
    out = []
    rng = np.random.default_rng(11)

    def case(name, dyn, n, d, y0, t_end, te, method="dopri5", tol=1e-6, ctrl=None,
             max_steps=10_000, dt0=None, trace=False, t_start=0.0):
        out.append((name, dict(dyn=dyn, n=n, d=d, y0=y0, t_start=t_start, t_end=t_end, te=te,
                               method=method, tol=tol, ctrl=ctrl or (1.0, 0.0, 0.0),
                               max_steps=max_steps, dt0=dt0, trace=trace, seed=len(out))))

    n = 64
    case("bs3_vdp_pi42", "vdp_closure", n, 2, np.tile([2.0, 0.0], (n, 1)), 10.0,
         np.linspace(0.0, 10.0, 21), method="bs3", ctrl=(0.6, -0.2, 0.0))
    case("bs3_neg_trace", "neg", 8, 2, 1.0 + rng.uniform(0, 1, (8, 2)), 3.0,
         np.array([0.5, 1.5, 3.0]), method="bs3", dt0=0.05, trace=True)
    case("ralston_forced", "forced_linear", 32, 1, rng.normal(size=(32, 1)), 4.0,
         np.linspace(0.0, 4.0, 9), method="ralston", tol=1e-5)
    case("lambda_forced_dopri5", "forced_linear", 48, 2, rng.normal(size=(48, 2)), 6.0,
         np.linspace(0.0, 6.0, 13), tol=1e-8)
    case("lambda_damped_tsit5", "damped_stack", 16, 2, np.tile([1.0, 0.0], (16, 1)), 10.0,
         np.linspace(0.0, 10.0, 11), method="tsit5", tol=1e-9)
    case("lambda_where_blowup", "where_blowup", 6, 1, np.array([[0.3], [0.45], [0.6], [1.0],
                                                                [1.5], [1.9]]), 2.0,
         np.array([0.5, 1.0]), max_steps=200)
    case("lambda_lorenz_setitem", "lorenz_setitem", 8, 3, 1.0 + 0.1 * rng.normal(size=(8, 3)),
         2.0, np.linspace(0.0, 2.0, 41), method="tsit5", tol=1e-8)
    case("lambda_matrix_bs3", "matrix", 16, 3, rng.normal(size=(16, 3)), 5.0,
         np.linspace(0.0, 5.0, 6), method="bs3", tol=1e-7)
    case("lambda_stiff_pair", "stiff_pair", 4, 1, np.ones((4, 1)), 1.0, np.array([1.0]),
         max_steps=100_000)
    return out


def step_cases():
    """BatchSolver.step_once per-iteration cases (solver.py:208-282)."""
    rng = np.random.default_rng(5)
    return [
        # test_solver.py:220-235: one instance accepts the first trial step, one rejects
        ("mixed_accept_reject", dict(dyn="neg_pos", n=2, d=1, y0=np.ones((2, 1)), t_end=1.0,
                                     te=np.empty(0), method="dopri5", atol=np.array([1e-2, 1e-10]),
                                     rtol=np.array([0.0, 0.0]), dt0=0.5, ctrl=(1.0, 0.0, 0.0),
                                     max_steps=10_000)),
        ("vdp_bs3_steps", dict(dyn="vdp_closure", n=24, d=2, y0=np.tile([2.0, 0.0], (24, 1)),
                               t_end=rng.uniform(2.0, 6.0, 24), te=np.linspace(0.0, 2.0, 5),
                               method="bs3", atol=1e-6, rtol=1e-6, dt0=None,
                               ctrl=(0.6, -0.2, 0.0), max_steps=10_000)),
    ]


def step_dynamics(name, n, rng):
    if name == "neg_pos":
        return lambda t, y: y
    return make_dynamics(name, n, rng)
