"""Seeded parity scenarios shared by the golden generator and the tests.

Each scenario is plain data: the problem (y0, bounds, ragged t_eval), the
dynamics as a registry spec ``(name, per-instance params, shared params)``,
the method, tolerances, controller gains and loop limits.  The golden
generator (``make_golden.py``) turns the spec into a NumPy callable and runs
the reference ``batchode.solve`` on it; the parity tests turn the same spec
into a registered device functor and run the CUDA path.  Nothing here
imports the reference or the product.

Scenario choices follow SURVEY.md §8(d) (C1-C5 concretisations, seeded
prefixes of the full-size draws) and Appendix B (status/edge-case scenarios).
"""

import math

import numpy as np

PI42 = (0.6, -0.2, 0.0)
H312 = (1 / 18, 1 / 9, 1 / 18)
ICTRL = (1.0, 0.0, 0.0)


def _ctrl(betas=ICTRL, safety=0.9, factor_min=0.2, factor_max=10.0, hist=True):
    return dict(betas=tuple(float(b) for b in betas), safety=safety,
                factor_min=factor_min, factor_max=factor_max, hist=hist)


def _scn(name, y0, t_start, t_end, t_eval, dyn, method="dopri5", atol=1e-6,
         rtol=1e-6, ctrl=None, max_steps=10_000, dt0=None, trace=False):
    y0 = np.atleast_2d(np.asarray(y0, dtype=float))
    n = y0.shape[0]
    t_start = np.broadcast_to(np.asarray(t_start, dtype=float), (n,)).copy()
    t_end = np.broadcast_to(np.asarray(t_end, dtype=float), (n,)).copy()
    if t_eval is None:
        t_eval = [np.empty(0)] * n
    t_eval = [np.asarray(te, dtype=float) for te in t_eval]
    return dict(name=name, y0=y0, t_start=t_start, t_end=t_end, t_eval=t_eval,
                dyn=dyn, method=method, atol=atol, rtol=rtol,
                ctrl=ctrl if ctrl is not None else _ctrl(), max_steps=max_steps,
                dt0=dt0, trace=trace)


def dyn(name, inst=None, shared=()):
    """Registry spec: per-instance params (n, p) array or None, shared tuple."""
    if inst is not None:
        inst = np.asarray(inst, dtype=float)
        if inst.ndim == 1:
            inst = inst[:, None]
    return dict(name=name, inst=inst, shared=tuple(float(s) for s in shared))


# --------------------------------------------------------------- C1..C5 --
def c1(n=256):
    rng = np.random.default_rng(0)
    mu = rng.uniform(1.0, 10.0, 256)[:n]
    return _scn("c1_vdp", np.tile([2.0, 0.0], (n, 1)), 0.0, 10.0,
                [np.linspace(0.0, 10.0, 50)] * n, dyn("vdp", mu),
                max_steps=100_000)


def c2_inputs(n_full=2 ** 20):
    rng = np.random.default_rng(0)
    mu = rng.uniform(1.0, 10.0, n_full)
    t_end = rng.uniform(5.0, 20.0, n_full)
    return mu, t_end


def c2(n=1024, n_full=2 ** 20):
    mu, t_end = c2_inputs(n_full)
    mu, t_end = mu[:n], t_end[:n]
    return _scn("c2_vdp_pi42", np.tile([2.0, 0.0], (n, 1)), 0.0, t_end,
                [np.array([te]) for te in t_end], dyn("vdp", mu),
                ctrl=_ctrl(PI42))


def c3_inputs(n_full=2 ** 18):
    rng = np.random.default_rng(0)
    return 1.0 + 0.1 * rng.normal(size=(n_full, 3))


def c3(n=16, n_full=2 ** 18):
    y0 = c3_inputs(n_full)[:n]
    return _scn("c3_lorenz", y0, 0.0, 10.0, [np.linspace(0.0, 10.0, 1000)] * n,
                dyn("lorenz", None, (10.0, 28.0, 8.0 / 3.0)), method="tsit5",
                atol=1e-8, rtol=1e-8, max_steps=100_000)


def c5_inputs(n_full=2 ** 20):
    rng = np.random.default_rng(0)
    return np.exp(rng.uniform(0.0, math.log(1000.0), n_full))


def c5(n=64, n_full=2 ** 20):
    mu = c5_inputs(n_full)[:n]
    return _scn("c5_vdp_stiff", np.tile([2.0, 0.0], (n, 1)), 0.0, 10.0, None,
                dyn("vdp", mu), ctrl=_ctrl(PI42), max_steps=100_000)


def c4_weights(D=64, H=256, seed=0):
    """Seeded MLP weights for C4: W1~N(0,1/D), W2~N(0,1/H),
    b~0.1 N(0,1); returned as float32 like the fp32 numpy oracle uses."""
    rng = np.random.default_rng(seed)
    W1 = (rng.normal(size=(H, D)) / math.sqrt(D)).astype(np.float32)
    b1 = (0.1 * rng.normal(size=H)).astype(np.float32)
    W2 = (rng.normal(size=(D, H)) / math.sqrt(H)).astype(np.float32)
    b2 = (0.1 * rng.normal(size=D)).astype(np.float32)
    return W1, b1, W2, b2


def c4_y0(n, D=64, seed=1):
    return np.random.default_rng(seed).normal(size=(n, D))


# ------------------------------------------------- Appendix B scenarios --
def vdp_tsit5_h312():
    rng = np.random.default_rng(1)
    n = 64
    mu = rng.uniform(1.0, 10.0, n)
    return _scn("vdp_tsit5_h312_nohist", np.tile([2.0, 0.0], (n, 1)), 0.0, 10.0,
                [np.linspace(0.0, 10.0, 20)] * n, dyn("vdp", mu), method="tsit5",
                ctrl=_ctrl(H312, hist=False), trace=True)


def linear_cos_backward():
    rng = np.random.default_rng(3)
    n = 6
    lam = rng.uniform(-3.0, 0.5, n)
    y0 = rng.normal(size=(n, 2))
    tol = 10.0 ** np.linspace(-9.0, -4.0, n)
    te = [np.array([2.0, 1.5, 0.25, 0.0]), np.empty(0), np.array([1.0]),
          np.array([1.9, 1.8, 1.7, 1.6, 1.5, 1.4, 1.3]), np.array([2.0, 2.0, 0.0]),
          np.sort(rng.uniform(0.0, 2.0, 9))[::-1]]
    return _scn("linear_cos_backward", y0, 2.0, 0.0, te,
                dyn("linear_cos", np.stack([lam, np.ones(n)], 1), (3.0,)),
                atol=tol, rtol=tol, trace=True)


def square_blowup(max_steps=100_000, name="square_blowup"):
    te = [np.array([0.5, 1.0, 1.5, 1.9])] * 3
    return _scn(name, [[0.3], [0.45], [0.9]], 0.0, 2.0, te,
                dyn("square", None, (math.inf,)), atol=1e-8, rtol=1e-8,
                max_steps=max_steps, trace=True)


def inf_threshold():
    te = [np.array([0.0, 1.0, 9.0])] * 3
    return _scn("inf_threshold", [[0.1], [0.5], [0.9]], 0.0, 10.0, te,
                dyn("square", None, (0.4,)), trace=True)


def vdp_dt0():
    rng = np.random.default_rng(4)
    n = 64
    mu = rng.uniform(1.0, 10.0, n)
    return _scn("vdp_dt0", np.tile([2.0, 0.0], (n, 1)), 0.0, 10.0,
                [np.linspace(0.0, 10.0, 50)] * n, dyn("vdp", mu), dt0=0.05)


def heun_vdp():
    rng = np.random.default_rng(5)
    n = 32
    mu = rng.uniform(1.0, 10.0, n)
    return _scn("heun_vdp", np.tile([2.0, 0.0], (n, 1)), 0.0, 10.0,
                [np.linspace(0.0, 10.0, 25)] * n, dyn("vdp", mu), method="heun",
                atol=1e-4, rtol=1e-4, trace=True)


def damped_fsal():
    return _scn("damped_fsal", [[1.0, 0.0]], 0.0, 10.0, None, dyn("damped"),
                atol=1e-9, rtol=1e-9, trace=True)


def mixed_accept_reject():
    return _scn("mixed_accept_reject", np.ones((2, 1)), 0.0, 1.0, None,
                dyn("linear", None, (1.0,)), atol=np.array([1e-2, 1e-10]),
                rtol=np.array([0.0, 0.0]), dt0=0.5, trace=True)


def zero_crossing():
    return _scn("zero_crossing", [[1.0]], 0.0, 1.0, [np.array([0.1, 0.2, 0.3])],
                dyn("zero"), dt0=0.4, trace=True)


def analytic_suite():
    rng = np.random.default_rng(6)
    n = 8
    out = []
    te = [np.sort(rng.uniform(0.0, 3.0, 5)) for _ in range(n)]
    lam = rng.uniform(-2.0, 1.0, n)
    out.append(_scn("exponential", rng.uniform(0.5, 2.0, (n, 1)), 0.0, 3.0, te,
                    dyn("linear", lam), atol=1e-9, rtol=1e-9))
    out.append(_scn("harmonic", rng.normal(size=(n, 2)), 0.0, 3.0, te,
                    dyn("harmonic"), atol=1e-9, rtol=1e-9, method="tsit5"))
    out.append(_scn("logistic", rng.uniform(0.05, 0.9, (n, 1)), 0.0, 3.0, te,
                    dyn("logistic"), atol=1e-9, rtol=1e-9))
    out.append(_scn("sin_plus_t", rng.normal(size=(n, 3)), 0.0, 3.0, te,
                    dyn("sin_plus_t"), ctrl=_ctrl(PI42)))
    out.append(_scn("relax_cos", rng.normal(size=(n, 4)), 0.0, 1.0, None,
                    dyn("relax_cos", rng.uniform(-50.0, 0.0, n), (1.0,)),
                    atol=1e-7, rtol=1e-7))
    lam2 = rng.uniform(-5.0, 0.5, 10)
    amp = rng.uniform(0.1, 2.0, 10)
    te2 = [np.sort(rng.uniform(0.0, 3.0, 6)) for _ in range(10)]
    out.append(_scn("linear_sin", rng.normal(size=(10, 2)), 0.0, 3.0, te2,
                    dyn("linear_sin", np.stack([lam2, amp], 1), (1.0,)), trace=True))
    out.append(_scn("constant_const", [[3.0, -1.0]], 0.0, 1.0,
                    [np.array([0.0, 0.3, 1.0])], dyn("zero")))
    out.append(_scn("const_quadrature", np.zeros((2, 2)), 0.0, 1.0,
                    [np.array([0.5, 1.0])] * 2, dyn("const", None, (1.0,)),
                    ctrl=_ctrl(H312)))
    return out


def all_solve_scenarios():
    return [c1(), c2(), c3(), c5(), vdp_tsit5_h312(), linear_cos_backward(),
            square_blowup(), square_blowup(20, "square_maxsteps"), inf_threshold(),
            vdp_dt0(), heun_vdp(), damped_fsal(), mixed_accept_reject(),
            zero_crossing()] + analytic_suite()


# ------------------------------------------------------ tableau builders --
def heun_tableau_data():
    """2-stage Heun-Euler pair: c=[0,1], a10=1,
    b=[1/2,1/2], b_err=[-1/2,1/2], order 2, error order 1, non-FSAL,
    interpolant w0=theta-theta^2/2, w1=theta^2/2."""
    a = np.zeros((2, 2))
    a[1, 0] = 1.0
    return dict(stages=2, a=a, b=np.array([0.5, 0.5]), b_err=np.array([-0.5, 0.5]),
                c=np.array([0.0, 1.0]), order=2, error_order=1,
                interp_coeffs=np.array([[1.0, -0.5], [0.0, 0.5]]), fsal=False)


# --------------------------------------------------- numpy dynamics -----
def numpy_dynamics(spec, n):
    """Reference-side NumPy callable for a registry spec.  The operation
    order here IS the definition the device functors reproduce."""
    name, inst, sh = spec["name"], spec["inst"], spec["shared"]
    col = (lambda j: inst[:, j][:, None]) if inst is not None else None
    if name == "vdp":
        mu = inst[:, 0]

        def f(t, y):
            x = y[:, 0]
            v = y[:, 1]
            return np.stack([v, mu * (1.0 - x * x) * v - x], axis=1)
    elif name == "lorenz":
        s, r, b = sh

        def f(t, y):
            x, yy, z = y[:, 0], y[:, 1], y[:, 2]
            return np.stack([s * (yy - x), x * (r - z) - yy, x * yy - b * z], axis=1)
    elif name == "zero":
        def f(t, y):
            return np.zeros_like(y)
    elif name == "const":
        c = sh[0]

        def f(t, y):
            return np.full_like(y, c)
    elif name == "linear":
        if inst is not None:
            lam = col(0)
        else:
            lam = sh[0]

        def f(t, y):
            return lam * y
    elif name == "linear_cos":
        lam, amp, om = col(0), col(1), sh[0]

        def f(t, y):
            return lam * y + amp * np.cos(om * t)[:, None]
    elif name == "linear_sin":
        lam, amp, om = col(0), col(1), sh[0]

        def f(t, y):
            return lam * y + amp * np.sin(om * t)[:, None]
    elif name == "relax_cos":
        lam, om = col(0), sh[0]

        def f(t, y):
            return lam * (y - np.cos(om * t)[:, None])
    elif name == "square":
        thr = sh[0]

        def f(t, y):
            return np.where(y > thr, np.inf, y * y)
    elif name == "logistic":
        def f(t, y):
            return y * (1.0 - y)
    elif name == "sin_plus_t":
        def f(t, y):
            return np.sin(y) + t[:, None]
    elif name == "harmonic":
        def f(t, y):
            return np.stack([y[:, 1], -y[:, 0]], axis=1)
    elif name == "damped":
        def f(t, y):
            return np.stack([y[:, 1], -y[:, 0] - 0.1 * y[:, 1] * np.abs(y[:, 1])], axis=1)
    else:
        raise KeyError(name)
    return f


# ------------------------------------------------ joint mode (solve_joint) --
def joint_scenarios():
    """solve_joint (solver.py:372-427) parity cases; the pathology case's
    inputs come from the reference's vdp_batch and are stored in its fixture."""
    rng = np.random.default_rng(5)
    out = []
    mu = rng.uniform(1.0, 10.0, 32)
    out.append(_scn("joint_vdp32_I", np.tile([2.0, 0.0], (32, 1)), 0.0, 10.0,
                    [np.linspace(0.0, 10.0, 20)] * 32, dyn("vdp", mu), max_steps=100_000))
    y0 = 1.0 + 0.1 * rng.normal(size=(8, 3))
    out.append(_scn("joint_lorenz_tsit5_trace", y0, 0.0, 2.0, [np.linspace(0.5, 2.0, 4)] * 8,
                    dyn("lorenz", None, (10.0, 28.0, 8.0 / 3.0)), method="tsit5", atol=1e-8,
                    rtol=1e-8, trace=True))
    mu = rng.uniform(1.0, 5.0, 16)
    out.append(_scn("joint_vdp16_pi42_dt0", np.tile([2.0, 0.0], (16, 1)), 0.0, 5.0,
                    [np.array([2.5, 5.0])] * 16, dyn("vdp", mu), ctrl=_ctrl(PI42), dt0=0.01))
    out.append(_scn("joint_single_linear", [[1.0, 2.0]], 0.0, 1.0, [np.array([0.5, 1.0])],
                    dyn("linear", None, (-1.0,))))
    out.append(_scn("joint_heun_harmonic", rng.normal(size=(8, 2)), 0.0, 3.0,
                    [np.linspace(0.0, 3.0, 7)] * 8, dyn("harmonic"), method="heun", atol=1e-4,
                    rtol=1e-4))
    mu = rng.uniform(1.0, 3.0, 300)  # N = 600 > 128: multi-leaf pairwise tree
    out.append(_scn("joint_vdp300_wide", np.tile([2.0, 0.0], (300, 1)), 0.0, 3.0, None,
                    dyn("vdp", mu), atol=1e-7, rtol=1e-7))
    out.append(_scn("joint_square_blowup", [[0.5], [1.0], [0.8]], 0.0, 2.0, [np.array([0.5])] * 3,
                    dyn("square", None, (1e300,)), max_steps=100_000))
    return out
