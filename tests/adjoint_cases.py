"""Seeded scenarios for the gradient (adjoint) tests: the same problem for
the C oracle (forward + trace), the autograd replay oracle and the GPU
adjoint.  Per-instance parameters occupy the leading slots, as the C
oracle's ``make_dyn`` expects."""

import numpy as np

PI42 = dict(betas=(0.6, -0.2, 0.0), safety=0.9, factor_min=0.2, factor_max=10.0, hist=True)
INTEGRAL = dict(betas=(1.0, 0.0, 0.0), safety=0.9, factor_min=0.2, factor_max=10.0, hist=True)
SLOTS = {"vdp": ("mu",), "lorenz": ("sigma", "rho", "beta"), "linear_cos": ("lam", "amp", "omega"),
         "damped": (), "harmonic": (), "logistic": (), "relax_cos": ("lam", "omega"),
         "linear": ("lam",), "sin_plus_t": (), "square": ("thr",)}


def case(name: str, n: int = 16):
    rng = np.random.default_rng(7)
    if name == "vdp_pi42":
        mu = rng.uniform(1.0, 10.0, n)
        y0 = np.tile([2.0, 0.0], (n, 1)) + 0.1 * rng.standard_normal((n, 2))
        t_end = rng.uniform(2.0, 6.0, n)
        te = [np.concatenate([[0.0], np.sort(rng.uniform(0.0, t_end[i], 5)), [t_end[i]]])
              for i in range(n)]
        return dict(method="dopri5", dyn="vdp", params={"mu": mu}, y0=y0, t_start=0.0,
                    t_end=t_end, t_eval=te, ctrl=PI42, tol=1e-6, max_steps=100_000)
    if name == "lorenz_tsit5":
        y0 = 1.0 + 0.1 * rng.standard_normal((n, 3))
        te = np.linspace(0.0, 1.0, 40)
        return dict(method="tsit5", dyn="lorenz",
                    params={"sigma": 10.0, "rho": 28.0, "beta": 8.0 / 3.0}, y0=y0, t_start=0.0,
                    t_end=np.full(n, 1.0), t_eval=[te] * n, ctrl=INTEGRAL, tol=1e-8,
                    max_steps=100_000)
    if name == "linear_cos_heun":
        lam = rng.uniform(-2.0, -0.5, n)
        y0 = rng.standard_normal((n, 2))
        te = np.linspace(0.0, 3.0, 7)
        return dict(method="heun", dyn="linear_cos", params={"lam": lam, "amp": 0.7, "omega": 2.0},
                    y0=y0, t_start=0.0, t_end=np.full(n, 3.0), t_eval=[te] * n, ctrl=INTEGRAL,
                    tol=1e-5, max_steps=100_000)
    if name == "damped_backward":
        y0 = rng.standard_normal((n, 2))
        te = np.linspace(2.0, 0.0, 9)  # backward in time, first point at t_start
        return dict(method="dopri5", dyn="damped", params={}, y0=y0, t_start=2.0,
                    t_end=np.zeros(n), t_eval=[te] * n, ctrl=PI42, tol=1e-7, max_steps=100_000)
    if name == "relax_cos_tsit5":
        lam = rng.uniform(-3.0, -1.0, n)
        y0 = rng.standard_normal((n, 3))
        te = [np.sort(rng.uniform(0.0, 2.0, 4)) for _ in range(n)]
        return dict(method="tsit5", dyn="relax_cos", params={"lam": lam, "omega": 1.5}, y0=y0,
                    t_start=0.0, t_end=np.full(n, 2.0), t_eval=te, ctrl=INTEGRAL, tol=1e-6,
                    max_steps=100_000)
    if name == "vdp_max_steps":  # some instances stop early (MAX_STEPS_EXCEEDED)
        mu = np.linspace(1.0, 30.0, n)
        y0 = np.tile([2.0, 0.0], (n, 1))
        te = np.linspace(0.0, 8.0, 17)
        return dict(method="dopri5", dyn="vdp", params={"mu": mu}, y0=y0, t_start=0.0,
                    t_end=np.full(n, 8.0), t_eval=[te] * n, ctrl=INTEGRAL, tol=1e-6, max_steps=60)
    if name == "square_blowup":  # y' = y^2: STEP_UNDERFLOW rows, INFINITE_DYNAMICS at init
        y0 = np.resize(np.array([0.3, 0.45, 0.9, 2.0]), n)[:, None] * np.ones((n, 1))
        te = np.linspace(0.0, 2.0, 5)
        return dict(method="dopri5", dyn="square", params={"thr": 1.5}, y0=y0, t_start=0.0,
                    t_end=np.full(n, 2.0), t_eval=[te] * n, ctrl=INTEGRAL, tol=1e-6,
                    max_steps=100_000)
    raise KeyError(name)


CASES = ["vdp_pi42", "lorenz_tsit5", "linear_cos_heun", "damped_backward", "relax_cos_tsit5",
         "vdp_max_steps", "square_blowup"]


def oracle_dyn(c: dict) -> dict:
    slots = SLOTS[c["dyn"]]
    inst = [np.asarray(c["params"][s]) for s in slots if np.ndim(c["params"][s])]
    shared = [c["params"][s] for s in slots if not np.ndim(c["params"][s])]
    spec = dict(name=c["dyn"], shared=shared)
    if inst:
        spec["inst"] = np.stack(inst, axis=1)
    return spec


def run_oracle(c: dict):
    import oracle as O

    return O.solve(c["y0"], c["t_start"], c["t_end"], c["t_eval"], oracle_dyn(c),
                   method=c["method"], atol=c["tol"], rtol=c["tol"], ctrl=c["ctrl"],
                   max_steps=c["max_steps"], trace=True)


def grad_seed(c: dict):
    """dL/dys per instance (L = sum <G_i, ys_i>), seeded."""
    rng = np.random.default_rng(11)
    d = c["y0"].shape[1]
    return [rng.standard_normal((len(te), d)) for te in c["t_eval"]]
