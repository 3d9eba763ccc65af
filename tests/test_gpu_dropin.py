"""The reference's plugin surface on the GPU: NumPy lambdas / closures as
dynamics (stepper.py:19-20, traced into device functors) and user-built
ButcherTableaus (tableau.py:17-83, compiled into run-time programs), through
every entry point a ``batchode`` user has -- ``solve``, ``BatchSolver``
(step_once / run / solution), ``Stepper`` / ``rk_step`` / ``interpolate``,
``solve_joint`` -- against golden fixtures produced by running the
reference itself on the SAME callables (tests/golden/make_golden_dropin.py).

Bars (as for the registered-functor parity tests): statuses, n_steps,
n_accepted, n_emitted, n_f_evals identical; ys within 1e-10 of each
instance's scale (exact mode).  Where a callable uses a transcendental
(np.cos / np.sin) the device libm differs from NumPy's by ~1 ulp, so those
cases are held to 1e-9 and are not expected to be bitwise.

The reference's own step_once / Stepper tests (tests/test_solver.py:186-241,
tests/test_stepper.py) are re-expressed below with their lambdas, imported
under the name ``batchode``.  One reference test does not apply:
test_stepper.py::test_fsal_evaluation_count counts Python calls of ``f``,
and a device solver never calls the Python callable per stage (it is
traced once).
"""
import os
import sys

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2210_12375_b200 as batchode

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import dropin_cases as DC  # noqa: E402

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "dropin.npz"))


def tableau(name):
    if name == "dopri5":
        return batchode.dopri5()
    if name == "tsit5":
        return batchode.tsit5()
    tab = batchode.ButcherTableau(**(DC.bs3_data() if name == "bs3" else DC.ralston_data()))
    tab.validate()
    return tab


def ctrl(b):
    return batchode.PidCoefficients(beta1=b[0], beta2=b[1], beta3=b[2])


TRANSCENDENTAL = {"forced_linear"}


def _scaled(a, b, counts, d):
    errs = []
    o = 0
    for c in counts:
        x, y = a[o:o + c].reshape(-1, d), b[o:o + c].reshape(-1, d)
        o += c
        if c:
            errs.append(float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300)))
    return max(errs) if errs else 0.0


@pytest.mark.parametrize("name", [c[0] for c in DC.solve_cases()])
def test_solve_lambda_and_custom_tableau_match_reference(name):
    c = dict(DC.solve_cases())[name]
    n, d = c["n"], c["d"]
    f = DC.make_dynamics(c["dyn"], n, np.random.default_rng(1000 + c["seed"]))
    t_end = np.broadcast_to(np.asarray(c["t_end"], dtype=float), (n,)).copy()
    prob = batchode.IvpBatch(c["y0"], np.full(n, c["t_start"]), t_end,
                             [c["te"].copy() for _ in range(n)])
    sol = batchode.solve(prob, f, tableau=tableau(c["method"]),
                         tol=batchode.Tolerances(c["tol"], c["tol"]), controller=ctrl(c["ctrl"]),
                         max_steps=c["max_steps"], dt0=c["dt0"], record_trace=c["trace"])
    k = f"solve/{name}/"
    assert np.array_equal(sol.status, G[k + "status"])
    assert np.array_equal(sol.stats.n_steps, G[k + "n_steps"])
    assert np.array_equal(sol.stats.n_accepted, G[k + "n_accepted"])
    assert np.array_equal(sol.stats.n_f_evals, G[k + "n_f_evals"])
    ne = np.array([len(y) for y in sol.ys])
    assert np.array_equal(ne, G[k + "n_emitted"])
    ys = np.concatenate([np.asarray(y).reshape(-1, d) for y in sol.ys])
    err = _scaled(ys, G[k + "ys"], ne, d)
    assert err <= (1e-9 if c["dyn"] in TRANSCENDENTAL else 1e-10), err
    fin = np.isfinite(G[k + "final_dt"])
    rel = np.abs(sol.stats.final_dt[fin] - G[k + "final_dt"][fin]) / np.abs(G[k + "final_dt"][fin])
    assert np.all(rel <= 1e-5)
    if c["trace"]:
        acc = np.concatenate(sol.stats.extra["trace_accept"])
        assert np.array_equal(acc, G[k + "trace_accept"])


@pytest.mark.parametrize("name", [c[0] for c in DC.step_cases()])
def test_batchsolver_step_once_per_iteration_matches_reference(name):
    c = dict(DC.step_cases())[name]
    n, d = c["n"], c["d"]
    f = DC.step_dynamics(c["dyn"], n, np.random.default_rng(2000))
    t_end = np.broadcast_to(np.asarray(c["t_end"], dtype=float), (n,)).copy()
    prob = batchode.IvpBatch(c["y0"], np.zeros(n), t_end, [c["te"].copy() for _ in range(n)])
    s = batchode.BatchSolver(prob, f, tableau=tableau(c["method"]),
                             tol=batchode.Tolerances(c["atol"], c["rtol"]),
                             controller=ctrl(c["ctrl"]), max_steps=c["max_steps"], dt0=c["dt0"],
                             record_trace=True)
    k = f"step/{name}/"
    iters = G[k + "n_steps"].shape[0]
    for it in range(iters):
        more = s.step_once()
        assert more == (it < iters - 1)
        assert np.array_equal(s.status, G[k + "status"][it])
        assert np.array_equal(s.n_steps, G[k + "n_steps"][it])
        assert np.array_equal(s.n_accepted, G[k + "n_accepted"][it])
        assert np.array_equal(s._cursor, G[k + "cursor"][it])
        assert np.array_equal(s.fsal_valid, G[k + "fsal_valid"][it])
        assert s.n_f_evals == int(G[k + "n_f_evals"][it])
        ref_t, ref_y = G[k + "t"][it], G[k + "y"][it]
        assert np.max(np.abs(s.t - ref_t) / np.maximum(np.abs(ref_t), 1e-300)) <= 1e-12
        assert np.max(np.abs(s.y - ref_y)) <= 1e-10 * max(np.max(np.abs(ref_y)), 1.0)
        rel = np.abs(s.ctrl.dt - G[k + "dt"][it]) / np.maximum(np.abs(G[k + "dt"][it]), 1e-300)
        assert np.all(rel <= 1e-5)
    assert s.step_once() is False
    sol = s.solution()
    ys = np.concatenate([np.asarray(y).reshape(-1, d) for y in sol.ys])
    assert ys.shape == G[k + "ys"].shape
    if ys.size:
        assert np.max(np.abs(ys - G[k + "ys"])) <= 1e-10 * max(np.max(np.abs(G[k + "ys"])), 1.0)
    assert np.array_equal(np.concatenate(sol.stats.extra["trace_accept"]), G[k + "trace_accept"])


# ---- the reference's tests/test_solver.py step_once cases (:186-241) ----
def make_problem(y0, t_end=1.0, t_eval=None):
    y0 = np.atleast_2d(y0)
    n = y0.shape[0]
    if t_eval is None:
        t_eval = [np.empty(0)] * n
    return batchode.IvpBatch(y0=y0, t_start=np.zeros(n), t_end=np.full(n, t_end), t_eval=t_eval)


def test_time_monotone_and_ends_exactly():
    problem = make_problem(np.ones((1, 1)), t_end=3.0)
    solver = batchode.BatchSolver(problem, lambda t, y: -y, record_trace=True)
    ts = [solver.t[0]]
    while solver.step_once():
        ts.append(solver.t[0])
    ts.append(solver.t[0])
    assert np.all(np.diff(ts) >= 0)
    assert solver.t[0] == 3.0


def test_fixpoint_when_all_finished():
    problem = make_problem(np.ones((1, 1)))
    solver = batchode.BatchSolver(problem, lambda t, y: np.zeros_like(y))
    while solver.step_once():
        pass
    calls = []

    def spy(t, y):
        calls.append(1)
        return np.zeros_like(y)

    solver.f = spy
    assert solver.step_once() is False
    assert not calls


def test_mixed_accept_reject():
    tol = batchode.Tolerances(atol=np.array([1e-2, 1e-10]), rtol=np.array([0.0, 0.0]))
    problem = make_problem(np.ones((2, 1)))
    solver = batchode.BatchSolver(problem, lambda t, y: y, tol=tol, dt0=0.5, record_trace=True)
    solver.step_once()
    acc = [solver._trace_accept[i][0] for i in range(2)]
    assert acc == [True, False]
    assert solver.t[0] == 0.5
    assert solver.t[1] == 0.0
    assert solver.ctrl.dt[0] != 0.5
    assert solver.ctrl.dt[1] != 0.5


def test_step_crossing_three_eval_points():
    problem = make_problem(np.ones((1, 1)), t_eval=[np.array([0.1, 0.2, 0.3])])
    solver = batchode.BatchSolver(problem, lambda t, y: np.zeros_like(y), dt0=0.4)
    solver.step_once()
    assert len(solver._ys[0]) == 3


def test_run_equals_solve():
    rng = np.random.default_rng(3)
    mu = rng.uniform(1.0, 10.0, 40)
    f = lambda t, y: np.stack([y[:, 1], mu * (1.0 - y[:, 0] ** 2) * y[:, 1] - y[:, 0]], 1)  # noqa: E731
    problem = batchode.IvpBatch(np.tile([2.0, 0.0], (40, 1)), np.zeros(40), np.full(40, 5.0),
                                [np.linspace(0.0, 5.0, 7)] * 40)
    a = batchode.BatchSolver(problem, f).run()
    b = batchode.solve(problem, f)
    reg = batchode.solve(problem, batchode.vdp_dynamics(batchode.VdpParams(mu)))
    for s in (b, reg):
        assert np.array_equal(a.stats.n_steps, s.stats.n_steps)
        assert np.array_equal(a.stats.n_f_evals, s.stats.n_f_evals)
        assert np.array_equal(a.ys_flat, s.ys_flat)  # traced == registered, bit for bit


def test_solve_joint_with_lambda_matches_reference():
    prob = batchode.IvpBatch(y0=np.array([[1.0, 2.0], [0.5, -1.0], [2.0, 0.1]]),
                             t_start=np.zeros(3), t_end=np.ones(3),
                             t_eval=[np.array([0.5, 1.0])] * 3)
    sol = batchode.solve_joint(prob, lambda t, y: -y)
    assert np.array_equal(np.stack([np.asarray(y) for y in sol.ys]), G["joint/ys"])
    assert np.array_equal(sol.stats.n_steps, G["joint/n_steps"])
    assert np.array_equal(sol.stats.n_f_evals, G["joint/n_f_evals"])


# ---- Stepper / rk_step / interpolate with user tableaus ----
@pytest.mark.parametrize("tname", ["bs3", "ralston"])
def test_stepper_user_tableau_matches_reference(tname):
    y, dt, t = G["units/y"], G["units/dt"], G["units/t"]
    f = lambda t, y: np.sin(y) + t[:, None]  # noqa: E731
    st_ = batchode.Stepper(tableau(tname), 5, 3)
    step = st_.step(f, t, dt, y, f(t, y))
    k = f"units/{tname}/"
    for got, want in ((step.y_next, G[k + "y_next"]), (step.error_estimate, G[k + "err"]),
                      (step.stage_derivs, G[k + "k"])):
        # np.sin vs the device sin: ~1 ulp per stage evaluation
        assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want)), np.max(np.abs(got - want))
    out = st_.interpolate(step, y, dt, G[k + "theta"])
    assert np.max(np.abs(out - G[k + "interp"])) <= 1e-14


# ---- the reference's tests/test_stepper.py, with its lambdas ----
def naive_interp_weights(coeffs, theta):
    s, m = coeffs.shape
    return np.array([sum(coeffs[i, j] * theta ** (j + 1) for j in range(m)) for i in range(s)])


def test_zero_dynamics_is_identity():
    tab = batchode.dopri5()
    y = np.array([[1.5, -2.0], [0.0, 3.0]])
    t = np.zeros(2)
    dt = np.array([0.3, 0.7])
    f = lambda t, y: np.zeros_like(y)  # noqa: E731
    step = batchode.rk_step(f, tab, t, dt, y, f(t, y))
    assert np.array_equal(step.y_next, y)
    assert np.array_equal(step.error_estimate, np.zeros_like(y))


def test_constant_dynamics_quadrature():
    tab = batchode.dopri5()
    y = np.zeros((1, 1))
    f = lambda t, y: np.ones_like(y)  # noqa: E731
    step = batchode.rk_step(f, tab, np.zeros(1), np.array([0.1]), y, f(None, y))
    assert step.y_next[0, 0] == pytest.approx(0.1, rel=1e-15)


@pytest.mark.parametrize("make", [batchode.dopri5, batchode.tsit5])
def test_exponential_single_step_accuracy(make):
    y = np.ones((1, 1))
    step = batchode.rk_step(lambda t, y: y, make(), np.zeros(1), np.array([0.1]), y, y.copy())
    assert abs(step.y_next[0, 0] - np.exp(0.1)) < 1e-9


def test_fsal_last_stage_is_f_next():
    f = lambda t, y: y  # noqa: E731
    y = np.ones((1, 1))
    step = batchode.rk_step(f, batchode.dopri5(), np.zeros(1), np.array([0.1]), y, y.copy())
    assert np.array_equal(step.f_next, f(None, step.y_next))


def test_nonfinite_propagates_into_error_estimate():
    def f(t, y):
        return np.where(y > 2.0, np.inf, y * y)

    y = np.array([[1.9]])
    step = batchode.rk_step(f, batchode.dopri5(), np.zeros(1), np.array([5.0]), y, f(None, y))
    assert not np.all(np.isfinite(step.error_estimate))


def test_interpolate_endpoints_and_naive_oracle_and_extrapolation():
    tab = batchode.dopri5()
    y = np.ones((1, 1))
    dt = np.array([0.1])
    stepper = batchode.Stepper(tab, 1, 1)
    step = stepper.step(lambda t, y: y, np.zeros(1), dt, y, y.copy())
    assert np.array_equal(stepper.interpolate(step, y, dt, np.zeros(1)), y)
    at1 = stepper.interpolate(step, y, dt, np.ones(1))
    assert abs(at1[0, 0] - step.y_next[0, 0]) < 1e-12
    horner = stepper.interpolate(step, y, dt, np.array([0.5]))
    w = naive_interp_weights(tab.interp_coeffs, 0.5)
    naive = y[0, 0] + dt[0] * sum(w[i] * step.stage_derivs[i, 0, 0] for i in range(7))
    assert abs(horner[0, 0] - naive) < 1e-13
    for bad in (1.5, -0.1):
        with pytest.raises(ValueError):
            stepper.interpolate(step, y, dt, np.array([bad]))


@given(coeffs=st.lists(st.lists(st.floats(-5, 5), min_size=4, max_size=4), min_size=7,
                       max_size=7),
       theta=st.floats(0.0, 1.0))
@settings(max_examples=50, deadline=None)
def test_horner_matches_power_form(coeffs, theta):
    coeffs = np.array(coeffs)
    tab = batchode.dopri5()
    object.__setattr__(tab, "interp_coeffs", coeffs)  # now a user tableau
    stepper = batchode.Stepper(tab, 1, 1)
    step = stepper.step(lambda t, y: y, np.zeros(1), np.array([0.1]), np.ones((1, 1)),
                        np.ones((1, 1)))
    horner = stepper.interpolate(step, np.ones((1, 1)), np.array([0.1]), np.array([theta]))
    w = naive_interp_weights(coeffs, theta)
    naive = 1.0 + 0.1 * sum(w[i] * step.stage_derivs[i, 0, 0] for i in range(7))
    assert horner[0, 0] == pytest.approx(naive, rel=1e-12, abs=1e-12)


def test_rk_step_batch_rows_match_single_rows():
    tab = batchode.dopri5()
    rng = np.random.default_rng(7)
    y = rng.normal(size=(5, 3))
    dt = rng.uniform(0.01, 0.2, size=5)
    t = rng.uniform(0, 1, size=5)
    f = lambda t, y: np.sin(y) + t[:, None]  # noqa: E731
    batch = batchode.rk_step(f, tab, t, dt, y, f(t, y))
    for i in range(5):
        single = batchode.rk_step(f, tab, t[i:i + 1], dt[i:i + 1], y[i:i + 1],
                                  f(t[i:i + 1], y[i:i + 1]))
        assert np.array_equal(batch.y_next[i], single.y_next[0])
        assert np.array_equal(batch.error_estimate[i], single.error_estimate[0])


def test_fsal_counting_formula_over_full_solve():
    problem = batchode.IvpBatch(y0=np.array([[1.0, 0.0]]), t_start=np.array([0.0]),
                                t_end=np.array([10.0]), t_eval=[np.empty(0)])

    def f(t, y):
        return np.stack([y[:, 1], -y[:, 0] - 0.1 * y[:, 1] * np.abs(y[:, 1])], axis=1)

    sol = batchode.solve(problem, f, tol=batchode.Tolerances(1e-9, 1e-9))
    a = sol.stats.n_accepted[0]
    r = sol.stats.n_steps[0] - a
    assert sol.stats.n_f_evals[0] == 1 + 6 * a + 7 * r


def test_solve_device_with_traced_dynamics_fast_mode():
    import torch
    rng = np.random.default_rng(9)
    n = 4096
    mu = rng.uniform(1.0, 10.0, n)
    f = lambda t, y: np.stack([y[:, 1], mu * (1.0 - y[:, 0] * y[:, 0]) * y[:, 1] - y[:, 0]], 1)  # noqa: E731
    f64 = dict(dtype=torch.float64, device="cuda")
    kw = dict(t_eval=torch.full((n, 1), 8.0, **f64), controller=batchode.pid_controller("PI42"),
              mode="fast")
    y0 = torch.tensor(np.tile([2.0, 0.0], (n, 1)), **f64)
    a = batchode.solve_device(y0, 0.0, 8.0, f, **kw)
    b = batchode.solve_device(y0, 0.0, 8.0,
                              batchode.vdp_dynamics(batchode.VdpParams(torch.tensor(mu, **f64))),
                              **kw)
    # the registered functor fuses its multiply-adds in fast mode, the traced
    # one keeps NumPy's separate roundings: the same steps up to ulp effects
    same = float((a["n_steps"] == b["n_steps"]).double().mean())
    assert same >= 0.99, same
    assert abs(int(a["n_steps"].sum()) / int(b["n_steps"].sum()) - 1.0) < 1e-4
    scale = b["ys"].abs().max()
    assert float((a["ys"] - b["ys"]).abs().max() / scale) <= 1e-8


def test_registered_functors_are_callable_like_the_reference():
    # problems.py:41-50 returns a callable; tests/test_problems.py calls it
    f = batchode.vdp_dynamics(batchode.VdpParams(mu=np.array([0.0, 3.0])))
    y = np.array([[1.5, -0.5], [0.3, 2.0]])
    out = f(np.zeros(2), y)
    mu = np.array([0.0, 3.0])
    want = np.stack([y[:, 1], mu * (1.0 - y[:, 0] * y[:, 0]) * y[:, 1] - y[:, 0]], axis=1)
    assert np.array_equal(out, want)
