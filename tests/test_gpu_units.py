"""Device unit ops (bode_rk_step / bode_interpolate / bode_error_norm /
bode_adapt_step / bode_initial_step through the C ABI) against the
reference's golden unit vectors (tests/golden/units.npz) and the reference's
own unit-test known answers (tests/test_stepper.py, test_controller.py)."""
import numpy as np
import pytest

import paper_2210_12375_b200 as bode
from paper_2210_12375_b200 import units as U
import golden_io as G
import scenarios as S
import devspec

pytestmark = pytest.mark.gpu
UNITS = np.load(G.os.path.join(G.GOLDEN, "units.npz"))


def _u(prefix):
    return {k[len(prefix):]: UNITS[k] for k in UNITS.files if k.startswith(prefix)}


def _dyn(dname, u):
    if dname == "vdp":
        return bode.vdp_dynamics(bode.VdpParams(u["mu"]))
    if dname == "lorenz":
        return bode.lorenz_dynamics()
    if dname == "zero":
        return bode.zero_dynamics()
    if dname == "square":
        return bode.square_dynamics(0.4)
    return bode.sin_plus_t_dynamics()


@pytest.mark.parametrize("method", ["dopri5", "tsit5", "heun"])
@pytest.mark.parametrize("dname", ["vdp", "lorenz", "sin_plus_t"])
def test_rk_step_and_interpolate_vs_golden(method, dname):
    u = _u(f"rk_{method}_{dname}_")
    tab = devspec.tableau(method)
    st = U.rk_step(_dyn(dname, u), tab, u["t"], u["dt"], u["y"], u["f0"])
    exact = dname != "sin_plus_t"  # CUDA sin differs from libm by <= 1 ulp
    cmp = np.array_equal if exact else (lambda a, b: np.allclose(a, b, rtol=1e-14, atol=1e-15))
    assert cmp(st.y_next, u["ynext"])
    assert cmp(st.stage_derivs, u["k"])
    if exact:  # no transcendental on this path: bit-identical to the reference
        assert np.array_equal(st.error_estimate, u["err"])
    else:
        np.testing.assert_allclose(st.error_estimate, u["err"], rtol=1e-9, atol=1e-17)
    yi = U.interpolate(st, tab, u["y"], u["dt"], u["theta"])
    assert cmp(yi, u["interp"])


@pytest.mark.parametrize("d", [1, 2, 3, 4, 7, 8, 9, 16, 64, 130, 300])
def test_error_norm_vs_golden_bit_exact(d):
    u = _u(f"norm_d{d}_")
    a = U.error_norm(u["err"], u["y0"], u["y1"], bode.Tolerances(1e-6, 1e-7))
    assert np.array_equal(a, u["scalar"])
    b = U.error_norm(u["err"], u["y0"], u["y1"], bode.Tolerances(u["atol"], u["rtol"]))
    assert np.array_equal(b, u["vector"])


@pytest.mark.parametrize("cname,betas,hist", [
    ("I", S.ICTRL, True), ("PI42", S.PI42, True), ("H312", S.H312, True),
    ("H312n", S.H312, False), ("H211", (1 / 6, 1 / 6, 0.0), True)])
def test_adapt_step_vs_golden(cname, betas, hist):
    p = f"adapt_{cname}_"
    norms = UNITS[p + "norms"]
    coeffs = bode.PidCoefficients(beta1=betas[0], beta2=betas[1], beta3=betas[2],
                                  update_history_on_reject=hist)
    state = U.ControllerState.initial(UNITS[p + "dt0"])
    for j in range(norms.shape[0]):
        acc, dtn = U.adapt_step(state, norms[j], 4, coeffs)
        assert np.array_equal(acc, UNITS[p + "accept"][j])
        np.testing.assert_allclose(dtn, UNITS[p + "dt"][j], rtol=1e-13)
        np.testing.assert_allclose(state.norm_prev, UNITS[p + "prev"][j], rtol=1e-13)
        # pow is the only non-IEEE op: CUDA pow vs glibc pow differ by <= 1 ulp
        np.testing.assert_allclose(state.norm_prev2, UNITS[p + "prev2"][j], rtol=1e-13)


@pytest.mark.parametrize("dname", ["vdp", "lorenz", "zero", "square"])
def test_initial_step_vs_golden(dname):
    p = f"init_{dname}_"
    u = _u(p)
    dt, f0 = U.initial_step(_dyn(dname, u), u["t0"], u["y0"], int(u["order"]),
                            bode.Tolerances(u["atol"], u["rtol"]), u["dir"])
    np.testing.assert_allclose(dt, u["dt"], rtol=1e-14)
    assert np.array_equal(np.isnan(dt), np.isnan(u["dt"]))
    assert np.array_equal(f0, u["f0"])


# ---- known answers from the reference's own unit tests ----------------
def test_zero_dynamics_is_identity():  # tests/test_stepper.py:17-25
    y = np.array([[1.5, -2.0], [0.0, 3.0]])
    st = U.rk_step(bode.zero_dynamics(), bode.dopri5(), np.zeros(2), np.array([0.3, 0.7]), y,
                   np.zeros_like(y))
    assert np.array_equal(st.y_next, y)
    assert np.array_equal(st.error_estimate, np.zeros_like(y))


def test_constant_dynamics_quadrature():  # tests/test_stepper.py:28-34
    st = U.rk_step(bode.constant_dynamics(1.0), bode.dopri5(), np.zeros(1), np.array([0.1]),
                   np.zeros((1, 1)), np.ones((1, 1)))
    assert st.y_next[0, 0] == pytest.approx(0.1, rel=1e-15)


@pytest.mark.parametrize("tab", [bode.dopri5, bode.tsit5])
def test_exponential_single_step_accuracy(tab):  # tests/test_stepper.py:37-43
    st = U.rk_step(bode.linear_dynamics(1.0), tab(), np.zeros(1), np.array([0.1]),
                   np.ones((1, 1)), np.ones((1, 1)))
    assert abs(st.y_next[0, 0] - np.exp(0.1)) < 1e-9


def test_fsal_last_stage_is_f_next():  # tests/test_stepper.py:61-66
    st = U.rk_step(bode.linear_dynamics(1.0), bode.dopri5(), np.zeros(1), np.array([0.1]),
                   np.ones((1, 1)), np.ones((1, 1)))
    assert np.array_equal(st.f_next, st.y_next)
    assert st.n_evals == 6


def test_nonfinite_propagates_into_error_estimate():  # tests/test_stepper.py:69-77
    y = np.array([[1.9]])
    st = U.rk_step(bode.square_dynamics(2.0), bode.dopri5(), np.zeros(1), np.array([5.0]), y,
                   y * y)
    assert not np.all(np.isfinite(st.error_estimate))


def test_interpolate_endpoints_and_extrapolation():  # tests/test_stepper.py:80-117
    y = np.ones((1, 1))
    dt = np.array([0.1])
    st = U.rk_step(bode.linear_dynamics(1.0), bode.dopri5(), np.zeros(1), dt, y, y.copy())
    assert np.array_equal(U.interpolate(st, bode.dopri5(), y, dt, np.zeros(1)), y)
    at1 = U.interpolate(st, bode.dopri5(), y, dt, np.ones(1))
    assert abs(at1[0, 0] - st.y_next[0, 0]) < 1e-12
    for bad in (1.5, -0.1):
        with pytest.raises(ValueError):
            U.interpolate(st, bode.dopri5(), y, dt, np.array([bad]))


def test_batch_rows_match_single_rows():  # tests/test_stepper.py:140-153
    rng = np.random.default_rng(7)
    y = rng.normal(size=(5, 3))
    dt = rng.uniform(0.01, 0.2, size=5)
    t = rng.uniform(0, 1, size=5)
    f = bode.sin_plus_t_dynamics()
    f0 = np.sin(y) + t[:, None]
    batch = U.rk_step(f, bode.dopri5(), t, dt, y, f0)
    for i in range(5):
        single = U.rk_step(f, bode.dopri5(), t[i:i + 1], dt[i:i + 1], y[i:i + 1], f0[i:i + 1])
        assert np.array_equal(batch.y_next[i], single.y_next[0])
        assert np.array_equal(batch.error_estimate[i], single.error_estimate[0])


def test_error_norm_known_answers():  # tests/test_controller.py:61-97
    assert np.array_equal(U.error_norm(np.zeros((3, 2)), np.ones((3, 2)), np.ones((3, 2)),
                                       bode.Tolerances(1e-6, 1e-6)), np.zeros(3))
    y = np.random.default_rng(0).normal(size=(2, 4))
    n = U.error_norm(np.full((2, 4), 1e-5), y, y, bode.Tolerances(1e-5, 0.0))
    assert n == pytest.approx([1.0, 1.0], rel=1e-14)
    n = U.error_norm(np.array([[1e-9, np.nan], [1e-9, 1e-9]]), np.ones((2, 2)), np.ones((2, 2)),
                     bode.Tolerances(1e-6, 1e-6))
    assert n[0] == np.inf and np.isfinite(n[1])


def test_adapt_step_known_answers():  # tests/test_controller.py:156-196
    st = U.ControllerState.initial(np.array([0.1]))
    acc, dtn = U.adapt_step(st, np.ones(1), 4, bode.integral_controller(0.9))
    assert acc[0] and dtn[0] == pytest.approx(0.09, rel=1e-15)
    st = U.ControllerState.initial(np.array([0.1]))
    acc, dtn = U.adapt_step(st, np.zeros(1), 4, bode.integral_controller())
    assert dtn[0] == pytest.approx(1.0)
    st = U.ControllerState.initial(np.array([0.1]))
    acc, dtn = U.adapt_step(st, np.array([4.0]), 4, bode.integral_controller())
    assert not acc[0] and dtn[0] == pytest.approx(0.1 * 0.9 * 4 ** (-0.2), rel=1e-15)
    assert st.norm_prev[0] == 4.0 and st.norm_prev2[0] == 1.0
    st = U.ControllerState.initial(np.array([0.1]))
    U.adapt_step(st, np.array([4.0]), 4, bode.PidCoefficients(update_history_on_reject=False))
    assert st.norm_prev[0] == 1.0
    st = U.ControllerState.initial(np.array([0.1]))
    acc, dtn = U.adapt_step(st, np.array([np.inf]), 4, bode.integral_controller())
    assert not acc[0] and dtn[0] == pytest.approx(0.02)


def test_initial_step_known_answers():  # tests/test_controller.py:113-153
    dt, _ = U.initial_step(bode.zero_dynamics(), np.zeros(1), np.ones((1, 1)), 5,
                           bode.Tolerances(1e-5, 1e-5))
    assert dt[0] > 0 and np.isfinite(dt[0])
    dt, _ = U.initial_step(bode.linear_dynamics(1.0), np.zeros(1), np.ones((1, 1)), 5,
                           bode.Tolerances(1e-5, 1e-5))
    d1, h0 = 1.0 / 2e-5, 0.01
    d2 = (h0 / 2e-5) / h0
    assert dt[0] == pytest.approx(min(100 * h0, (0.01 / max(d1, d2)) ** (1 / 6)), rel=1e-12)
    dt, _ = U.initial_step(bode.linear_dynamics(1.0), np.zeros(1), np.ones((1, 1)), 5,
                           bode.Tolerances(1e-5, 1e-5), direction=-1.0)
    assert dt[0] < 0
    dt, _ = U.initial_step(bode.square_dynamics(-1.0), np.zeros(1), np.ones((1, 1)), 5,
                           bode.Tolerances(1e-5, 1e-5))
    assert np.isnan(dt[0])
