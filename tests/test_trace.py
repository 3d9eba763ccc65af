"""CPU tests of the plugin-surface compiler: NumPy callables traced into
device functors (paper_2210_12375_b200/trace.py) and user tableaus rendered
as compile-time coefficient tables (program.py), compiled with NVRTC for
sm_100a by libbode (bode_program_check: no GPU needed)."""
import ctypes as C

import numpy as np
import pytest

import paper_2210_12375_b200 as bode
from paper_2210_12375_b200 import _abi, program, trace
from paper_2210_12375_b200.dynamics import as_device_dynamics


def _compile(method, dyn, d, kernels=program.SOLVE | program.STEP | program.UNITS):
    lib = _abi.load()
    custom = not isinstance(method, str)
    src = (program.tableau_source(method) if custom else "") + program.dynamics_source(dyn, d)
    desc = _abi.ProgramDesc()
    desc.method = _abi.METHOD_CUSTOM if custom else _abi.METHOD[method]
    desc.kernels, desc.d = kernels, d
    desc.n_params = getattr(dyn, "n_params", 0) if getattr(dyn, "kind", "") == "program" else 0
    tab = method if custom else {"dopri5": bode.dopri5, "tsit5": bode.tsit5,
                                 "heun": bode.heun}[method]()
    desc.stages, desc.order, desc.error_order = tab.stages, tab.order, tab.error_order
    desc.fsal = int(bool(tab.fsal))
    rc = lib.bode_program_check(src.encode(), C.byref(desc))
    assert rc == 0, lib.bode_last_error().decode()


def test_trace_row_template_and_params():
    n = 5
    mu = np.linspace(1.0, 2.0, n)
    A = np.array([[0.0, 1.0], [-1.0, 0.0]])

    def f(t, y):
        x, v = y[:, 0], y[:, 1]
        out = np.empty_like(y)
        out[:, 0] = v + (y @ A.T)[:, 0] * 0.0
        out[:, 1] = np.where(x > 1.0, mu * (1.0 - x * x) * v - x, np.cos(t) ** 2)
        return out

    tf = trace.trace_dynamics(f, n, 2)
    assert tf.params.shape == (n, 1) and np.array_equal(tf.params[:, 0], mu)
    for frag in ("__dmul_rn", "__dsub_rn", "cos(t)", "p[0]", "y[1]", "f[0] =", "f[1] ="):
        assert frag in tf.source, frag
    # a (d,) array broadcasts along the state axis: constants, not parameters
    tf2 = trace.trace_dynamics(lambda t, y: y * np.array([2.0, 3.0]), 2, 2)
    assert tf2.params is None and float(3.0).hex() in tf2.source


def test_numpy_power_and_reduction_semantics():
    tf = trace.trace_dynamics(lambda t, y: y ** 2 + y ** 0.5 + y.sum(axis=1, keepdims=True), 3, 2)
    src = tf.source
    assert "__dsqrt_rn(y[" in src and "user_pow(y" not in src  # fast_scalar_power short cuts
    assert src.count("__dadd_rn(0.0,") == 1  # NumPy's pairwise sum seeds 0.0 below 8 terms


@pytest.mark.parametrize("bad", [
    lambda t, y: y if y[0, 0] > 0 else -y,          # Python control flow on values
    lambda t, y: y[0:1] * np.ones((3, 1)),          # indexing across instances
    lambda t, y: y - y.sum(axis=0),                 # reduction over the batch
    lambda t, y: np.array([y[:, 0], y[:, 1]]).T,    # conversion to a concrete array
])
def test_untraceable_callables_raise_not_implemented(bad):
    with pytest.raises(NotImplementedError):
        trace.trace_dynamics(bad, 3, 2)


def test_traced_and_registered_functors_compile_for_sm100a():
    lam = -np.linspace(0.5, 2.0, 4)
    dyn = as_device_dynamics(lambda t, y: lam[:, None] * y + np.sin(3.0 * t)[:, None], 4, 1)
    _compile("dopri5", dyn, 1)
    _compile("tsit5", as_device_dynamics(lambda t, y: np.stack(
        [y[:, 1], -y[:, 0] - 0.1 * y[:, 1] * np.abs(y[:, 1])], axis=1), 4, 2), 2,
        kernels=program.SOLVE | program.JOINT)
    _compile("heun", bode.linear_dynamics(-1.0), 6)  # registered functor beyond the compiled widths


def test_user_tableau_compiles_and_sources_its_coefficients():
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import dropin_cases as DC
    bs3 = bode.ButcherTableau(**DC.bs3_data())
    bs3.validate()
    src = program.tableau_source(bs3)
    assert "S = 4, ORDER = 3, ERR_ORDER = 2, NI = 3" in src and "FSAL = true" in src
    assert float(0.5).hex() in src  # a[1][0]
    _compile(bs3, as_device_dynamics(lambda t, y: -y, 2, 2), 2)
    ral = bode.ButcherTableau(**DC.ralston_data())
    _compile(ral, bode.vdp_dynamics(bode.VdpParams(2.0)), 2, kernels=program.SOLVE)
