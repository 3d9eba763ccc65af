"""Host-side API (no GPU): validation mirrors the reference's ValueErrors,
the C-ABI library loads and exports every symbol include/bode.h declares,
and the binding's struct layout matches the compiled one."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2210_12375_b200 as bode
from paper_2210_12375_b200 import _abi
from paper_2210_12375_b200.tableau import method_of

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "bode.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(bode_\w+)\(", src, re.M)))


def test_library_exports_every_header_symbol():
    lib = _abi.load()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _abi.SIGNATURES, f"binding lacks {s}"
    assert lib.bode_abi_version() == _abi.ABI_VERSION
    assert lib.bode_sizeof_args() == C.sizeof(_abi.SolveArgs)
    assert C.sizeof(O.Args) == C.sizeof(_abi.SolveArgs)


def test_workspace_size_and_einval_without_gpu():
    lib = _abi.load()
    a = _abi.SolveArgs()
    a.abi_version = _abi.ABI_VERSION
    assert lib.bode_workspace_size(C.byref(a)) == 0  # n = 0 is invalid
    assert "instance" in lib.bode_last_error().decode()
    with pytest.raises(ValueError):
        _abi.check(lib.bode_solve(C.byref(a)))


def test_ivpbatch_validation():  # reference tests/test_solver.py:24-40
    with pytest.raises(ValueError):
        bode.IvpBatch(np.ones((1, 1)), np.zeros(1), np.zeros(1), [np.empty(0)])
    with pytest.raises(ValueError):
        bode.IvpBatch(np.ones((1, 1)), np.zeros(1), np.ones(1), [np.array([0.5, 0.2])])
    with pytest.raises(ValueError):
        bode.IvpBatch(np.ones((1, 1)), np.zeros(1), np.ones(1), [np.array([0.5, 2.0])])
    with pytest.raises(ValueError):
        bode.IvpBatch(np.ones((2, 1)), np.zeros(2), np.ones(2), [np.empty(0)])
    with pytest.raises(ValueError):  # vectorised 2-D form, same rules
        bode.IvpBatch(np.ones((2, 1)), np.zeros(2), np.ones(2), np.array([[0.1, 0.2], [0.3, 1.5]]))
    with pytest.raises(ValueError):
        bode.IvpBatch(np.ones((2, 1)), np.zeros(2), np.ones(2), np.array([0.5, 0.2]))
    p = bode.IvpBatch(np.ones((2, 1)), np.ones(2), np.zeros(2), np.array([[0.9, 0.1], [1.0, 0.0]]))
    assert p.t_eval[1].tolist() == [1.0, 0.0]


def test_config_validation():  # reference tests/test_controller.py:31-58
    with pytest.raises(ValueError):
        bode.Tolerances(atol=-1.0, rtol=1e-6)
    with pytest.raises(ValueError):
        bode.Tolerances(atol=0.0, rtol=0.0)
    with pytest.raises(ValueError):
        bode.PidCoefficients(safety=0.0)
    with pytest.raises(ValueError):
        bode.PidCoefficients(factor_min=1.5)
    for name in ("PI42", "PI33", "PI34", "H211", "H312"):
        bode.pid_controller(name)
    with pytest.raises(ValueError):
        bode.pid_controller("nope")
    with pytest.raises(ValueError):
        bode.VdpParams(-1.0)


def test_tableaus_validate_and_custom_resolution():
    for tab in (bode.dopri5(), bode.tsit5(), bode.heun()):
        tab.validate()
        assert method_of(tab) == tab.method
    t = bode.dopri5()
    # the same coefficients on any object (e.g. a reference-built tableau) are the built-in pair
    clone = bode.ButcherTableau(stages=7, a=t.a.copy(), b=t.b.copy(), b_err=t.b_err.copy(),
                                c=t.c.copy(), order=5, error_order=4,
                                interp_coeffs=t.interp_coeffs.copy(), fsal=True)
    assert method_of(clone) == "dopri5"
    custom = bode.ButcherTableau(stages=t.stages, a=t.a, b=t.b, b_err=t.b_err * 2, c=t.c,
                                 order=5, error_order=4, interp_coeffs=t.interp_coeffs, fsal=True)
    assert method_of(custom) is custom  # runs through a run-time program
    with pytest.raises(TypeError):
        method_of(object())


def test_dynamics_packing_and_untraceable_callables():
    f = bode.forced_linear_dynamics(np.array([1.0, 2.0]), 0.5, 3.0)
    shared, mask, cols = f.pack(2)
    assert mask == 0b001 and shared[1] == 0.5 and shared[2] == 3.0
    assert np.array_equal(cols[0], [1.0, 2.0])
    with pytest.raises(ValueError):
        f.pack(3)
    with pytest.raises(ValueError):
        bode.vdp_dynamics(bode.VdpParams(2.0)).check_width(3)

    def branchy(t, y):  # Python control flow on state values cannot be traced
        return y if y[0, 0] > 0 else -y

    with pytest.raises(NotImplementedError):
        bode.solve(bode.IvpBatch(np.ones((1, 1)), [0.0], [1.0], [np.empty(0)]), branchy)
    # a registered functor is callable like the reference's dynamics, but it
    # is evaluated on the device: no CUDA device here -> no CPU fallback
    with pytest.raises(bode._abi.BodeLibraryError):
        bode.vdp_dynamics(bode.VdpParams(2.0))(np.zeros(1), np.ones((1, 2)))


def test_solve_joint_validation_matches_reference():
    """solve_joint raises the reference's ValueErrors (solver.py:391-403)
    before touching the device."""
    import paper_2210_12375_b200 as bode
    f = bode.vdp_dynamics(bode.VdpParams(np.array([1.0, 2.0])))
    y0 = np.tile([2.0, 0.0], (2, 1))
    with pytest.raises(ValueError, match="identical integration bounds"):
        bode.solve_joint(bode.IvpBatch(y0, np.zeros(2), np.array([1.0, 2.0]),
                                       [np.empty(0)] * 2), f)
    with pytest.raises(ValueError, match="identical evaluation points"):
        bode.solve_joint(bode.IvpBatch(y0, np.zeros(2), np.ones(2),
                                       [np.array([0.5]), np.array([0.6])]), f)
    with pytest.raises(ValueError, match="scalar tolerances"):
        bode.solve_joint(bode.IvpBatch(y0, np.zeros(2), np.ones(2), [np.empty(0)] * 2), f,
                         tol=bode.Tolerances(np.array([1e-6, 1e-6]), 1e-6))


def test_cli_parser_mirrors_reference_flags():
    """Flag validation of the experiment CLI (reference cli.py:242-288) runs
    before any solve: bad values exit with argparse's code 2."""
    from paper_2210_12375_b200 import cli
    p = cli.build_parser()
    a = p.parse_args(["vdp-batching", "--out", "x.csv"])
    assert (a.n, a.mu, a.mode, a.method, a.n_eval, a.max_steps) == (4, 25.0, "independent",
                                                                     "dopri5", 200, 100_000)
    for bad in (["vdp-batching", "--n", "0", "--out", "x"],
                ["vdp-batching", "--controller", "pid:nope", "--out", "x"],
                ["looptime", "--steps", "-1", "--out", "x"]):
        with pytest.raises(SystemExit) as e:
            p.parse_args(bad)
        assert e.value.code == 2
    assert cli.main(["pid-sweep", "--presets", "nope", "--out", "/dev/null"]) == 2


def _valid_args(kind="vdp", d=2, hidden=0):
    a = _abi.SolveArgs()
    a.abi_version = _abi.ABI_VERSION
    a.n, a.d = 4, d
    a.dyn.kind = _abi.DYN[kind]
    a.dyn.hidden = hidden
    if kind == "mlp":  # fake non-null pointers: validation never dereferences them
        a.dyn.W1 = a.dyn.b1 = a.dyn.W2 = a.dyn.b2 = 0x1000
    a.ctrl.beta1, a.ctrl.safety, a.ctrl.factor_min, a.ctrl.factor_max = 1.0, 0.9, 0.2, 10.0
    a.max_steps = 10
    a.atol = a.rtol = 1e-6
    a.y0 = a.t_start = a.t_end = 0x1000
    a.n_emitted = a.n_steps = a.n_accepted = a.final_dt = a.status = a.n_f_evals = 0x1000
    return a


def test_adjoint_abi_validation_without_gpu():
    """bode_solve_adjoint / trajectory recording reject what they do not
    support before touching the device (BODE_EINVAL / BODE_EUNSUPPORTED)."""
    lib = _abi.load()
    a = _valid_args()
    assert lib.bode_adjoint_workspace_size(C.byref(a)) > 0
    g = _abi.AdjointArgs()
    with pytest.raises(ValueError, match="traj"):  # no trajectory
        _abi.check(lib.bode_solve_adjoint(C.byref(a), C.byref(g)))
    g.traj = g.traj_offsets = g.n_emitted = g.grad_y0 = 0x1000
    with pytest.raises(ValueError, match="workspace"):
        _abi.check(lib.bode_solve_adjoint(C.byref(a), C.byref(g)))
    a.joint = 1
    with pytest.raises(NotImplementedError):
        _abi.check(lib.bode_solve_adjoint(C.byref(a), C.byref(g)))
    # one MLP path: the 64-wide tensor-core tile (the facade zero-pads
    # narrower networks, dynamics.mlp_pad); anything else is unsupported
    for d, hidden in ((6, 32), (64, 40), (64, 288)):
        m = _valid_args("mlp", d=d, hidden=hidden)
        with pytest.raises(NotImplementedError, match="MLP dynamics"):
            _abi.check(lib.bode_solve(C.byref(m)))
        with pytest.raises(NotImplementedError, match="MLP dynamics"):
            _abi.check(lib.bode_solve_adjoint(C.byref(m), C.byref(g)))
    m = _valid_args("mlp", d=64, hidden=64)  # gradients need the recorded stage inputs
    with pytest.raises(ValueError, match="traj_stages"):
        _abi.check(lib.bode_solve_adjoint(C.byref(m), C.byref(g)))
    r = _valid_args()
    r.traj = 0x1000  # recording without offsets
    with pytest.raises(ValueError, match="traj_offsets"):
        _abi.check(lib.bode_solve(C.byref(r)))
    assert _abi.traj_stride(2) == 8 and _abi.traj_stride(64) == 68 and _abi.traj_stride(1) == 4


def test_adjoint_oracle_tableau_matches_product_tableau():
    """The gradient oracle's coefficients (parsed from the generated header)
    equal the facade's ButcherTableau data (pinned to the reference)."""
    import adjoint_oracle as AO

    for name, tab in (("dopri5", bode.dopri5()), ("tsit5", bode.tsit5()), ("heun", bode.heun())):
        T = AO.tableau(name)
        S = T["S"]
        assert np.array_equal(T["a"], np.asarray(tab.a)[:S, :S])
        assert np.array_equal(T["b"], np.asarray(tab.b)[:S])
        assert np.array_equal(T["c"], np.asarray(tab.c)[:S])


def test_solve_multi_validates_before_touching_the_gpu():
    """bode_solve_multi rejects an empty shard list with
    BODE_EINVAL and a message, without a device."""
    from paper_2210_12375_b200 import _abi
    lib = _abi.load()
    assert lib.bode_solve_multi(None, 0, None) == _abi.EINVAL
    assert b"at least one shard" in lib.bode_last_error()
