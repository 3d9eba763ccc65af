"""solve_joint (reference solver.py:372-427) on the GPU vs fixtures produced
by the reference's own batchode.solve_joint (tests/golden/make_golden.py
joint): the batch as one problem of size n*d -- one error norm (NumPy's
pairwise order over the flattened row, multi-leaf for n*d > 128), one step
size and accept decision, statistics replicated per instance."""
import glob
import os

import numpy as np
import pytest

import paper_2210_12375_b200 as bode

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "joint")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz")))
YS_TOL = 1e-10
DT_TOL = 1e-5


def dynamics(g):
    name = str(g["dyn_name"])
    inst = g["dyn_inst"]
    shared = tuple(float(x) for x in g["dyn_shared"])
    if name == "vdp":
        return bode.vdp_dynamics(bode.VdpParams(inst[:, 0]))
    if name == "lorenz":
        return bode.lorenz_dynamics(*shared)
    if name == "linear":
        return bode.linear_dynamics(shared[0])
    if name == "harmonic":
        return bode.harmonic_dynamics()
    if name == "square":
        return bode.square_dynamics(shared[0])
    raise KeyError(name)


def run(name, mode="exact"):
    g = np.load(os.path.join(HERE, name + ".npz"))
    n = g["y0"].shape[0]
    te = g["te"]
    prob = bode.IvpBatch(g["y0"], g["t_start"], g["t_end"], [te] * n)
    tab = {"dopri5": bode.dopri5, "tsit5": bode.tsit5, "heun": bode.heun}[str(g["method"])]()
    b = g["betas"]
    ctrl = bode.PidCoefficients(b[0], b[1], b[2], update_history_on_reject=bool(g["hist"]))
    dt0 = None if np.isnan(g["dt0"]) else float(g["dt0"])
    sol = bode.solve_joint(prob, dynamics(g), tableau=tab,
                           tol=bode.Tolerances(float(g["atol"]), float(g["rtol"])),
                           controller=ctrl, max_steps=int(g["max_steps"]), dt0=dt0,
                           record_trace=bool(g["trace"]), mode=mode)
    return g, sol


@pytest.mark.parametrize("name", CASES)
def test_joint_matches_reference(name):
    g, sol = run(name)
    n = g["y0"].shape[0]
    assert np.array_equal(sol.status, g["status"])
    assert np.array_equal(sol.stats.n_steps, g["n_steps"])
    assert np.array_equal(sol.stats.n_accepted, g["n_accepted"])
    assert np.all(sol.stats.n_f_evals == g["n_f_evals"][0])
    assert np.array_equal(sol.n_emitted, g["n_emitted"])
    np.testing.assert_allclose(sol.stats.final_dt, g["final_dt"], rtol=DT_TOL, atol=0)
    for i in range(n):
        m = g["n_emitted"][i]
        if m == 0:
            continue
        ref = g["ys"][i, :m]
        err = np.max(np.abs(sol.ys[i] - ref)) / max(np.max(np.abs(ref)), 1e-300)
        assert err <= YS_TOL, (i, err)
    if bool(g["trace"]):
        assert np.array_equal(sol.stats.extra["trace_accept"][0], g["trace_accept"])
        np.testing.assert_allclose(sol.stats.extra["trace_dt"][0], g["trace_dt"], rtol=DT_TOL)


def test_joint_pathology_step_ratio():
    """The paper's §4.1 pathology (reference acceptance criterion 3): the
    joint solve needs far more steps than the slowest independent instance."""
    g, sol = run("joint_pathology_vdp4_mu25")
    ratio = sol.stats.n_steps[0] / g["independent_n_steps"].max()
    assert ratio >= 1.3, ratio


def test_joint_single_instance_equals_independent():
    g, sol = run("joint_single_linear")
    prob = bode.IvpBatch(g["y0"], g["t_start"], g["t_end"], [g["te"]])
    ind = bode.solve(prob, bode.linear_dynamics(-1.0))
    assert np.array_equal(ind.ys[0], sol.ys[0])
    assert ind.stats.n_steps[0] == sol.stats.n_steps[0]


@pytest.mark.parametrize("name", ["joint_vdp32_I", "joint_vdp300_wide"])
def test_joint_fast_mode(name):
    g, sol = run(name, mode="fast")
    assert np.array_equal(sol.status, g["status"])
    assert np.array_equal(sol.stats.n_steps, g["n_steps"])
