"""torchode-style API (ODETerm / InitialValueProblem / Dopri5 / Tsit5 / Heun /
IntegralController / PIDController / AutoDiffAdjoint.solve) on device
tensors, checked against the reference golden vectors, plus the sharded
solve driver on one rank with the real GPU solver."""
import numpy as np
import pytest

import golden_io as G
import paper_2210_12375_b200 as bode
import paper_2210_12375_b200.torchode as to
from paper_2210_12375_b200 import distributed as D

pytestmark = pytest.mark.gpu


def test_torchode_api_c1_matches_reference():
    import torch

    g = G.load("c1_vdp")
    sc = G.scenario_map()["c1_vdp"]
    n = len(g["status"])
    dev = "cuda"
    mu = torch.tensor(sc["dyn"]["inst"][:, 0], device=dev)
    term = to.ODETerm(bode.vdp_dynamics(bode.VdpParams(mu)))
    te = torch.linspace(0.0, 10.0, 50, dtype=torch.float64, device=dev)
    ivp = to.InitialValueProblem(y0=torch.tensor(sc["y0"], device=dev), t_eval=te)
    solver = to.AutoDiffAdjoint(to.Dopri5(term=term), to.IntegralController(1e-6, 1e-6, term=term),
                                max_steps=100_000)
    sol = solver.solve(ivp)
    assert sol.ys.shape == (n, 50, 2)
    assert torch.equal(sol.status.cpu(), torch.tensor(g["status"]))
    assert np.array_equal(sol.stats["n_steps"].cpu().numpy(), g["n_steps"])
    assert np.array_equal(sol.stats["n_accepted"].cpu().numpy(), g["n_accepted"])
    assert np.all(sol.stats["n_f_evals"].cpu().numpy() == g["n_f_evals"][0])
    ref = g["ys"].reshape(n, 50, 2)
    err = np.max(np.abs(sol.ys.cpu().numpy() - ref) / np.abs(ref).max(axis=(1, 2), keepdims=True))
    assert err <= 1e-10


def test_torchode_pid_presets_and_heun():
    import torch

    g = G.load("heun_vdp")
    sc = G.scenario_map()["heun_vdp"]
    mu = torch.tensor(sc["dyn"]["inst"][:, 0], device="cuda")
    term = to.ODETerm(bode.vdp_dynamics(bode.VdpParams(mu)))
    te = torch.linspace(0.0, 10.0, 25, dtype=torch.float64, device="cuda")
    ivp = to.InitialValueProblem(y0=torch.tensor(sc["y0"], device="cuda"), t_eval=te)
    sol = to.AutoDiffAdjoint(to.Heun(term), to.IntegralController(1e-4, 1e-4)).solve(ivp, term)
    assert np.array_equal(sol.stats["n_steps"].cpu().numpy(), g["n_steps"])
    # PIDController(preset) == the batchode preset; gains map onto betas
    pi42 = to.PIDController(1e-6, 1e-6, preset="PI42")
    assert (pi42.coeffs.beta1, pi42.coeffs.beta2, pi42.coeffs.beta3) == (0.6, -0.2, 0.0)
    p = to.PIDController(1e-6, 1e-6, pcoeff=0.2, icoeff=0.4)
    assert p.coeffs.beta1 == pytest.approx(0.6) and p.coeffs.beta2 == pytest.approx(-0.2)
    with pytest.raises(NotImplementedError):
        to.ODETerm(lambda t, y: y)
    with pytest.raises(ValueError):
        to.InitialValueProblem(y0=torch.ones(2, 1, device="cuda"), t_start=0.0, t_end=0.0)


def test_unreached_points_are_nan():
    import torch

    y0 = torch.ones(1, 1, dtype=torch.float64, device="cuda")
    te = torch.tensor([[0.5, 1.9]], dtype=torch.float64, device="cuda")
    ivp = to.InitialValueProblem(y0=y0, t_start=0.0, t_end=2.0, t_eval=te)
    c = to.IntegralController(1e-8, 1e-8)
    sol = to.AutoDiffAdjoint(to.Dopri5(), c, max_steps=100_000).solve(
        ivp, to.ODETerm(bode.square_dynamics()))
    assert int(sol.status[0]) == int(to.Status.STEP_UNDERFLOW)
    assert abs(float(sol.ys[0, 0, 0]) - 2.0) < 1e-6 and bool(torch.isnan(sol.ys[0, 1, 0]))


def test_sharded_driver_single_rank_gpu():
    sc = G.scenario_map()["c2_vdp_pi42"]
    g = G.load("c2_vdp_pi42")
    prob = bode.IvpBatch(sc["y0"], sc["t_start"], sc["t_end"], sc["t_eval"])
    mu = sc["dyn"]["inst"][:, 0]
    sol = D.solve_sharded(prob, bode.vdp_dynamics(bode.VdpParams(mu)),
                          controller=bode.pid_controller("PI42"), cost_hint=mu * sc["t_end"])
    assert np.array_equal(sol.stats.n_steps, g["n_steps"])
    assert np.all(sol.stats.n_f_evals == g["n_f_evals"][0])
