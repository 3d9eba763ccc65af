"""GPU gradient path (bode_solve_adjoint, csrc/bode_adjoint.cu) against the
autograd replay oracle (oracle/adjoint_oracle.py, pinned on the CPU by
tests/test_adjoint_oracle.py).

Tolerance: the adjoint is fp64 with FMA contraction and the forward's step
sequence agrees with the oracle's to the last few ulps (exact mode), so
gradients must agree to 1e-9 of each instance's largest gradient entry
(observed ~1e-13)."""

import numpy as np
import pytest

import adjoint_oracle as AO
from adjoint_cases import CASES, SLOTS, case, grad_seed, run_oracle

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _gpu(c, mode="exact", grad=False):
    import torch

    import paper_2210_12375_b200 as bode
    from paper_2210_12375_b200.dynamics import DeviceDynamics

    dev = torch.device("cuda:0")
    n = c["y0"].shape[0]
    params = {}
    for k, v in c["params"].items():
        params[k] = torch.tensor(np.asarray(v, dtype=np.float64), device=dev) if np.ndim(v) else v
    dyn = DeviceDynamics(c["dyn"], params)
    lens = np.array([len(t) for t in c["t_eval"]])
    offs = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64, device=dev)
    tv = torch.tensor(np.concatenate(c["t_eval"]), dtype=torch.float64, device=dev)
    ctrl = bode.PidCoefficients(*c["ctrl"]["betas"], c["ctrl"]["safety"],
                                c["ctrl"]["factor_min"], c["ctrl"]["factor_max"],
                                c["ctrl"]["hist"])
    out = bode.solve_device(torch.tensor(c["y0"], device=dev), c["t_start"],
                            torch.tensor(np.broadcast_to(c["t_end"], (n,)).copy(), device=dev),
                            dyn, t_eval=tv, t_eval_offsets=offs, method=c["method"],
                            atol=c["tol"], rtol=c["tol"], controller=ctrl,
                            max_steps=c["max_steps"], mode=mode, record_trajectory=grad)
    return out


@pytest.mark.parametrize("name", CASES)
def test_adjoint_matches_autograd_oracle(name):
    import torch

    import paper_2210_12375_b200 as bode

    c = case(name, n=16)
    ref = run_oracle(c)
    G = grad_seed(c)
    gy0_ref, gp_ref = AO.gradients(c["method"], c["dyn"], c["params"], c["y0"], c["t_start"],
                                   ref, c["t_eval"], G)
    out = _gpu(c, grad=True)
    np.testing.assert_array_equal(out["n_accepted"].cpu().numpy(), ref["n_accepted"])
    np.testing.assert_array_equal(out["n_emitted"].cpu().numpy(), ref["n_emitted"])
    gy = torch.tensor(np.concatenate(G), device="cuda:0")
    gy0, gp = bode.adjoint_device(out, gy)
    gy0, gp = gy0.cpu().numpy(), gp.cpu().numpy()
    assert out["adjoint_launches"] > 0
    for i in range(c["y0"].shape[0]):
        ref_i = np.concatenate([gy0_ref[i], [gp_ref[k][i] for k in gp_ref]])
        got_i = np.concatenate([gy0[i], [gp[i, SLOTS[c["dyn"]].index(k)] for k in gp_ref]])
        scale = max(1.0, np.abs(ref_i).max())
        assert np.abs(got_i - ref_i).max() <= TOL * scale, (name, i, got_i, ref_i)


@pytest.mark.parametrize("name", ["vdp_pi42", "lorenz_tsit5"])
def test_trajectory_matches_oracle_steps(name):
    c = case(name, n=16)
    ref = run_oracle(c)
    out = _gpu(c, grad=True)
    traj = out["traj"].cpu().numpy()
    toff = out["traj_offsets"].cpu().numpy()
    for i in range(16):
        steps = np.array(AO.accepted_steps(ref, i))
        rec = traj[toff[i]:toff[i + 1]]
        assert rec.shape[0] == steps.shape[0]
        # step sizes agree to a few ulps grown through the controller (one
        # ulp of pow), like the final_dt comparisons
        np.testing.assert_allclose(rec[:, :2], steps, rtol=1e-6, atol=1e-300)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_recording_does_not_change_the_solve(mode):
    c = case("vdp_pi42", n=64)
    a = _gpu(c, mode=mode, grad=False)
    b = _gpu(c, mode=mode, grad=True)
    for k in ("ys", "n_steps", "n_accepted", "n_emitted", "final_dt", "status", "n_f_evals"):
        assert bool((a[k] == b[k]).all()), k


def test_fast_mode_adjoint_within_tolerance():
    import torch

    import paper_2210_12375_b200 as bode

    c = case("vdp_pi42", n=16)
    ref = run_oracle(c)
    G = grad_seed(c)
    gy0_ref, _ = AO.gradients(c["method"], c["dyn"], c["params"], c["y0"], c["t_start"], ref,
                              c["t_eval"], G)
    out = _gpu(c, mode="fast", grad=True)
    gy0, _ = bode.adjoint_device(out, torch.tensor(np.concatenate(G), device="cuda:0"))
    gy0 = gy0.cpu().numpy()
    scale = np.maximum(1.0, np.abs(gy0_ref).max(axis=1, keepdims=True))
    assert (np.abs(gy0 - gy0_ref) <= 1e-7 * scale).all()


def test_torchode_backward():
    """AutoDiffAdjoint.solve: y0 and dynamics-parameter tensors get .grad
    from loss.backward(), equal to the oracle's."""
    import torch

    import paper_2210_12375_b200.torchode as to
    from paper_2210_12375_b200.dynamics import lorenz_dynamics, vdp_dynamics, VdpParams

    dev = torch.device("cuda:0")
    c = case("lorenz_tsit5", n=8)
    ref = run_oracle(c)
    G = grad_seed(c)
    gy0_ref, gp_ref = AO.gradients(c["method"], c["dyn"], c["params"], c["y0"], c["t_start"],
                                   ref, c["t_eval"], G)
    y0 = torch.tensor(c["y0"], device=dev, requires_grad=True)
    sigma = torch.tensor(10.0, dtype=torch.float64, device=dev, requires_grad=True)
    term = to.ODETerm(lorenz_dynamics(sigma=sigma))
    solver = to.AutoDiffAdjoint(to.Tsit5(term), to.IntegralController(atol=1e-8, rtol=1e-8))
    te = torch.tensor(c["t_eval"][0], device=dev)
    sol = solver.solve(to.InitialValueProblem(y0=y0, t_eval=te))
    assert sol.ys.requires_grad
    loss = (sol.ys * torch.tensor(np.stack(G), device=dev)).sum()
    loss.backward()
    np.testing.assert_allclose(y0.grad.cpu().numpy(), gy0_ref, rtol=0, atol=TOL * max(1.0, np.abs(gy0_ref).max()))
    assert abs(float(sigma.grad) - gp_ref["sigma"].sum()) <= TOL * max(1.0, abs(gp_ref["sigma"]).sum())

    # per-instance parameter tensor (VdP mu), PI controller
    c = case("vdp_max_steps", n=8)
    c["t_eval"] = [np.linspace(0.0, 8.0, 17)] * 8
    ref = run_oracle(c)
    G = grad_seed(c)
    _, gp_ref = AO.gradients(c["method"], c["dyn"], c["params"], c["y0"], c["t_start"], ref,
                             c["t_eval"], G)
    mu = torch.tensor(c["params"]["mu"], device=dev, requires_grad=True)
    term = to.ODETerm(vdp_dynamics(VdpParams(mu)))
    solver = to.AutoDiffAdjoint(to.Dopri5(term), to.IntegralController(atol=1e-6, rtol=1e-6),
                                max_steps=60)
    sol = solver.solve(to.InitialValueProblem(y0=torch.tensor(c["y0"], device=dev),
                                              t_eval=torch.tensor(c["t_eval"][0], device=dev)))
    ys = torch.nan_to_num(sol.ys)  # unreached points (MAX_STEPS rows) are NaN
    (ys * torch.tensor(np.stack(G), device=dev)).sum().backward()
    np.testing.assert_allclose(mu.grad.cpu().numpy(), gp_ref["mu"], rtol=0,
                               atol=TOL * max(1.0, np.abs(gp_ref["mu"]).max()))


def _mlp_weights(D, H, seed=3):
    rng = np.random.default_rng(seed)
    W1 = (rng.normal(size=(H, D)) / np.sqrt(D)).astype(np.float32)
    b1 = (0.1 * rng.normal(size=H)).astype(np.float32)
    W2 = (rng.normal(size=(D, H)) / np.sqrt(H)).astype(np.float32)
    b2 = (0.1 * rng.normal(size=D)).astype(np.float32)
    return W1, b1, W2, b2


@pytest.mark.parametrize("D,H,method,n", [(4, 32, "dopri5", 12), (8, 64, "tsit5", 12),
                                          (16, 48, "heun", 12), (64, 256, "dopri5", 12),
                                          (64, 256, "tsit5", 160), (64, 96, "dopri5", 140),
                                          (64, 128, "heun", 130)])
def test_mlp_adjoint_matches_autograd_oracle(D, H, method, n):
    """Neural-ODE gradients (dL/dy0 and the batch-summed dL/dW1, db1, dW2,
    db2) against torch autograd through the fp32-MLP replay of the GPU's own
    accepted steps (fp32 dynamics: tolerance 2e-4 of each gradient's scale).
    At D=64 the solve and its recording run the fused tcgen05 kernel and the
    backward runs on the tensor cores (bode_mlp_adjoint_tc.cu): n > 128 spans
    several 128-row tiles, a partial last tile, trajectories of different
    lengths (y0 scales vary), and H not a multiple of 128."""
    import torch

    import paper_2210_12375_b200 as bode

    dev = torch.device("cuda:0")
    W = _mlp_weights(D, H)
    m = 6
    rng = np.random.default_rng(4)
    y0 = rng.normal(size=(n, D)) * rng.uniform(0.2, 3.0, size=(n, 1))
    te = np.linspace(0.0, 1.0, m)
    dyn = bode.mlp_dynamics(*[torch.tensor(w, device=dev) for w in W])
    kw = dict(t_eval=torch.tensor(te, device=dev), method=method, atol=1e-6, rtol=1e-6,
              max_steps=100_000)
    plain = bode.solve_device(torch.tensor(y0, device=dev), 0.0, 1.0, dyn, **kw)
    out = bode.solve_device(torch.tensor(y0, device=dev), 0.0, 1.0, dyn, record_trajectory=True, **kw)
    for k in ("ys", "n_steps", "n_accepted", "status"):
        assert bool((plain[k] == out[k]).all()), k
    G = rng.normal(size=(n, m, D))
    gy0, gw = bode.adjoint_device(out, torch.tensor(G.reshape(-1, D), device=dev))
    traj = out["traj"].cpu().numpy()
    toff = out["traj_offsets"].cpu().numpy()
    steps = [[tuple(r) for r in traj[toff[i]:toff[i + 1], :2]] for i in range(n)]
    gy0_ref, gw_ref = AO.gradients_mlp(method, W, y0, 0.0, steps, [te] * n, list(G))
    got = gy0.cpu().numpy()
    assert np.abs(got - gy0_ref).max() <= 2e-4 * np.abs(gy0_ref).max()
    for k in ("W1", "b1", "W2", "b2"):
        g, r = gw[k].cpu().numpy(), gw_ref[k]
        assert g.shape == r.shape
        assert np.abs(g - r).max() <= 2e-4 * np.abs(r).max(), k


def test_torchode_mlp_backward():
    """AutoDiffAdjoint on neural-ODE dynamics: .grad of y0 and of the weight
    tensors equals the adjoint_device results."""
    import torch

    import paper_2210_12375_b200 as bode
    import paper_2210_12375_b200.torchode as to

    dev = torch.device("cuda:0")
    D, H, n = 8, 32, 10
    W = [torch.tensor(w, device=dev, requires_grad=True) for w in _mlp_weights(D, H)]
    y0 = torch.tensor(np.random.default_rng(5).normal(size=(n, D)), device=dev, requires_grad=True)
    te = torch.linspace(0.0, 1.0, 5, dtype=torch.float64, device=dev)
    term = to.ODETerm(bode.mlp_dynamics(*W))
    sol = to.AutoDiffAdjoint(to.Dopri5(term), to.IntegralController(1e-6, 1e-6)).solve(
        to.InitialValueProblem(y0=y0, t_eval=te))
    G = torch.randn_like(sol.ys)
    (sol.ys * G).sum().backward()
    dyn = bode.mlp_dynamics(*[w.detach() for w in W])
    out = bode.solve_device(y0.detach(), 0.0, 1.0, dyn, t_eval=te, atol=1e-6, rtol=1e-6,
                            record_trajectory=True)
    gy0, gw = bode.adjoint_device(out, G.reshape(-1, D))
    assert torch.equal(y0.grad, gy0)
    for w, k in zip(W, ("W1", "b1", "W2", "b2")):
        assert torch.allclose(w.grad, gw[k], rtol=1e-5, atol=1e-6), k
