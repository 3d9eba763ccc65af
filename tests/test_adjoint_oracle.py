"""Pins the gradient oracle (oracle/adjoint_oracle.py) on the CPU: its
replay of the accepted steps reproduces the pinned C oracle's ys, and its
autograd gradients equal central finite differences of the same replay."""

import numpy as np
import pytest
import torch

import adjoint_oracle as AO
from adjoint_cases import CASES, case, grad_seed, run_oracle


@pytest.mark.parametrize("name", CASES)
def test_replay_reproduces_oracle_ys(name):
    c = case(name, n=6)
    ref = run_oracle(c)
    ys = AO.replay_ys(c["method"], c["dyn"], c["params"], c["y0"], c["t_start"], ref, c["t_eval"])
    offs = ref["te_offs"]
    for i in range(6):
        r = ref["ys"][offs[i]:offs[i] + ref["n_emitted"][i]]
        assert ys[i].shape == r.shape
        if r.size:
            scale = max(np.abs(r).max(), 1e-300)
            assert np.abs(ys[i] - r).max() <= 1e-12 * scale, name


@pytest.mark.parametrize("name", ["vdp_pi42", "lorenz_tsit5", "linear_cos_heun",
                                  "damped_backward", "relax_cos_tsit5"])
def test_autograd_matches_finite_differences(name):
    c = case(name, n=2)
    ref = run_oracle(c)
    G = grad_seed(c)
    gy0, gp = AO.gradients(c["method"], c["dyn"], c["params"], c["y0"], c["t_start"], ref,
                           c["t_eval"], G)
    f = AO.dynamics(c["dyn"])
    i = 0
    steps = AO.accepted_steps(ref, i)
    te = np.asarray(c["t_eval"][i])
    t0 = float(np.broadcast_to(c["t_start"], (2,))[i])

    def loss(y0, params):
        with torch.no_grad():
            p = {k: torch.tensor(float(np.broadcast_to(v, (2,))[i]), dtype=torch.float64)
                 for k, v in params.items()}
            ys = AO.replay(c["method"], f, p, torch.tensor(y0, dtype=torch.float64), t0, steps, te)
            g = torch.as_tensor(G[i][:ys.shape[0]])
            return float((ys * g).sum())

    eps = 1e-6
    for j in range(c["y0"].shape[1]):
        yp, ym = c["y0"][i].copy(), c["y0"][i].copy()
        yp[j] += eps
        ym[j] -= eps
        fd = (loss(yp, c["params"]) - loss(ym, c["params"])) / (2 * eps)
        assert abs(fd - gy0[i, j]) <= 1e-6 * max(1.0, abs(fd)), (name, j, fd, gy0[i, j])
    for k, v in c["params"].items():
        vp, vm = dict(c["params"]), dict(c["params"])
        base = np.broadcast_to(v, (2,)).astype(float).copy()
        hp, hm = base.copy(), base.copy()
        hp[i] += eps
        hm[i] -= eps
        vp[k], vm[k] = hp, hm
        fd = (loss(c["y0"][i], vp) - loss(c["y0"][i], vm)) / (2 * eps)
        assert abs(fd - gp[k][i]) <= 1e-6 * max(1.0, abs(fd)), (name, k, fd, gp[k][i])
