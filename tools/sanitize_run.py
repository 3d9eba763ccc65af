"""Small solves through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck; tools/sanitize.sh): the persistent
analytic kernel (LPT queue, dense output, trace), the fused tcgen05 MLP
kernel (TMEM / mbarrier pipeline, row refill), a run-time program (traced
lambda + user tableau), the stepping API and the adjoint kernels."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import bench  # noqa: E402
import dropin_cases as DC  # noqa: E402
import paper_2210_12375_b200 as bode  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
f64 = dict(dtype=torch.float64, device="cuda")
if which in ("all", "analytic"):
    rng = np.random.default_rng(0)
    n = 6000
    mu = rng.uniform(1.0, 10.0, n)
    te = rng.uniform(5.0, 20.0, n)
    for mode in ("fast", "exact"):
        out = bode.solve_device(torch.tensor(np.tile([2.0, 0.0], (n, 1)), **f64),
                                torch.zeros(n, **f64), torch.tensor(te, **f64),
                                bode.vdp_dynamics(bode.VdpParams(torch.tensor(mu, **f64))),
                                t_eval=torch.tensor(np.stack([te / 2, te], 1), **f64),
                                controller=bode.pid_controller("PI42"), mode=mode,
                                cost_hint=torch.tensor(mu * te, **f64), record_trace=mode == "exact",
                                max_steps=400)
    torch.cuda.synchronize()
    print("analytic ok", int(out["n_steps"].sum()))
if which in ("all", "mlp"):
    cfg = bench.make_config("c4", 0, n_override=600)
    sol = bode.solve(bode.IvpBatch(cfg["y0"], cfg["t_start"], np.full(600, 2.0),
                                   np.full((600, 1), 2.0)), bode.mlp_dynamics(*cfg["mlp"]))
    print("mlp ok", int(sol.stats.n_steps.sum()))
if which in ("all", "program"):
    tab = bode.ButcherTableau(**DC.bs3_data())
    mu = np.random.default_rng(1).uniform(1, 5, 500)
    f = lambda t, y: np.stack([y[:, 1], mu * (1 - y[:, 0] ** 2) * y[:, 1] - y[:, 0]], 1)  # noqa: E731
    prob = bode.IvpBatch(np.tile([2.0, 0.0], (500, 1)), np.zeros(500), np.full(500, 3.0),
                         np.linspace(0, 3, 4))
    sol = bode.solve(prob, f, tableau=tab)
    s = bode.BatchSolver(prob, f, tableau=tab)
    for _ in range(20):
        s.step_once()
    print("program ok", int(sol.stats.n_steps.sum()))
if which in ("all", "adjoint"):
    n = 300
    mu = torch.tensor(np.random.default_rng(2).uniform(1, 5, n), **f64)
    fwd = bode.solve_device(torch.tensor(np.tile([2.0, 0.0], (n, 1)), **f64), 0.0, 3.0,
                            bode.vdp_dynamics(bode.VdpParams(mu)),
                            t_eval=torch.tensor([1.0, 3.0], **f64), record_trajectory=True)
    g0, gp = bode.adjoint_device(fwd, torch.ones_like(fwd["ys"]))
    torch.cuda.synchronize()
    print("adjoint ok", float(g0.abs().sum()))
if which in ("all", "mlp_adjoint"):
    # tensor-core MLP backward (D=64): fused recording with stage inputs,
    # the VJP kernels and the split-K weight-gradient GEMM over 3 tiles
    cfg = bench.make_config("c4", 0, n_override=300)
    W = [torch.tensor(w, device="cuda") for w in cfg["mlp"]]
    fwd = bode.solve_device(torch.tensor(cfg["y0"], **f64), 0.0, 1.0, bode.mlp_dynamics(*W),
                            t_eval=torch.tensor([0.5, 1.0], **f64), record_trajectory=True)
    g0, gw = bode.adjoint_device(fwd, torch.ones_like(fwd["ys"]))
    torch.cuda.synchronize()
    print("mlp adjoint ok", float(g0.abs().sum()), float(gw["W1"].abs().sum()))
