"""Per-attempted-step cost vs instance length (refill overhead probe): C2
with t_end scaled by 1x / 4x / 16x (same instance count)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2210_12375_b200 as bode
dev = torch.device("cuda", 0)
f64 = dict(dtype=torch.float64, device=dev)
cfg = bench.make_config("c2", 0)
for scale in (1, 4, 16):
    n = cfg["n"] // scale
    y0 = torch.tensor(cfg["y0"][:n], **f64); ts = torch.zeros(n, **f64)
    tn = torch.tensor(cfg["t_end"][:n] * scale, **f64)
    dyn = bode.vdp_dynamics(bode.VdpParams(torch.tensor(cfg["mu"][:n], **f64)))
    cost = torch.tensor(cfg["mu"][:n] * cfg["t_end"][:n] * scale, **f64)
    ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"])
    for notev in (False, True):
        kw = {} if notev else dict(t_eval=tn[:, None].clone())
        run = lambda: bode.solve_device(y0, ts, tn, dyn, controller=ctrl, max_steps=100000, cost_hint=cost, mode="fast", **kw)
        for _ in range(2): o = run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); o = run(); e1.record(); e1.synchronize()
        att = int(o["n_steps"].sum()); rej = att - int(o["n_accepted"].sum())
        print(f"scale {scale:2d} n={n:7d} t_eval={not notev}: {e0.elapsed_time(e1):.3f} ms, {att/n:.0f} steps/inst, "
              f"{1e9*e0.elapsed_time(e1)/1e3/att:.2f} ps/step, reject {rej/att:.3f}")
