"""Persistent-kernel time vs launch shape (threads per block) on a bench
config: CUDA events around the integrator launch, L2 flushed between runs.
    python tools/launch_shape_probe.py [c2|c5|c3] [threads ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2210_12375_b200 as bode  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
shapes = [int(x) for x in sys.argv[2:]] or [128, 96, 64]
cfg = bench.make_config(name, 0)
dev = torch.device("cuda:0")
f64 = dict(dtype=torch.float64, device=dev)
y0, ts, tn = (torch.tensor(cfg[k], **f64) for k in ("y0", "t_start", "t_end"))
dyn = (bode.vdp_dynamics(bode.VdpParams(torch.tensor(cfg["mu"], **f64))) if cfg["dyn"] == "vdp"
       else bode.lorenz_dynamics())
te = {k2: torch.tensor(cfg[k1], **f64) for k1, k2 in (("te2d", "t_eval"), ("te1d", "t_eval")) if k1 in cfg}
cost = torch.tensor(cfg["cost"], **f64) if cfg["cost"] is not None else None
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
for thr in shapes:
    ks, acc = [], None
    for r in range(13):
        flush.zero_()
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(), k1.record()
        out = bode.solve_device(y0, ts, tn, dyn, method=cfg["method"], atol=cfg["tol"],
                                rtol=cfg["tol"], controller=bode.PidCoefficients(*cfg["ctrl"]["betas"]),
                                max_steps=cfg["max_steps"], mode="fast", cost_hint=cost,
                                prof_events=(k0, k1), threads_per_block=thr, **te)
        torch.cuda.synchronize()
        if r >= 3:
            ks.append(k0.elapsed_time(k1))
        acc = int(out["n_accepted"].sum())
    print(f"{name} threads={thr}: kernel {np.median(ks):.4f} ms (min {min(ks):.4f}), accepted {acc}")
