"""Strong-scaling floor of the sharded 2^20 batches: the
time the single most expensive instance needs on an otherwise idle GPU
bounds any N-GPU time from below, whatever the partition.  Prints, per
config, the one-GPU solve time, that floor and the efficiency ceiling
T1 / (N * max(T1 / N, floor)) for N = 2, 4, 8."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2210_12375_b200 as bode  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, out


def main():
    f64 = dict(dtype=torch.float64, device="cuda")
    for name in ("c2", "c5"):
        cfg = bench.make_config(name, 0)
        n = cfg["n"]
        y0 = torch.tensor(cfg["y0"], **f64)
        ts, tn = torch.tensor(cfg["t_start"], **f64), torch.tensor(cfg["t_end"], **f64)
        mu = torch.tensor(cfg["mu"], **f64)
        cost = torch.tensor(cfg["cost"], **f64)
        kw = dict(controller=bode.PidCoefficients(*cfg["ctrl"]["betas"]), mode="fast",
                  max_steps=cfg["max_steps"])
        t1, out = timed(lambda: bode.solve_device(y0, ts, tn, bode.vdp_dynamics(bode.VdpParams(mu)),
                                                  cost_hint=cost, **kw))
        i = int(torch.argmax(out["n_steps"]))
        steps = int(out["n_steps"][i])
        tf, _ = timed(lambda: bode.solve_device(y0[i:i + 1], ts[i:i + 1], tn[i:i + 1],
                                                bode.vdp_dynamics(bode.VdpParams(mu[i:i + 1])), **kw))
        ceil = {N: t1 / (N * max(t1 / N, tf)) for N in (2, 4, 8)}
        print(f"{name}: one-GPU solve {t1:.3f} ms; heaviest instance {i} ({steps} steps) alone "
              f"{tf:.3f} ms; strong-scaling efficiency ceiling "
              + ", ".join(f"N={N}: {100 * c:.0f}%" for N, c in ceil.items()))


if __name__ == "__main__":
    main()
