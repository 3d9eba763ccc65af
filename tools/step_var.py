"""Per-step device timing of the C2 solve (variance diagnosis): gap before the
persistent kernel, kernel, gap after, for K back-to-back steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2210_12375_b200 as bode
cfg = bench.make_config("c2", 0)
dev = torch.device("cuda", 0)
f64 = dict(dtype=torch.float64, device=dev)
y0 = torch.tensor(cfg["y0"], **f64); ts = torch.tensor(cfg["t_start"], **f64); tn = torch.tensor(cfg["t_end"], **f64)
dyn = bode.vdp_dynamics(bode.VdpParams(torch.tensor(cfg["mu"], **f64)))
te = torch.tensor(cfg["te2d"], **f64); cost = torch.tensor(cfg["cost"], **f64)
ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"])
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream(dev)
def one(prof=None):
    return bode.solve_device(y0, ts, tn, dyn, t_eval=te, controller=ctrl, max_steps=cfg["max_steps"],
                             cost_hint=cost, mode="fast", prof_events=prof)
for _ in range(3): one()
torch.cuda.synchronize()
for trial in range(3):
    pend = []
    for _ in range(10):
        if "noflush" not in sys.argv: flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[1].record(st); ev[2].record(st); ev[0].record(st)
        o = one((ev[1], ev[2])); ev[3].record(st)
        pend.append((ev, o))
    torch.cuda.synchronize()
    rows = [(e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])) for e, _ in pend]
    print("trial", trial, " ".join(f"{a:.2f}/{b:.2f}/{c:.2f}" for a, b, c in rows))
