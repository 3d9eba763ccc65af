"""GPU timeline of one device-resident solve (torch.profiler/CUPTI): kernel
start offsets and durations, to find idle gaps outside the persistent kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2210_12375_b200 as bode
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
cfg = bench.make_config(cfgname, 0)
dev = torch.device("cuda", 0)
f64 = dict(dtype=torch.float64, device=dev)
y0 = torch.tensor(cfg["y0"], **f64); ts = torch.tensor(cfg["t_start"], **f64); tn = torch.tensor(cfg["t_end"], **f64)
dyn = bode.vdp_dynamics(bode.VdpParams(torch.tensor(cfg["mu"], **f64))) if cfg["dyn"] == "vdp" else bode.lorenz_dynamics()
te = torch.tensor(cfg["te2d"] if "te2d" in cfg else cfg["te1d"], **f64)
cost = torch.tensor(cfg["cost"], **f64) if cfg["cost"] is not None else None
ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"])
def one():
    return bode.solve_device(y0, ts, tn, dyn, t_eval=te, method=cfg["method"], atol=cfg["tol"], rtol=cfg["tol"],
                             controller=ctrl, max_steps=cfg["max_steps"], cost_hint=cost, mode=mode)
for _ in range(3): one()
torch.cuda.synchronize()
t0 = time.perf_counter(); o = one(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0):.3f} ms, total wall {1e3*(t2-t0):.3f} ms")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    o = one(); torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
base = evs[0].time_range.start if evs else 0
for e in evs:
    print(f"{(e.time_range.start-base)/1e3:9.3f} ms  {e.time_range.elapsed_us()/1e3:8.3f} ms  {e.name[:90]}")
