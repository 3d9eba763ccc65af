"""GPU timeline (CUPTI via torch.profiler) of one e2e bode.solve on C2 with
page-locked inputs: copies, kernels and gaps; plus host-side time split."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2210_12375_b200 as bode
chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = bench.make_config("c2", 0)
P = bode.pinned
prob = bode.IvpBatch(P(cfg["y0"]), P(cfg["t_start"]), P(cfg["t_end"]), P(cfg["te2d"]))
f = bode.vdp_dynamics(bode.VdpParams(P(cfg["mu"])))
kw = dict(tableau=bode.dopri5(), tol=bode.Tolerances(1e-6, 1e-6),
          controller=bode.PidCoefficients(*cfg["ctrl"]["betas"]), max_steps=cfg["max_steps"],
          cost_hint=P(cfg["cost"]), pipeline_chunks=chunks, mode="fast")
for _ in range(3):
    s = bode.solve(prob, f, **kw); del s
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter(); s = bode.solve(prob, f, **kw); t1 = time.perf_counter(); del s
pr.disable()
print(f"solve wall {1e3*(t1-t0):.2f} ms")
pstats.Stats(pr).sort_stats("cumulative").print_stats(8)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    s = bode.solve(prob, f, **kw); del s
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
base = evs[0].time_range.start if evs else 0
for e in evs:
    print(f"{(e.time_range.start-base)/1e3:8.3f} ms +{e.time_range.elapsed_us()/1e3:7.3f}  {e.name[:70]}")
