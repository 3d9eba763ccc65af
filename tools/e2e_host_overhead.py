"""Split of one e2e bode.solve call (C2, page-locked inputs): Python facade
time before the C call, the C call (bode_solve_host: copies + solve + sync),
and the remaining facade time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2210_12375_b200 as bode
from paper_2210_12375_b200 import _abi
cfg = bench.make_config("c2", 0)
P = bode.pinned
prob = bode.IvpBatch(P(cfg["y0"]), P(cfg["t_start"]), P(cfg["t_end"]), P(cfg["te2d"]))
f = bode.vdp_dynamics(bode.VdpParams(P(cfg["mu"])))
kw = dict(tableau=bode.dopri5(), tol=bode.Tolerances(1e-6, 1e-6),
          controller=bode.PidCoefficients(*cfg["ctrl"]["betas"]), max_steps=cfg["max_steps"],
          cost_hint=P(cfg["cost"]), mode="fast")
lib = _abi.load()
orig = lib.bode_solve_host
marks = {}
class Wrap:
    def __call__(self, a):
        marks["c0"] = time.perf_counter()
        r = orig(a)
        marks["c1"] = time.perf_counter()
        return r
_abi._lib.bode_solve_host = Wrap()
for _ in range(3):
    s = bode.solve(prob, f, **kw); del s
res = []
for _ in range(10):
    t0 = time.perf_counter(); s = bode.solve(prob, f, **kw); t1 = time.perf_counter(); del s
    res.append((marks["c0"] - t0, marks["c1"] - marks["c0"], t1 - marks["c1"]))
r = 1e3 * np.median(np.array(res), axis=0)
print(f"python pre {r[0]:.3f} ms, C call {r[1]:.3f} ms, python post {r[2]:.3f} ms")
import torch
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
res = []
for _ in range(10):
    flush.zero_(); torch.cuda.synchronize()
    t0 = time.perf_counter(); s = bode.solve(prob, f, **kw); t1 = time.perf_counter(); del s
    res.append((marks["c0"] - t0, marks["c1"] - marks["c0"], t1 - marks["c1"]))
r = 1e3 * np.median(np.array(res), axis=0)
print(f"with L2 flush: python pre {r[0]:.3f} ms, C call {r[1]:.3f} ms, python post {r[2]:.3f} ms")
