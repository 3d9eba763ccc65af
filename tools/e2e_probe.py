"""e2e breakdown for C2: bode.solve with pinned vs pageable host inputs,
pipeline chunk counts; prints ms per solve."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2210_12375_b200 as bode
cfg = bench.make_config("c2", 0)
n = cfg["n"]
ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"])
for pin in (True, False):
    P = bode.pinned if pin else (lambda x: x)
    prob = bode.IvpBatch(P(cfg["y0"]), P(cfg["t_start"]), P(cfg["t_end"]), P(cfg["te2d"]))
    f = bode.vdp_dynamics(bode.VdpParams(P(cfg["mu"])))
    cost = P(cfg["cost"])
    for chunks in (1, 2, 3, 4, 6, 8):
        kw = dict(tableau=bode.dopri5(), tol=bode.Tolerances(1e-6, 1e-6), controller=ctrl,
                  max_steps=cfg["max_steps"], cost_hint=cost, pipeline_chunks=chunks, mode="fast")
        bode.solve(prob, f, **kw)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); s = bode.solve(prob, f, **kw); ts.append(time.perf_counter() - t0)
            del s
        print(f"pinned_inputs={pin} chunks={chunks}: {1e3*np.median(ts):.2f} ms (min {1e3*min(ts):.2f})", flush=True)
