"""e2e (C2, page-locked inputs) vs pipeline chunk count; run under
different BODE_EDGE_FRAC values (first/last chunk size relative to a middle one)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2210_12375_b200 as bode
cfg = bench.make_config("c2", 0)
ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"])
P = bode.pinned
prob = bode.IvpBatch(P(cfg["y0"]), P(cfg["t_start"]), P(cfg["t_end"]), P(cfg["te2d"]))
f = bode.vdp_dynamics(bode.VdpParams(P(cfg["mu"])))
cost = P(cfg["cost"])
for chunks in (3, 4, 5):
    kw = dict(tableau=bode.dopri5(), tol=bode.Tolerances(1e-6, 1e-6), controller=ctrl,
              max_steps=cfg["max_steps"], cost_hint=cost, pipeline_chunks=chunks, mode="fast")
    bode.solve(prob, f, **kw)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter(); s = bode.solve(prob, f, **kw); ts.append(time.perf_counter() - t0)
        del s
    print(f"edge={os.environ.get('BODE_EDGE_FRAC', '0.5')} chunks={chunks}: {1e3*np.median(ts):.2f} ms", flush=True)
