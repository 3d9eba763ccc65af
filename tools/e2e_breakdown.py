"""Where the C2 end-to-end solve() time goes: total wall per call vs the
time inside bode_solve_host (C call) -- the rest is the Python facade.
    python tools/e2e_breakdown.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2210_12375_b200 as bode  # noqa: E402
from paper_2210_12375_b200 import _abi  # noqa: E402

cfg = bench.make_config("c2", 0)
P = bode.pinned
prob = bode.IvpBatch(P(cfg["y0"]), P(cfg["t_start"]), P(cfg["t_end"]), P(cfg["te2d"]))
dyn = bode.vdp_dynamics(bode.VdpParams(P(cfg["mu"])))
kw = dict(tableau=bode.dopri5(), tol=bode.Tolerances(cfg["tol"], cfg["tol"]),
          controller=bode.PidCoefficients(*cfg["ctrl"]["betas"]), max_steps=cfg["max_steps"],
          mode="fast", cost_hint=P(cfg["cost"]))
lib = _abi.load()
inner = []
orig = lib.bode_solve_host


def timed(*a):
    t0 = time.perf_counter()
    r = orig(*a)
    inner.append(time.perf_counter() - t0)
    return r


lib.bode_solve_host = timed
for chunks in ("auto", 1, 2, 3, 4, 6):
    inner.clear()
    tot = []
    for _ in range(6):
        t0 = time.perf_counter()
        sol = bode.solve(prob, dyn, pipeline_chunks=chunks, **kw)
        tot.append(time.perf_counter() - t0)
        del sol
    print(f"chunks={chunks}: solve() {1e3 * np.median(tot[1:]):.2f} ms, "
          f"bode_solve_host {1e3 * np.median(inner[1:]):.2f} ms")
