"""Conditioning of a bench config under fused arithmetic, measured on the
oracle itself: the C restatement of batchode (oracle/bode_oracle.c) built
twice -- as pinned (-ffp-contract=off, NumPy's roundings) and with FMA
contraction -- on the same seeded batch.  The scaled ys difference between
the two is the floor any FMA-fused implementation (the GPU fast mode) can
be held to.  Test infrastructure only.

    make -C oracle fma && python tools/oracle_sensitivity.py c5
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import bench  # noqa: E402
import oracle as O  # noqa: E402


def run(cfg, te):
    dyn = (dict(name="vdp", inst=cfg["mu"][:, None]) if cfg["dyn"] == "vdp"
           else dict(name="lorenz", inst=None, shared=(10.0, 28.0, 8.0 / 3.0)))
    return O.solve(cfg["y0"], cfg["t_start"], cfg["t_end"], te, dyn, method=cfg["method"],
                   atol=cfg["tol"], rtol=cfg["tol"], ctrl=cfg["ctrl"],
                   max_steps=cfg["max_steps"], nthreads=os.cpu_count())


def main(name):
    cfg = bench.make_config(name, 0)
    n = cfg["n"]
    te = cfg.get("te1d")
    if te is None:
        te = [np.array([t]) for t in cfg["t_end"]]
    t0 = time.time()
    a = run(cfg, te)
    t1 = time.time()
    O._lib = None
    O.LIB_PATH = os.path.join(ROOT, "oracle", "_build", "liboracle_fma.so")
    b = run(cfg, te)
    same = a["n_steps"] == b["n_steps"]
    ya, yb = a["ys"].reshape(n, -1), b["ys"].reshape(n, -1)
    e = np.abs(ya - yb).max(1) / np.maximum(np.abs(ya).max(1), 1e-300)
    print(f"{name}: n={n}, oracle {t1 - t0:.1f} s; FMA-contracted vs pinned oracle: "
          f"n_steps differ on {int((~same).sum())} rows, statuses differ on "
          f"{int((a['status'] != b['status']).sum())}; scaled ys diff max {e[same].max():.3e}, "
          f"p99.99 {np.quantile(e[same], 0.9999):.3e}, rows > 1e-10: {int((e[same] > 1e-10).sum())}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c5")
