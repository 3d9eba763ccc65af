"""Gradient path at full scale (C2: 2^20 Van der Pol instances, dopri5,
PI42, fast mode): time of the recording forward solve and of the adjoint
kernel, trajectory bytes, and a parity check of a seeded 32-instance
subsample against the autograd replay oracle (batch independence makes a
subsample exact) plus linearity of the adjoint in dL/dys.

    python tools/adjoint_bench.py [--n N] [--reps R]   (prints one JSON line)
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)


def main():
    import torch

    import bench
    import paper_2210_12375_b200 as bode
    from paper_2210_12375_b200 import _abi

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2 ** 20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--config", default="c2", choices=["c2", "c4"])
    args = ap.parse_args()
    if args.config == "c4":
        return main_c4(args)
    cfg = bench.make_config("c2", 0, n_override=args.n)
    dev = torch.device("cuda:0")
    n = cfg["n"]
    T = lambda x: torch.tensor(x, device=dev)  # noqa: E731
    mu = T(cfg["mu"])
    ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"], cfg["ctrl"]["safety"],
                                cfg["ctrl"]["factor_min"], cfg["ctrl"]["factor_max"],
                                cfg["ctrl"]["hist"])
    kw = dict(t_eval=T(cfg["te2d"]), method="dopri5", atol=cfg["tol"], rtol=cfg["tol"],
              controller=ctrl, max_steps=cfg["max_steps"], mode=args.mode,
              cost_hint=T(cfg["cost"]))
    y0, t0, t1 = T(cfg["y0"]), T(cfg["t_start"]), T(cfg["t_end"])
    dyn = bode.vdp_dynamics(bode.VdpParams(mu))
    out = bode.solve_device(y0, t0, t1, dyn, record_trajectory=True, **kw)
    lib = _abi.load()
    a = out["_args"]
    gy = torch.ones_like(out["ys"])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    t_plain, t_rec, t_adj = [], [], []
    plain_traj = a.traj
    for _ in range(args.reps):
        torch.cuda.synchronize()
        a.traj = None
        ev[0].record()
        _abi.check(lib.bode_solve(_abi.C.byref(a)))
        ev[1].record()
        a.traj = plain_traj
        ev[2].record()
        _abi.check(lib.bode_solve(_abi.C.byref(a)))
        ev[3].record()
        g0, gp = bode.adjoint_device(out, gy)
        ev[4].record()
        torch.cuda.synchronize()
        t_plain.append(ev[0].elapsed_time(ev[1]))
        t_rec.append(ev[2].elapsed_time(ev[3]))
        t_adj.append(ev[3].elapsed_time(ev[4]))
    acc = int(out["n_accepted"].sum())
    rows = int(out["traj_offsets"][-1])

    # linearity in dL/dys
    g1 = torch.randn_like(gy)
    g2 = torch.randn_like(gy)
    a1, _ = bode.adjoint_device(out, g1)
    a2, _ = bode.adjoint_device(out, g2)
    a12, _ = bode.adjoint_device(out, g1 + 2.0 * g2)
    lin = float(((a12 - (a1 + 2.0 * a2)).abs().max() / a12.abs().max()))

    # subsample parity against the autograd replay oracle
    import adjoint_oracle as AO
    import oracle as O

    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(n, 32, replace=False))
    ref = O.solve(cfg["y0"][idx], 0.0, cfg["t_end"][idx], [cfg["te2d"][i] for i in idx],
                  dict(name="vdp", inst=cfg["mu"][idx, None]), method="dopri5", atol=cfg["tol"],
                  rtol=cfg["tol"], ctrl=cfg["ctrl"], max_steps=cfg["max_steps"], trace=True)
    G = [np.ones((1, 2)) for _ in idx]
    gy0_ref, gp_ref = AO.gradients("dopri5", "vdp", {"mu": cfg["mu"][idx]}, cfg["y0"][idx], 0.0,
                                   ref, [cfg["te2d"][i] for i in idx], G)
    g0n, gpn = g0.cpu().numpy()[idx], gp.cpu().numpy()[idx, 0]
    scale = np.maximum(1.0, np.abs(np.concatenate([gy0_ref, gp_ref["mu"][:, None]], 1)).max(1))
    err = np.max(np.abs(np.concatenate([g0n - gy0_ref, (gpn - gp_ref["mu"])[:, None]], 1)).max(1)
                 / scale)
    med = lambda v: float(np.median(v))  # noqa: E731
    print(json.dumps(dict(
        workload=cfg["workload"] + "_gradient", n=n, mode=args.mode,
        accepted_steps=acc, traj_rows=rows, traj_bytes=rows * _abi.traj_stride(2) * 8,
        forward_ms=med(t_plain), recording_forward_ms=med(t_rec), adjoint_ms=med(t_adj),
        gradient_instance_steps_per_s=acc / ((med(t_rec) + med(t_adj)) / 1e3),
        adjoint_launches=out.get("adjoint_launches"),
        linearity_rel_err=lin, subsample_max_scaled_err=float(err),
        subsample_counts_equal=bool(np.array_equal(out["n_accepted"].cpu().numpy()[idx],
                                                   ref["n_accepted"])))))


def main_c4(args):
    """Neural ODE (C4: 64K instances, D=64, H=256, dopri5, t in [0,10]):
    recording forward, adjoint (dL/dy0 + weight gradients), subsample
    parity of dL/dy0 vs the autograd replay of the GPU's own steps."""
    import torch

    import bench
    import paper_2210_12375_b200 as bode
    from paper_2210_12375_b200 import _abi

    cfg = bench.make_config("c4", 0, n_override=None if args.n == 2 ** 20 else args.n)
    dev = torch.device("cuda:0")
    n, D = cfg["n"], cfg["d"]
    W = [torch.tensor(w, device=dev) for w in cfg["mlp"]]
    dyn = bode.mlp_dynamics(*W)
    kw = dict(t_eval=torch.tensor(cfg["te2d"], device=dev), method="dopri5", atol=cfg["tol"],
              rtol=cfg["tol"], max_steps=cfg["max_steps"])
    y0 = torch.tensor(cfg["y0"], device=dev)
    out = bode.solve_device(y0, 0.0, 10.0, dyn, record_trajectory=True, **kw)
    lib = _abi.load()
    a = out["_args"]
    gy = torch.ones_like(out["ys"])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    t_plain, t_rec, t_adj = [], [], []
    rec_traj = a.traj
    for _ in range(args.reps):
        torch.cuda.synchronize()
        a.traj = None
        ev[0].record()
        _abi.check(lib.bode_solve(_abi.C.byref(a)))
        ev[1].record()
        a.traj = rec_traj
        _abi.check(lib.bode_solve(_abi.C.byref(a)))
        ev[2].record()
        g0, gw = bode.adjoint_device(out, gy)
        ev[3].record()
        torch.cuda.synchronize()
        t_plain.append(ev[0].elapsed_time(ev[1]))
        t_rec.append(ev[1].elapsed_time(ev[2]))
        t_adj.append(ev[2].elapsed_time(ev[3]))
    acc = int(out["n_accepted"].sum())
    print("timed", t_plain, t_rec, t_adj, file=sys.stderr, flush=True)
    import adjoint_oracle as AO

    idx = np.sort(np.random.default_rng(5).choice(n, 4, replace=False))
    traj = out["traj"].cpu().numpy()
    toff = out["traj_offsets"].cpu().numpy()
    steps = [[tuple(r) for r in traj[toff[i]:toff[i + 1], :2]] for i in idx]
    gy0_ref, _ = AO.gradients_mlp("dopri5", cfg["mlp"], cfg["y0"][idx], 0.0, steps,
                                  [cfg["te2d"][i] for i in idx], [np.ones((1, D))] * len(idx))
    err = float(np.abs(g0.cpu().numpy()[idx] - gy0_ref).max() / np.abs(gy0_ref).max())
    med = lambda v: float(np.median(v))  # noqa: E731
    print(json.dumps(dict(
        workload=cfg["workload"] + "_gradient", n=n, accepted_steps=acc,
        traj_bytes=int(toff[-1]) * _abi.traj_stride(D) * 8,
        forward_ms=med(t_plain), recording_forward_ms=med(t_rec), adjoint_ms=med(t_adj),
        gradient_instance_steps_per_s=acc / ((med(t_rec) + med(t_adj)) / 1e3),
        adjoint_launches=out.get("adjoint_launches"), subsample_rel_err_dy0=err,
        weight_grad_norms={k: float(v.norm()) for k, v in gw.items()})))


if __name__ == "__main__":
    main()
