import sys, time, os
sys.path[:0] = ["/root/repo", "/root/repo/oracle", "/root/repo/tests"]
import numpy as np, torch
import bench, paper_2210_12375_b200 as bode
n = int(sys.argv[1])
cfg = bench.make_config("c4", 0, n_override=n)
dev = torch.device("cuda:0")
W = [torch.tensor(w, device=dev) for w in cfg["mlp"]]
dyn = bode.mlp_dynamics(*W)
kw = dict(t_eval=torch.tensor(cfg["te2d"], device=dev), method="dopri5", atol=1e-6, rtol=1e-6, max_steps=100000)
y0 = torch.tensor(cfg["y0"], device=dev)
t0 = time.time(); out = bode.solve_device(y0, 0.0, 10.0, dyn, **kw); torch.cuda.synchronize(); print("plain", time.time() - t0, int(out["n_accepted"].sum()), flush=True)
t0 = time.time(); out = bode.solve_device(y0, 0.0, 10.0, dyn, record_trajectory=True, **kw); torch.cuda.synchronize(); print("record", time.time() - t0, flush=True)
t0 = time.time(); g0, gw = bode.adjoint_device(out, torch.ones_like(out["ys"])); torch.cuda.synchronize(); print("adjoint", time.time() - t0, flush=True)
t0 = time.time(); g0, gw = bode.adjoint_device(out, torch.ones_like(out["ys"])); torch.cuda.synchronize(); print("adjoint2", time.time() - t0, flush=True)
if len(sys.argv) > 2:
    from paper_2210_12375_b200 import _abi
    lib = _abi.load(); a = out["_args"]; rt = a.traj
    a.traj = None
    t0 = time.time(); _abi.check(lib.bode_solve(_abi.C.byref(a))); torch.cuda.synchronize(); print("rerun plain", time.time() - t0, flush=True)
    a.traj = rt
    t0 = time.time(); _abi.check(lib.bode_solve(_abi.C.byref(a))); torch.cuda.synchronize(); print("rerun rec", time.time() - t0, flush=True)
