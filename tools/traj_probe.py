"""Probe: consistency of a recorded MLP trajectory (every row written,
cursor in range, t/h finite)."""
import sys
sys.path[:0] = ["/root/repo"]
import numpy as np, torch
import bench, paper_2210_12375_b200 as bode
n = int(sys.argv[1])
cfg = bench.make_config("c4", 0, n_override=n)
dev = torch.device("cuda:0")
junk = torch.full((4 << 20,), float("nan"), dtype=torch.float64, device=dev); del junk  # poison the cache
dyn = bode.mlp_dynamics(*[torch.tensor(w, device=dev) for w in cfg["mlp"]])
kw = dict(t_eval=torch.tensor(cfg["te2d"], device=dev), method="dopri5", atol=1e-6, rtol=1e-6, max_steps=100000)
out = bode.solve_device(torch.tensor(cfg["y0"], device=dev), 0.0, 10.0, dyn, record_trajectory=True, **kw)
tr = out["traj"].cpu().numpy(); toff = out["traj_offsets"].cpu().numpy()
bad = ~np.isfinite(tr[:, :3]).all(1) | (tr[:, 1] <= 0) | (tr[:, 2] < 0) | (tr[:, 2] > 1)
rows = np.nonzero(bad)[0]
inst = np.searchsorted(toff, rows, side="right") - 1
print("n", n, "rows", tr.shape, "bad rows", rows.size, "instances", np.unique(inst)[:10], "k within instance", (rows - toff[inst])[:10])
print("nacc of bad", out["n_accepted"].cpu().numpy()[np.unique(inst)[:10]])
