"""Probe: fused tcgen05 MLP kernel vs the lockstep tcgen05 path at C4 scale
(per-instance step counts and ys)."""
import sys
sys.path[:0] = ["/root/repo"]
import numpy as np, torch
import bench, paper_2210_12375_b200 as bode
n = int(sys.argv[1])
cfg = bench.make_config("c4", 0, n_override=n)
dev = torch.device("cuda:0")
dyn = bode.mlp_dynamics(*[torch.tensor(w, device=dev) for w in cfg["mlp"]])
kw = dict(t_eval=torch.tensor(cfg["te2d"], device=dev), method="dopri5", atol=1e-6, rtol=1e-6, max_steps=100000)
y0 = torch.tensor(cfg["y0"], device=dev)
a = bode.solve_device(y0, 0.0, 10.0, dyn, mlp_backend="fused", **kw)
b = bode.solve_device(y0, 0.0, 10.0, dyn, mlp_backend="tcgen05", **kw)
d = (a["n_accepted"] != b["n_accepted"]).nonzero().flatten()
print("n", n, "count mismatches", d.numel(), "ys bit-equal", bool((a["ys"] == b["ys"]).all()),
      "first", d[:10].tolist(), a["n_accepted"][d[:5]].tolist(), b["n_accepted"][d[:5]].tolist())
