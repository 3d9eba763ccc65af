"""Debug: distribution of persistent-kernel warp exit times (tail length),
needs a library built with -DBODE_EXIT_PROF (BODE_LIB=...)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2210_12375_b200 as bode
from paper_2210_12375_b200 import _abi
lib = _abi.load()
lib.bode_debug_exit_times.restype = C.c_int
for cname in sys.argv[1:] or ["c2", "c5"]:
    cfg = bench.make_config(cname, 0)
    dev = torch.device("cuda", 0); f64 = dict(dtype=torch.float64, device=dev)
    y0 = torch.tensor(cfg["y0"], **f64); ts = torch.tensor(cfg["t_start"], **f64); tn = torch.tensor(cfg["t_end"], **f64)
    dyn = bode.vdp_dynamics(bode.VdpParams(torch.tensor(cfg["mu"], **f64)))
    kw = {"t_eval": torch.tensor(cfg["te2d"], **f64)} if "te2d" in cfg else {}
    cost = torch.tensor(cfg["cost"], **f64)
    ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"])
    run = lambda: bode.solve_device(y0, ts, tn, dyn, controller=ctrl, max_steps=cfg["max_steps"], cost_hint=cost, mode="fast", **kw)
    run(); torch.cuda.synchronize()
    buf = (C.c_ulonglong * 65536)()
    lib.bode_debug_exit_times(buf, 1)
    run(); torch.cuda.synchronize()
    cnt = lib.bode_debug_exit_times(buf, 1)
    t = np.sort(np.array(buf[:cnt], dtype=np.float64))
    t = (t - t[0]) / 1e3  # us since the first warp exit
    span = t[-1]
    print(f"{cname}: {cnt} warps; exit spread {span:.1f} us; quantiles (us after first exit): "
          + " ".join(f"p{q}={np.percentile(t, q):.1f}" for q in (10, 50, 90, 99)))
