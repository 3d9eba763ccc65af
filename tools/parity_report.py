"""Parity report: CUDA path vs reference golden vectors and vs the oracle at
full C2 scale -- step-count identity, scaled ys error, bit-identical share.
Run on the GPU box:  python tools/parity_report.py [--mode exact|fast]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden"),
                os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402

import devspec  # noqa: E402
import golden_io as G  # noqa: E402
import oracle as O  # noqa: E402
import paper_2210_12375_b200 as bode  # noqa: E402
import scenarios as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="exact")
    ap.add_argument("--skip-1m", action="store_true")
    args = ap.parse_args()
    print(f"| scenario | n | steps identical | ys scaled err | bit-identical ys | bit-identical final_dt |")
    print("|---|---|---|---|---|---|")
    for name, sc in sorted(G.scenario_map().items()):
        g = G.load(name)
        sol = devspec.solve_scenario(sc, mode=args.mode)
        same_steps = np.array_equal(sol.stats.n_steps, g["n_steps"]) and np.array_equal(
            sol.stats.n_accepted, g["n_accepted"])
        ys = devspec.flat_ys(sol, g["te_offs"], sc["y0"].shape[1])
        em = np.minimum(g["n_emitted"], sol.n_emitted)
        err = G.scaled_err(np.nan_to_num(ys), np.nan_to_num(g["ys"]), g["te_offs"], em)
        offs = g["te_offs"]
        bit = np.mean([np.array_equal(ys[offs[i]:offs[i + 1]], g["ys"][offs[i]:offs[i + 1]],
                                      equal_nan=True) for i in range(len(offs) - 1)])
        bfd = np.mean(sol.stats.final_dt == g["final_dt"])
        print(f"| {name} | {len(g['status'])} | {same_steps} | {err:.2e} | {bit:.1%} | {bfd:.1%} |")
    if args.skip_1m:
        return
    mu, t_end = S.c2_inputs()
    n = mu.shape[0]
    y0 = np.tile([2.0, 0.0], (n, 1))
    sol = bode.solve(bode.IvpBatch(y0, np.zeros(n), t_end, t_end[:, None]),
                     bode.vdp_dynamics(bode.VdpParams(mu)), controller=bode.pid_controller("PI42"),
                     cost_hint=mu * t_end, mode=args.mode)
    ref = O.solve(y0, 0.0, t_end, [np.array([x]) for x in t_end], dict(name="vdp", inst=mu[:, None]),
                  ctrl=dict(betas=S.PI42, safety=0.9, factor_min=0.2, factor_max=10.0, hist=True))
    a, b = sol.ys_flat.reshape(n, -1), ref["ys"].reshape(n, -1)
    err = np.max(np.abs(a - b).max(axis=1) / np.abs(b).max(axis=1))
    print(f"C2 instances with a different n_steps: {int(np.sum(sol.stats.n_steps != ref['n_steps']))}, "
          f"n_accepted: {int(np.sum(sol.stats.n_accepted != ref['n_accepted']))}")
    print(f"\nC2 full scale (n={n}, vs oracle): status identical "
          f"{np.array_equal(sol.status, ref['status'])}, n_steps identical "
          f"{np.array_equal(sol.stats.n_steps, ref['n_steps'])}, n_accepted identical "
          f"{np.array_equal(sol.stats.n_accepted, ref['n_accepted'])}, n_f_evals "
          f"{sol.stats.n_f_evals[0]} vs {ref['n_f_evals'][0]}, max scaled ys err {err:.2e}, "
          f"bit-identical ys {np.mean(np.all(a == b, axis=1)):.2%}, bit-identical final_dt "
          f"{np.mean(sol.stats.final_dt == ref['final_dt']):.2%}")


if __name__ == "__main__" and "--extra" not in sys.argv:
    main()


def full_scale_extra(mode):
    """C5 (stiff VdP, 1M) and C3 (Lorenz tsit5 1e-8, 256K, 1000 points) at
    full size vs the oracle: per-instance step-count mismatches, scaled ys."""
    sys.path.insert(0, ROOT)
    import bench
    for name in ("c5", "c3"):
        cfg = bench.make_config(name, 0)
        n = cfg["n"]
        te = cfg.get("te1d")
        dyn = (bode.vdp_dynamics(bode.VdpParams(cfg["mu"])) if cfg["dyn"] == "vdp"
               else bode.lorenz_dynamics())
        tab = {"dopri5": bode.dopri5, "tsit5": bode.tsit5}[cfg["method"]]()
        ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"])
        sol = bode.solve(bode.IvpBatch(cfg["y0"], cfg["t_start"], cfg["t_end"],
                                       te if te is not None else [np.empty(0)] * n),
                         dyn, tableau=tab, tol=bode.Tolerances(cfg["tol"], cfg["tol"]),
                         controller=ctrl, max_steps=cfg["max_steps"], mode=mode,
                         cost_hint=cfg["cost"])
        odyn = (dict(name="vdp", inst=cfg["mu"][:, None]) if cfg["dyn"] == "vdp"
                else dict(name="lorenz", inst=None, shared=(10.0, 28.0, 8.0 / 3.0)))
        ref = O.solve(cfg["y0"], cfg["t_start"], cfg["t_end"], te, odyn, method=cfg["method"],
                      atol=cfg["tol"], rtol=cfg["tol"], ctrl=cfg["ctrl"], max_steps=cfg["max_steps"],
                      nthreads=os.cpu_count())
        ds = int(np.sum(sol.stats.n_steps != ref["n_steps"]))
        da = int(np.sum(sol.stats.n_accepted != ref["n_accepted"]))
        msg = ""
        if te is not None:
            a, b = sol.ys_flat.reshape(n, -1), ref["ys"].reshape(n, -1)
            msg = f", max scaled ys err {np.max(np.abs(a - b).max(axis=1) / np.abs(b).max(axis=1)):.2e}"
        print(f"{name} full scale (n={n}, mode={mode}, vs oracle): status identical "
              f"{np.array_equal(sol.status, ref['status'])}, instances with different n_steps {ds}, "
              f"n_accepted {da}, n_f_evals {sol.stats.n_f_evals[0]} vs {ref['n_f_evals'][0]}{msg}")


if __name__ == "__main__" and "--extra" in sys.argv:
    full_scale_extra(sys.argv[sys.argv.index("--extra") + 1])
