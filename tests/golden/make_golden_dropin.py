"""Golden fixtures for the drop-in cases (tests/golden/dropin_cases.py),
produced by running the REFERENCE (batchode) on the very same NumPy
callables and user tableaus.  Build container only (needs /root/reference):

    python tests/golden/make_golden_dropin.py

NumPy is pinned to libm pow as in make_golden.py.  Output:
tests/golden/dropin.npz (small).
"""

import os
import sys

os.environ["NPY_DISABLE_CPU_FEATURES"] = (
    "AVX512F AVX512CD AVX512_SKX AVX512_CLX AVX512_CNL AVX512_ICL AVX512_SPR"
)
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import batchode as bo  # noqa: E402
import dropin_cases as DC  # noqa: E402


def tableau(name):
    if name == "dopri5":
        return bo.dopri5()
    if name == "tsit5":
        return bo.tsit5()
    data = DC.bs3_data() if name == "bs3" else DC.ralston_data()
    tab = bo.ButcherTableau(**data)
    tab.validate()
    return tab


def ctrl(betas):
    return bo.PidCoefficients(beta1=betas[0], beta2=betas[1], beta3=betas[2])


def main():
    out = {}
    for name, c in DC.solve_cases():
        n = c["n"]
        f = DC.make_dynamics(c["dyn"], n, np.random.default_rng(1000 + c["seed"]))
        t_start = np.full(n, c["t_start"])
        t_end = np.broadcast_to(np.asarray(c["t_end"], dtype=float), (n,)).copy()
        te = [c["te"].copy() for _ in range(n)]
        prob = bo.IvpBatch(y0=c["y0"], t_start=t_start, t_end=t_end, t_eval=te)
        sol = bo.solve(prob, f, tableau=tableau(c["method"]),
                       tol=bo.Tolerances(c["tol"], c["tol"]), controller=ctrl(c["ctrl"]),
                       max_steps=c["max_steps"], dt0=c["dt0"], record_trace=c["trace"])
        k = f"solve/{name}/"
        out[k + "ys"] = np.concatenate([np.asarray(y).reshape(-1, c["d"]) for y in sol.ys])
        out[k + "n_emitted"] = np.array([len(y) for y in sol.ys], dtype=np.int64)
        out[k + "n_steps"] = sol.stats.n_steps
        out[k + "n_accepted"] = sol.stats.n_accepted
        out[k + "n_f_evals"] = sol.stats.n_f_evals
        out[k + "final_dt"] = sol.stats.final_dt
        out[k + "status"] = sol.status
        if c["trace"]:
            for key in ("trace_t", "trace_dt", "trace_accept"):
                out[k + key] = np.concatenate(sol.stats.extra[key])
        print(name, "steps", int(sol.stats.n_steps.sum()), "statuses", np.bincount(sol.status))

    for name, c in DC.step_cases():
        n = c["n"]
        f = DC.step_dynamics(c["dyn"], n, np.random.default_rng(2000))
        t_end = np.broadcast_to(np.asarray(c["t_end"], dtype=float), (n,)).copy()
        prob = bo.IvpBatch(y0=c["y0"], t_start=np.zeros(n), t_end=t_end,
                           t_eval=[c["te"].copy() for _ in range(n)])
        s = bo.BatchSolver(prob, f, tableau=tableau(c["method"]),
                           tol=bo.Tolerances(c["atol"], c["rtol"]), controller=ctrl(c["ctrl"]),
                           max_steps=c["max_steps"], dt0=c["dt0"], record_trace=True)
        snaps = []
        while True:
            more = s.step_once()
            snaps.append(dict(t=s.t.copy(), y=s.y.copy(), dt=s.ctrl.dt.copy(),
                              norm_prev=s.ctrl.norm_prev.copy(), norm_prev2=s.ctrl.norm_prev2.copy(),
                              n_steps=s.n_steps.copy(), n_accepted=s.n_accepted.copy(),
                              status=s.status.copy(), n_f_evals=np.array(s.n_f_evals),
                              cursor=s._cursor.copy(), fsal_valid=s.fsal_valid.copy()))
            if not more:
                break
        k = f"step/{name}/"
        for key in snaps[0]:
            out[k + key] = np.stack([sn[key] for sn in snaps])
        sol = s.solution()
        out[k + "ys"] = np.concatenate([np.asarray(y).reshape(-1, c["d"]) for y in sol.ys])
        out[k + "trace_accept"] = np.concatenate(sol.stats.extra["trace_accept"])
        print(name, "iterations", len(snaps))

    # Stepper units with a user tableau and traced dynamics (stepper.py:54-139)
    rng = np.random.default_rng(7)
    y = rng.normal(size=(5, 3))
    dt = rng.uniform(0.01, 0.2, size=5)
    t = rng.uniform(0, 1, size=5)
    f = lambda t, y: np.sin(y) + t[:, None]  # noqa: E731  (test_stepper.py:146)
    for tname in ("bs3", "ralston"):
        tab = tableau(tname)
        st = bo.Stepper(tab, 5, 3)
        step = st.step(f, t, dt, y, f(t, y))
        theta = rng.uniform(0, 1, 5)
        k = f"units/{tname}/"
        out[k + "y_next"], out[k + "err"] = step.y_next.copy(), step.error_estimate.copy()
        out[k + "k"] = step.stage_derivs.copy()
        out[k + "theta"] = theta
        out[k + "interp"] = st.interpolate(step, y, dt, theta)
    out["units/y"], out["units/dt"], out["units/t"] = y, dt, t

    # solve_joint with a lambda (test_solver.py:244-257)
    prob = bo.IvpBatch(y0=np.array([[1.0, 2.0], [0.5, -1.0], [2.0, 0.1]]), t_start=np.zeros(3),
                       t_end=np.ones(3), t_eval=[np.array([0.5, 1.0])] * 3)
    sol = bo.solve_joint(prob, lambda t, y: -y)
    out["joint/ys"] = np.stack([np.asarray(y) for y in sol.ys])
    out["joint/n_steps"] = sol.stats.n_steps
    out["joint/n_f_evals"] = sol.stats.n_f_evals
    np.savez_compressed(os.path.join(HERE, "dropin.npz"), **out)
    print("wrote", os.path.join(HERE, "dropin.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
