"""Generate the golden fixtures by running the REFERENCE (batchode) here.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    python tests/golden/make_golden.py

The reference is imported read-only from ``/root/reference/pkg/src``.
NumPy's AVX-512 SVML ``pow`` differs from glibc ``pow`` in ~5% of inputs
(SURVEY.md finding 1); pinning ``NPY_DISABLE_CPU_FEATURES`` before NumPy is
imported makes the reference use libm, the same ``pow`` the C oracle calls,
so the fixtures are reproducible bit for bit.

Outputs (committed, small):
  tests/golden/solve/<scenario>.npz   full solves (inputs + ys/stats/status/trace)
  tests/golden/units.npz              rk_step / interpolate / error_norm /
                                      adapt_step / initial_step vectors
  tests/golden/tableaus.npz           the reference's dopri5/tsit5 coefficients
"""

import os
import sys

os.environ["NPY_DISABLE_CPU_FEATURES"] = (
    "AVX512F AVX512CD AVX512_SKX AVX512_CLX AVX512_CNL AVX512_ICL AVX512_SPR"
)
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import batchode as bo  # noqa: E402
import scenarios as S  # noqa: E402


def tableau(method):
    if method == "dopri5":
        return bo.dopri5()
    if method == "tsit5":
        return bo.tsit5()
    if method == "heun":
        h = S.heun_tableau_data()
        tab = bo.ButcherTableau(**h)
        tab.validate()
        return tab
    raise KeyError(method)


def controller(c):
    b1, b2, b3 = c["betas"]
    return bo.PidCoefficients(beta1=b1, beta2=b2, beta3=b3, safety=c["safety"],
                              factor_min=c["factor_min"], factor_max=c["factor_max"],
                              update_history_on_reject=c["hist"])


def csr(arrs, d=None):
    lens = np.array([len(a) for a in arrs], dtype=np.int64)
    offs = np.zeros(len(arrs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    if d is None:
        vals = np.concatenate([np.asarray(a, float) for a in arrs]) if offs[-1] else np.empty(0)
    else:
        vals = (np.concatenate([np.asarray(a, float).reshape(-1, d) for a in arrs])
                if offs[-1] else np.empty((0, d)))
    return vals, offs


def run_scenario(sc):
    n = sc["y0"].shape[0]
    problem = bo.IvpBatch(y0=sc["y0"], t_start=sc["t_start"], t_end=sc["t_end"],
                          t_eval=sc["t_eval"])
    f = S.numpy_dynamics(sc["dyn"], n)
    tol = bo.Tolerances(atol=sc["atol"], rtol=sc["rtol"])
    sol = bo.solve(problem, f, tableau=tableau(sc["method"]), tol=tol,
                   controller=controller(sc["ctrl"]), max_steps=sc["max_steps"],
                   dt0=sc["dt0"], record_trace=sc["trace"])
    d = sc["y0"].shape[1]
    te_vals, te_offs = csr(sc["t_eval"])
    ys = np.full((te_offs[-1], d), np.nan)
    n_emitted = np.zeros(n, dtype=np.int64)
    for i in range(n):
        m = sol.ys[i].shape[0]
        ys[te_offs[i]:te_offs[i] + m] = sol.ys[i]
        n_emitted[i] = m
    spec = sc["dyn"]
    out = dict(
        y0=sc["y0"], t_start=sc["t_start"], t_end=sc["t_end"],
        dyn_inst=spec["inst"] if spec["inst"] is not None else np.zeros((0, 0)),
        atol=np.asarray(sc["atol"], float), rtol=np.asarray(sc["rtol"], float),
        te_vals=te_vals, te_offs=te_offs,
        ys=ys, n_emitted=n_emitted,
        n_steps=sol.stats.n_steps, n_accepted=sol.stats.n_accepted,
        n_f_evals=sol.stats.n_f_evals, final_dt=sol.stats.final_dt,
        status=sol.status,
    )
    if sc["trace"]:
        for key in ("trace_t", "trace_dt", "trace_accept"):
            vals, offs = csr(sol.stats.extra[key])
            out[key] = vals
        out["trace_offs"] = offs
    return out


def unit_vectors():
    rng = np.random.default_rng(123)
    out = {}
    # rk_step + interpolate on three tableaus x three dynamics
    for method in ("dopri5", "tsit5", "heun"):
        tab = tableau(method)
        for dname, d, spec in (
            ("vdp", 2, S.dyn("vdp", rng.uniform(0.5, 20.0, 16))),
            ("lorenz", 3, S.dyn("lorenz", None, (10.0, 28.0, 8.0 / 3.0))),
            ("sin_plus_t", 3, S.dyn("sin_plus_t")),
        ):
            n = 16
            f = S.numpy_dynamics(spec, n)
            t = rng.uniform(0.0, 1.0, n)
            dt = rng.uniform(0.001, 0.3, n)
            dt[0] = 0.0
            y = rng.normal(size=(n, d))
            f0 = np.asarray(f(t, y), float)
            st = bo.rk_step(f, tab, t, dt, y, f0)
            theta = rng.uniform(0.0, 1.0, n)
            theta[1], theta[2] = 0.0, 1.0
            yi = bo.interpolate(st, tab, y, dt, theta)
            key = f"rk_{method}_{dname}"
            out[key + "_t"] = t
            out[key + "_dt"] = dt
            out[key + "_y"] = y
            out[key + "_f0"] = f0
            out[key + "_ynext"] = st.y_next
            out[key + "_err"] = st.error_estimate
            out[key + "_k"] = st.stage_derivs.copy()
            out[key + "_theta"] = theta
            out[key + "_interp"] = yi
            if dname == "vdp":
                out[key + "_mu"] = spec["inst"][:, 0]
    # error_norm, several widths (numpy pairwise order from d >= 8)
    for d in (1, 2, 3, 4, 7, 8, 9, 16, 64, 130, 300):
        n = 32
        err = rng.normal(scale=1e-6, size=(n, d))
        y0 = rng.normal(size=(n, d))
        y1 = y0 + rng.normal(scale=1e-3, size=(n, d))
        err[0, 0] = np.nan if d > 1 else err[0, 0]
        atol = rng.uniform(1e-8, 1e-5, n)
        rtol = rng.uniform(1e-8, 1e-5, n)
        out[f"norm_d{d}_err"] = err
        out[f"norm_d{d}_y0"] = y0
        out[f"norm_d{d}_y1"] = y1
        out[f"norm_d{d}_atol"] = atol
        out[f"norm_d{d}_rtol"] = rtol
        out[f"norm_d{d}_scalar"] = bo.error_norm(err, y0, y1, bo.Tolerances(1e-6, 1e-7))
        out[f"norm_d{d}_vector"] = bo.error_norm(err, y0, y1, bo.Tolerances(atol, rtol))
    # adapt_step: 200 random norm sequences per controller, 60 attempts each
    for cname, betas, hist in (("I", S.ICTRL, True), ("PI42", S.PI42, True),
                               ("H312", S.H312, True), ("H312n", S.H312, False),
                               ("H211", (1 / 6, 1 / 6, 0.0), True)):
        coeffs = bo.PidCoefficients(beta1=betas[0], beta2=betas[1], beta3=betas[2],
                                    update_history_on_reject=hist)
        n, T = 64, 60
        norms = 10.0 ** rng.uniform(-12.0, 3.0, size=(T, n))
        norms[5, 0] = np.inf
        norms[7, 1] = 0.0
        dt0 = rng.uniform(1e-3, 1.0, n)
        state = bo.ControllerState.initial(dt0)
        acc_all, dt_all, p1, p2 = [], [], [], []
        for j in range(T):
            acc, dtn = bo.adapt_step(state, norms[j], 4, coeffs)
            acc_all.append(acc.copy())
            dt_all.append(dtn.copy())
            p1.append(state.norm_prev.copy())
            p2.append(state.norm_prev2.copy())
        out[f"adapt_{cname}_norms"] = norms
        out[f"adapt_{cname}_dt0"] = dt0
        out[f"adapt_{cname}_accept"] = np.array(acc_all)
        out[f"adapt_{cname}_dt"] = np.array(dt_all)
        out[f"adapt_{cname}_prev"] = np.array(p1)
        out[f"adapt_{cname}_prev2"] = np.array(p2)
    # initial_step: vdp / lorenz / zero / inf-threshold, both directions
    for dname, d, spec, order in (
        ("vdp", 2, S.dyn("vdp", rng.uniform(0.5, 50.0, 32)), 5),
        ("lorenz", 3, S.dyn("lorenz", None, (10.0, 28.0, 8.0 / 3.0)), 5),
        ("zero", 2, S.dyn("zero"), 5),
        ("square", 1, S.dyn("square", None, (0.4,)), 2),
    ):
        n = 32
        f = S.numpy_dynamics(spec, n)
        t0 = rng.uniform(-1.0, 1.0, n)
        y0 = rng.normal(size=(n, d))
        if dname == "zero":
            y0[0] = 0.0
        direction = np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)
        atol = rng.uniform(1e-9, 1e-4, n)
        rtol = rng.uniform(1e-9, 1e-4, n)
        dt, f0 = bo.initial_step(f, t0, y0, order, bo.Tolerances(atol, rtol), direction)
        key = f"init_{dname}"
        out[key + "_t0"] = t0
        out[key + "_y0"] = y0
        out[key + "_dir"] = direction
        out[key + "_atol"] = atol
        out[key + "_rtol"] = rtol
        out[key + "_order"] = np.array(order)
        out[key + "_dt"] = dt
        out[key + "_f0"] = f0
        if spec["inst"] is not None:
            out[key + "_mu"] = spec["inst"][:, 0]
    return out


def mlp_golden(n=64):
    W1, b1, W2, b2 = S.c4_weights()
    y0 = S.c4_y0(n)

    def f(t, y):
        h = np.tanh(y.astype(np.float32) @ W1.T + b1)
        return (h @ W2.T + b2).astype(np.float64)

    problem = bo.IvpBatch(y0=y0, t_start=np.zeros(n), t_end=np.full(n, 10.0),
                          t_eval=[np.array([10.0])] * n)
    sol = bo.solve(problem, f, tol=bo.Tolerances(1e-6, 1e-6), max_steps=100_000)
    ys = np.stack([s[-1] for s in sol.ys])
    return dict(W1=W1, b1=b1, W2=W2, b2=b2, y0=y0, ys=ys, n_steps=sol.stats.n_steps,
                n_accepted=sol.stats.n_accepted, status=sol.status,
                n_f_evals=sol.stats.n_f_evals)


def run_joint(sc, problem=None):
    """batchode.solve_joint on a scenario; stores inputs and outputs."""
    n, d = sc["y0"].shape
    if problem is None:
        problem = bo.IvpBatch(y0=sc["y0"], t_start=sc["t_start"], t_end=sc["t_end"],
                              t_eval=sc["t_eval"])
    f = S.numpy_dynamics(sc["dyn"], n)
    tol = bo.Tolerances(atol=sc["atol"], rtol=sc["rtol"])
    sol = bo.solve_joint(problem, f, tableau=tableau(sc["method"]), tol=tol,
                         controller=controller(sc["ctrl"]), max_steps=sc["max_steps"],
                         dt0=sc["dt0"], record_trace=sc["trace"])
    te0 = np.asarray(problem.t_eval[0], float)
    ys = np.full((n, te0.size, d), np.nan)
    n_emitted = np.zeros(n, dtype=np.int64)
    for i in range(n):
        ys[i, :sol.ys[i].shape[0]] = sol.ys[i]
        n_emitted[i] = sol.ys[i].shape[0]
    spec = sc["dyn"]
    c = sc["ctrl"]
    out = dict(
        y0=problem.y0, t_start=problem.t_start, t_end=problem.t_end, te=te0,
        dyn_name=np.array(spec["name"]),
        dyn_inst=spec["inst"] if spec["inst"] is not None else np.zeros((0, 0)),
        dyn_shared=np.array(spec["shared"], float), method=np.array(sc["method"]),
        atol=np.asarray(sc["atol"], float), rtol=np.asarray(sc["rtol"], float),
        betas=np.array(c["betas"], float), hist=np.array(c["hist"]),
        max_steps=np.array(sc["max_steps"]), dt0=np.array(np.nan if sc["dt0"] is None else sc["dt0"]),
        trace=np.array(sc["trace"]),
        ys=ys, n_emitted=n_emitted, n_steps=sol.stats.n_steps, n_accepted=sol.stats.n_accepted,
        n_f_evals=sol.stats.n_f_evals, final_dt=sol.stats.final_dt, status=sol.status,
    )
    if sc["trace"]:
        for key in ("trace_t", "trace_dt", "trace_accept"):
            out[key] = np.asarray(sol.stats.extra[key][0])
    return out


def joint_goldens():
    os.makedirs(os.path.join(HERE, "joint"), exist_ok=True)
    scs = list(S.joint_scenarios())
    # the paper's pathology (tests/test_acceptance.py:103-113): 4 VdP on the
    # mu = 25 limit cycle, tol 1e-5; inputs from the reference's vdp_batch
    batch = bo.vdp_batch(4, 25.0)
    path = S._scn("joint_pathology_vdp4_mu25", batch.y0, batch.t_start, batch.t_end,
                  batch.t_eval, S.dyn("vdp", np.full(4, 25.0)), atol=1e-5, rtol=1e-5,
                  max_steps=1_000_000)
    for sc in scs + [path]:
        out = run_joint(sc, batch if sc is path else None)
        if sc is path:  # the independent solve, for the step ratio
            ind = bo.solve(batch, S.numpy_dynamics(sc["dyn"], 4), tol=bo.Tolerances(1e-5, 1e-5),
                           max_steps=1_000_000)
            out["independent_n_steps"] = ind.stats.n_steps
        np.savez_compressed(os.path.join(HERE, "joint", sc["name"] + ".npz"), **out)
        print(f"{sc['name']:28s} n={sc['y0'].shape[0]:4d} steps={out['n_steps'][0]:6d} "
              f"status={out['status'][0]} nfe={out['n_f_evals'][0]}")


CLI_RUNS = {
    # name: reference cli argv (output paths appended); compared by tests/test_gpu_cli.py
    "vdp_ind": ["vdp-batching", "--n", "4", "--mu", "25"],
    "vdp_joint": ["vdp-batching", "--n", "4", "--mu", "25", "--mode", "joint"],
    "vdp_random_tsit5_pi42": ["vdp-batching", "--n", "6", "--mu", "5", "--random-phases", "--seed",
                              "3", "--controller", "pid:PI42", "--method", "tsit5", "--n-eval", "0"],
    "pid_sweep": ["pid-sweep", "--mu", "5,25"],
}


def cli_goldens():
    """Run the reference CLI (cli.py) and keep its CSV output, plus the batch
    builders' arrays (problems.py:53-143)."""
    import batchode.cli as bcli
    out_dir = os.path.join(HERE, "cli")
    os.makedirs(out_dir, exist_ok=True)
    for name, argv in CLI_RUNS.items():
        extra = ["--out", os.path.join(out_dir, name + ".csv")]
        if argv[0] == "vdp-batching":
            extra += ["--trace-out", os.path.join(out_dir, name + "_trace.csv")]
        rc = bcli.main(argv + extra)
        print(f"cli {name}: rc={rc}")
    anchor, period = bo.vdp_limit_cycle(25.0)
    batch = bo.vdp_batch(4, 25.0, n_eval=5)
    np.savez_compressed(os.path.join(out_dir, "problems.npz"), anchor=np.array(anchor),
                        period=np.array(period), y0=batch.y0, t_end=batch.t_end,
                        t_eval=np.array(batch.t_eval))


def main():
    joint_goldens()
    cli_goldens()
    os.makedirs(os.path.join(HERE, "solve"), exist_ok=True)
    for sc in S.all_solve_scenarios():
        out = run_scenario(sc)
        np.savez_compressed(os.path.join(HERE, "solve", sc["name"] + ".npz"), **out)
        print(f"{sc['name']:24s} n={sc['y0'].shape[0]:5d} steps={out['n_steps'].sum():8d} "
              f"status={np.bincount(out['status'], minlength=5).tolist()} "
              f"nfe={out['n_f_evals'][0]}")
    np.savez_compressed(os.path.join(HERE, "units.npz"), **unit_vectors())
    tabs = {}
    for m in ("dopri5", "tsit5"):
        t = tableau(m)
        for k in ("a", "b", "b_err", "c", "interp_coeffs"):
            tabs[f"{m}_{k}"] = getattr(t, k)
    np.savez_compressed(os.path.join(HERE, "tableaus.npz"), **tabs)
    np.savez_compressed(os.path.join(HERE, "mlp.npz"), **mlp_golden())
    print("mlp done")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "joint":
        joint_goldens()
    elif len(sys.argv) > 1 and sys.argv[1] == "cli":
        cli_goldens()
    else:
        main()
