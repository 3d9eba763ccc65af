"""Map scenario registry specs onto the product's device dynamics."""
import numpy as np

import paper_2210_12375_b200 as bode
import paper_2210_12375_b200.dynamics as D


def device_dynamics(spec):
    name, inst, sh = spec["name"], spec["inst"], spec["shared"]
    slots = D.SLOTS[name]
    params = {}
    ninst = 0 if inst is None else inst.shape[1]
    for k, s in enumerate(slots):
        params[s] = inst[:, k] if k < ninst else sh[k - ninst]
    if name == "mlp":
        return bode.mlp_dynamics(*spec["mlp"])
    return D.DeviceDynamics(name, params)


def controller(c):
    b1, b2, b3 = c["betas"]
    return bode.PidCoefficients(beta1=b1, beta2=b2, beta3=b3, safety=c["safety"],
                                factor_min=c["factor_min"], factor_max=c["factor_max"],
                                update_history_on_reject=c["hist"])


def tableau(method):
    return {"dopri5": bode.dopri5, "tsit5": bode.tsit5, "heun": bode.heun}[method]()


def solve_scenario(sc, **kw):
    prob = bode.IvpBatch(sc["y0"], sc["t_start"], sc["t_end"], sc["t_eval"])
    return bode.solve(prob, device_dynamics(sc["dyn"]), tableau=tableau(sc["method"]),
                      tol=bode.Tolerances(sc["atol"], sc["rtol"]),
                      controller=controller(sc["ctrl"]), max_steps=sc["max_steps"],
                      dt0=sc["dt0"], record_trace=sc["trace"], **kw)


def flat_ys(sol, te_offs, d):
    """Solution.ys (ragged) -> golden layout (te rows, NaN where absent)."""
    out = np.full((te_offs[-1], d), np.nan)
    for i, y in enumerate(sol.ys):
        out[te_offs[i]:te_offs[i] + y.shape[0]] = y
    return out
