"""Helpers to load golden fixtures and compare solve results."""
import os

import numpy as np

import scenarios as S

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, "solve", name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def scenario_map():
    """Scenario specs with every input replaced by the golden's stored copy
    (input generation uses NumPy transcendentals whose SIMD paths differ
    across hosts, so inputs are data, not recomputed)."""
    out = {}
    for sc in S.all_solve_scenarios():
        g = load(sc["name"])
        sc = dict(sc)
        sc["y0"], sc["t_start"], sc["t_end"] = g["y0"], g["t_start"], g["t_end"]
        offs = g["te_offs"]
        sc["t_eval"] = [g["te_vals"][offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
        dyn = dict(sc["dyn"])
        if dyn["inst"] is not None:
            dyn["inst"] = g["dyn_inst"]
        sc["dyn"] = dyn
        sc["atol"] = g["atol"] if g["atol"].ndim else float(g["atol"])
        sc["rtol"] = g["rtol"] if g["rtol"].ndim else float(g["rtol"])
        out[sc["name"]] = sc
    return out


def scaled_err(ys_a, ys_b, offs, n_emitted):
    """max_i max|a_i - b_i| / max(|b_i|, tiny) per instance."""
    worst = 0.0
    for i in range(len(n_emitted)):
        m = n_emitted[i]
        if m == 0:
            continue
        a = ys_a[offs[i]:offs[i] + m]
        b = ys_b[offs[i]:offs[i] + m]
        scale = max(np.max(np.abs(b)), 1e-300)
        worst = max(worst, float(np.max(np.abs(a - b)) / scale))
    return worst


def trace_lists(g):
    offs = g["trace_offs"]
    n = len(offs) - 1
    return [(g["trace_t"][offs[i]:offs[i + 1]], g["trace_dt"][offs[i]:offs[i + 1]],
             g["trace_accept"][offs[i]:offs[i + 1]].astype(bool)) for i in range(n)]
