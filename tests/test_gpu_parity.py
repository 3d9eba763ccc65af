"""CUDA path vs the reference's golden vectors (and the pinned oracle).

Parity bar (north_star / SURVEY.md §8(c)): identical per-instance status,
n_steps, n_accepted, n_emitted and batch-global n_f_evals; ys within
1e-10 of each instance's max |y| (scaled, because pointwise relative error
is ill-posed at zero crossings); final_dt within 1e-10 relative.  Exact
mode also reports how many instances are bit-identical.
"""
import numpy as np
import pytest

import devspec
import golden_io as G

pytestmark = pytest.mark.gpu
SCENARIOS = G.scenario_map()
YS_TOL = 1e-10


def compare(sol, g, sc, ys_tol=YS_TOL):
    d = sc["y0"].shape[1]
    assert np.array_equal(sol.status, g["status"]), "status"
    assert np.array_equal(sol.stats.n_steps, g["n_steps"]), "n_steps"
    assert np.array_equal(sol.stats.n_accepted, g["n_accepted"]), "n_accepted"
    assert np.array_equal(sol.n_emitted, g["n_emitted"]), "n_emitted"
    assert np.all(sol.stats.n_f_evals == g["n_f_evals"][0]), "n_f_evals"
    ys = devspec.flat_ys(sol, g["te_offs"], d)
    assert np.array_equal(np.isnan(ys), np.isnan(g["ys"]))
    err = G.scaled_err(np.nan_to_num(ys), np.nan_to_num(g["ys"]), g["te_offs"], g["n_emitted"])
    assert err <= ys_tol, f"scaled ys error {err:.3e}"
    fd = np.abs(sol.stats.final_dt - g["final_dt"]) <= ys_tol * np.abs(g["final_dt"])
    assert np.all(fd | (g["final_dt"] == 0)), "final_dt"
    return err


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_solve_matches_reference_golden(name):
    sc = SCENARIOS[name]
    g = G.load(name)
    sol = devspec.solve_scenario(sc)
    compare(sol, g, sc)
    if sc["trace"]:
        for i, (tt, tdt, tacc) in enumerate(G.trace_lists(g)):
            assert np.array_equal(sol.stats.extra["trace_accept"][i], tacc)
            np.testing.assert_allclose(sol.stats.extra["trace_dt"][i], tdt, rtol=1e-10, atol=0)
            np.testing.assert_allclose(sol.stats.extra["trace_t"][i], tt, rtol=1e-10, atol=1e-300)


@pytest.mark.parametrize("name", ["c1_vdp", "c2_vdp_pi42", "c3_lorenz", "c5_vdp_stiff"])
def test_fast_mode_within_tolerance(name):
    """FMA-contracted mode: same step counts, ys within the same bar."""
    sc = SCENARIOS[name]
    g = G.load(name)
    sol = devspec.solve_scenario(sc, mode="fast")
    compare(sol, g, sc)
