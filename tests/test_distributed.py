"""Multi-rank host logic (no GPU): partition, the global n_f_evals exchange
and the gather, run as world_size-2 gloo processes with the pinned oracle as
each rank's shard solver.  The sharded result must equal the unsharded
reference solve bit for bit (batch independence)."""
import os
import socket

import numpy as np
import pytest

import golden_io as G
import oracle as O
import paper_2210_12375_b200 as bode
from paper_2210_12375_b200 import distributed as D
from paper_2210_12375_b200.dynamics import SLOTS


def oracle_shard_solve(problem, f, tableau=None, tol=None, controller=None, max_steps=10_000,
                       dt0=None, with_refresh_map=False, **_):
    """Adapter: bode.solve's signature, computed by the CPU oracle."""
    inst = [np.asarray(f.params[s], float) for s in SLOTS[f.kind] if np.ndim(f.params[s])]
    shared = [float(f.params[s]) for s in SLOTS[f.kind] if not np.ndim(f.params[s])]
    dyn = dict(name=f.kind, inst=np.stack(inst, 1) if inst else None, shared=shared)
    c = controller or bode.integral_controller()
    tol = tol or bode.Tolerances()
    method = tableau.method if tableau is not None else "dopri5"
    n = problem.batch_size
    o = problem.te_offsets
    te = [problem.te_values[o[i]:o[i + 1]] for i in range(n)]
    r = O.solve(problem.y0, problem.t_start, problem.t_end, te, dyn, method=method,
                atol=tol.atol, rtol=tol.rtol, max_steps=max_steps, dt0=dt0, nthreads=2,
                ctrl=dict(betas=(c.beta1, c.beta2, c.beta3), safety=c.safety,
                          factor_min=c.factor_min, factor_max=c.factor_max,
                          hist=c.update_history_on_reject), with_refresh=True)
    stats = bode.SolveStats(n_steps=r["n_steps"], n_accepted=r["n_accepted"],
                            n_f_evals=np.full(n, r["n_f_evals"][0]), final_dt=r["final_dt"],
                            extra=dict(max_iterations=int(r["max_iterations"][0]),
                                       refresh_map=r["refresh_map"]))
    return bode.Solution(r["ys"], r["te_offs"], 0, r["n_emitted"], stats,
                         r["status"].astype(np.int64), problem.n_features)


def test_partition_covers_and_balances():
    rng = np.random.default_rng(0)
    cost = np.exp(rng.uniform(0, np.log(1000), 10_000))
    for world in (1, 2, 3, 8):
        parts = D.partition(10_000, world, cost)
        allidx = np.concatenate(parts)
        assert np.array_equal(np.sort(allidx), np.arange(10_000))
        loads = [cost[p].sum() for p in parts]
        assert max(loads) - min(loads) <= cost.max() + 1e-9
        plain = D.partition(10_000, world)
        assert np.array_equal(np.concatenate(plain), np.arange(10_000))


def test_combine_f_evals_matches_unsharded():
    """n_f_evals of a batch rebuilt from two half-batch solves equals the
    reference's batch-global count (golden C2 prefix)."""
    sc = G.scenario_map()["c2_vdp_pi42"]
    g = G.load("c2_vdp_pi42")
    prob = bode.IvpBatch(sc["y0"], sc["t_start"], sc["t_end"], sc["t_eval"])
    f = bode.vdp_dynamics(bode.VdpParams(sc["dyn"]["inst"][:, 0]))
    maxes, maps = [], []
    for idx in D.partition(prob.batch_size, 2):
        s = oracle_shard_solve(D.subset_problem(prob, idx), f.subset(idx),
                               controller=bode.pid_controller("PI42"), with_refresh_map=True)
        maxes.append(s.stats.extra["max_iterations"])
        maps.append(s.stats.extra["refresh_map"])
    assert D.combine_f_evals(maxes, maps, 7, True) == g["n_f_evals"][0]
    assert D.combine_f_evals([5, 9], [np.zeros(12)] * 2, 2, False) == 1 + 2 * 9


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = G.scenario_map()[name]
        prob = bode.IvpBatch(sc["y0"], sc["t_start"], sc["t_end"], sc["t_eval"])
        inst = sc["dyn"]["inst"]
        f = bode.vdp_dynamics(bode.VdpParams(inst[:, 0]))
        c = sc["ctrl"]
        ctrl = bode.PidCoefficients(*c["betas"], c["safety"], c["factor_min"], c["factor_max"],
                                    c["hist"])
        tab = {"dopri5": bode.dopri5, "tsit5": bode.tsit5, "heun": bode.heun}[sc["method"]]()
        sol = D.solve_sharded(prob, f, cost_hint=inst[:, 0] * np.abs(sc["t_end"]), gather_to=0,
                              shard_solve=oracle_shard_solve, tableau=tab,
                              tol=bode.Tolerances(sc["atol"], sc["rtol"]), controller=ctrl,
                              max_steps=sc["max_steps"])
        if rank == 0:
            np.savez(out, ys=sol.ys_flat, n_steps=sol.stats.n_steps,
                     n_accepted=sol.stats.n_accepted, n_f_evals=sol.stats.n_f_evals,
                     final_dt=sol.stats.final_dt, status=sol.status, n_emitted=sol.n_emitted)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2_vdp_pi42", "c1_vdp", "heun_vdp"])
def test_gloo_world2_sharded_equals_reference(name, tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
    r = np.load(out)
    g = G.load(name)
    assert np.array_equal(r["status"], g["status"])
    assert np.array_equal(r["n_steps"], g["n_steps"])
    assert np.array_equal(r["n_accepted"], g["n_accepted"])
    assert np.array_equal(r["n_emitted"], g["n_emitted"])
    assert np.all(r["n_f_evals"] == g["n_f_evals"][0])
    assert np.array_equal(r["final_dt"], g["final_dt"])
    assert np.array_equal(r["ys"], g["ys"], equal_nan=True)
