"""The device-side sharded-solve helpers with a real NCCL process group
(world size 1 on the one-GPU test box; the multi-rank logic is covered by
tests/test_distributed.py with gloo and tools/multirank_check.sh)."""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2210_12375_b200 as bode
from paper_2210_12375_b200 import distributed as D

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_global_f_evals_device_and_gather(nccl_group):
    rng = np.random.default_rng(4)
    n = 5000
    mu = rng.uniform(1.0, 10.0, n)
    t_end = rng.uniform(5.0, 20.0, n)
    f64 = dict(dtype=torch.float64, device="cuda")
    out = bode.solve_device(torch.tensor(np.tile([2.0, 0.0], (n, 1)), **f64),
                            torch.zeros(n, **f64), torch.tensor(t_end, **f64),
                            bode.vdp_dynamics(bode.VdpParams(torch.tensor(mu, **f64))),
                            t_eval=torch.tensor(t_end[:, None], **f64),
                            controller=bode.pid_controller("PI42"), with_refresh_map=True)
    nfe = D.global_f_evals_device(out)
    assert int(nfe) == int(out["n_f_evals"][0])  # one shard == the unsharded count
    g = D.gather_device(out, dst=0)
    for k in ("n_steps", "n_accepted", "final_dt", "status", "n_emitted", "ys"):
        assert torch.equal(g[k], out[k].contiguous()), k


def test_solve_sharded_over_nccl_equals_unsharded(nccl_group):
    rng = np.random.default_rng(5)
    n = 3000
    mu = rng.uniform(1.0, 10.0, n)
    t_end = rng.uniform(5.0, 20.0, n)
    prob = bode.IvpBatch(np.tile([2.0, 0.0], (n, 1)), np.zeros(n), t_end, t_end[:, None])
    f = bode.vdp_dynamics(bode.VdpParams(mu))
    ref = bode.solve(prob, f, controller=bode.pid_controller("PI42"))
    sol = D.solve_sharded(prob, f, cost_hint=mu * t_end, controller=bode.pid_controller("PI42"))
    assert np.array_equal(sol.stats.n_steps, ref.stats.n_steps)
    assert np.array_equal(sol.stats.n_f_evals, ref.stats.n_f_evals)
    assert np.array_equal(sol.ys_flat, ref.ys_flat)
