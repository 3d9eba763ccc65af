"""The device-side sharded solve (distributed.solve_sharded_device: device
shard plan, shard gathers, per-shard persistent solve, n_f_evals
all-reduce, gather to rank 0 in batch order) against the unsharded solve:
world size 1 over a real NCCL group, and 2 / 3 ranks sharing the one GPU
of the test box over gloo (bitwise equal per instance, reference
tests/test_solver.py:140-168)."""
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


def test_solve_sharded_device_world1_equals_solve_device(nccl_group):
    rng = np.random.default_rng(6)
    n = 4099
    f64 = dict(dtype=torch.float64, device="cuda")
    mu = torch.tensor(rng.uniform(1.0, 10.0, n), **f64)
    t_end = torch.tensor(rng.uniform(5.0, 20.0, n), **f64)
    y0 = torch.tensor(np.tile([2.0, 0.0], (n, 1)), **f64)
    f = bode.vdp_dynamics(bode.VdpParams(mu))
    kw = dict(controller=bode.pid_controller("PI42"), mode="fast")
    ref = bode.solve_device(y0, torch.zeros(n, **f64), t_end, f, t_eval=t_end[:, None], **kw)
    got = D.solve_sharded_device(y0, 0.0, t_end, f, t_eval=t_end[:, None], cost_hint=mu * t_end, **kw)
    for k in ("n_steps", "n_accepted", "final_dt", "status", "n_emitted", "ys", "n_f_evals"):
        assert torch.equal(got[k], ref[k]), k


# ---------------------------------------------------------------- N > 1 --
# The box has one GPU and NCCL refuses two ranks on one device, so the
# multi-rank device path runs with W processes sharing cuda:0 over a gloo
# group (collectives on host copies, distributed._on_backend); the plan,
# the shard gathers, the persistent kernels and the batch-order scatter are
# the same code the NCCL path runs.
def _shard_worker(rank, world, port, n, path):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    rng = np.random.default_rng(7)
    f64 = dict(dtype=torch.float64, device="cuda")
    mu_np = np.exp(rng.uniform(0.0, np.log(300.0), n))  # heavy-tailed costs (C5-like)
    mu = torch.tensor(mu_np, **f64)
    y0 = torch.tensor(np.tile([2.0, 0.0], (n, 1)), **f64)
    te = torch.tensor(np.linspace(0.0, 5.0, 7), **f64)
    f = bode.vdp_dynamics(bode.VdpParams(mu))
    kw = dict(controller=bode.pid_controller("PI42"), mode="fast", max_steps=100_000)
    got = D.solve_sharded_device(y0, 0.0, 5.0, f, t_eval=te, cost_hint=mu, **kw)
    if rank == 0:
        torch.save({k: v.cpu() for k, v in got.items() if isinstance(v, torch.Tensor)}, path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_solve_sharded_device_multirank_bitwise_equals_unsharded(world, tmp_path):
    import torch.multiprocessing as mp
    n = 6007
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    path = str(tmp_path / "sharded.pt")
    mp.start_processes(_shard_worker, args=(world, port, n, path), nprocs=world,
                       start_method="spawn")
    got = torch.load(path)
    rng = np.random.default_rng(7)
    f64 = dict(dtype=torch.float64, device="cuda")
    mu = torch.tensor(np.exp(rng.uniform(0.0, np.log(300.0), n)), **f64)
    ref = bode.solve_device(torch.tensor(np.tile([2.0, 0.0], (n, 1)), **f64),
                            torch.zeros(n, **f64), torch.full((n,), 5.0, **f64),
                            bode.vdp_dynamics(bode.VdpParams(mu)),
                            t_eval=torch.tensor(np.linspace(0.0, 5.0, 7), **f64),
                            controller=bode.pid_controller("PI42"), mode="fast",
                            max_steps=100_000)
    for k in ("n_steps", "n_accepted", "final_dt", "status", "n_emitted", "ys", "n_f_evals"):
        assert torch.equal(got[k], ref[k].cpu()), k
