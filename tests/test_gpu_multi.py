"""bode_solve_multi (include/bode.h): one batch sharded over
the GPUs of one process.  On a one-GPU box the shards share device 0, which
exercises the same plan / launch / combine path; per-instance results must
equal the unsharded solve's rows and the combined n_f_evals the unsharded
batch-global count (the reference's definition, solver.py:184,224,239)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _batch(n, seed=3):
    import torch

    import paper_2210_12375_b200 as bode
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda:0")
    mu = torch.tensor(rng.uniform(1.0, 30.0, n), dtype=torch.float64, device=dev)
    t_end = torch.tensor(rng.uniform(5.0, 20.0, n), dtype=torch.float64, device=dev)
    y0 = torch.tensor(np.tile([2.0, 0.0], (n, 1)), dtype=torch.float64, device=dev)
    te = torch.stack([t_end * 0.5, t_end], dim=1)
    return bode, y0, t_end, te, bode.vdp_dynamics(bode.VdpParams(mu)), mu * t_end


@pytest.mark.parametrize("ndev,cost", [(2, False), (3, True), (1, True)])
def test_solve_multi_equals_unsharded(ndev, cost):
    import torch

    from paper_2210_12375_b200 import distributed as D
    bode, y0, t_end, te, dyn, c = _batch(3000)
    kw = dict(method="dopri5", atol=1e-6, rtol=1e-6, controller=bode.pid_controller("PI42"),
              mode="fast")
    ref = bode.solve_device(y0, 0.0, t_end, dyn, t_eval=te, **kw)
    got = D.solve_multi(y0, 0.0, t_end, dyn, devices=[0] * ndev, t_eval=te,
                        cost_hint=c if cost else None, **kw)
    torch.cuda.synchronize()
    for k in ("n_steps", "n_accepted", "status", "n_emitted"):
        assert torch.equal(got[k], ref[k]), k
    assert torch.equal(got["final_dt"], ref["final_dt"])
    assert torch.equal(got["ys"], ref["ys"])
    assert int(got["n_f_evals"][0]) == int(ref["n_f_evals"][0])


def test_solve_multi_shards_hold_global_counts():
    import torch

    from paper_2210_12375_b200 import distributed as D
    bode, y0, t_end, te, dyn, c = _batch(2000, seed=5)
    kw = dict(method="tsit5", atol=1e-7, rtol=1e-7, mode="exact")
    ref = bode.solve_device(y0, 0.0, t_end, dyn, t_eval=te, **kw)
    shards = D.solve_multi(y0, 0.0, t_end, dyn, devices=[0, 0], t_eval=te, gather=False, **kw)
    torch.cuda.synchronize()
    nmax = int(ref["n_steps"].max())
    for o in shards:
        assert int(o["n_f_evals"][0]) == int(ref["n_f_evals"][0])
        assert int(o["max_iterations"][0]) == nmax
        assert torch.equal(o["n_steps"], ref["n_steps"][o["idx"]])


def test_solve_multi_over_nccl_communicator():
    """The NCCL combine path: a one-device communicator made with
    ncclCommInitAll (the library loads NCCL at run time)."""
    import torch

    from paper_2210_12375_b200 import distributed as D
    try:
        nccl = ctypes.CDLL("libnccl.so.2")
    except OSError:
        pytest.skip("libnccl.so.2 not loadable")
    comm = ctypes.c_void_p()
    devs = (ctypes.c_int * 1)(0)
    assert nccl.ncclCommInitAll(ctypes.byref(comm), 1, devs) == 0
    try:
        bode, y0, t_end, te, dyn, c = _batch(1500, seed=7)
        kw = dict(method="dopri5", atol=1e-6, rtol=1e-6, mode="fast")
        ref = bode.solve_device(y0, 0.0, t_end, dyn, t_eval=te, **kw)
        got = D.solve_multi(y0, 0.0, t_end, dyn, devices=[0], t_eval=te, comms=[comm.value],
                            cost_hint=c, **kw)
        torch.cuda.synchronize()
        assert int(got["n_f_evals"][0]) == int(ref["n_f_evals"][0])
        assert torch.equal(got["n_steps"], ref["n_steps"])
    finally:
        nccl.ncclCommDestroy(comm)

