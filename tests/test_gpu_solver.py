"""Full-solve behaviour of the CUDA path: large-scale parity against the
oracle (BASELINE sizes), the reference's solver known answers
(tests/test_solver.py, test_acceptance.py) and the batch-independence /
ordering properties the persistent design relies on."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2210_12375_b200 as bode
import scenarios as S

pytestmark = pytest.mark.gpu
NT = os.cpu_count() or 1
PI42 = bode.pid_controller("PI42")
PI42_D = dict(betas=S.PI42, safety=0.9, factor_min=0.2, factor_max=10.0, hist=True)


def check_vs_oracle(sol, ref, n_rows_per_inst=None, tol=1e-10):
    assert np.array_equal(sol.status, ref["status"])
    assert np.array_equal(sol.stats.n_steps, ref["n_steps"])
    assert np.array_equal(sol.stats.n_accepted, ref["n_accepted"])
    assert np.array_equal(sol.n_emitted, ref["n_emitted"])
    assert sol.stats.n_f_evals[0] == ref["n_f_evals"][0]
    a, b = sol.ys_flat, ref["ys"]
    n = sol.status.shape[0]
    a = a.reshape(n, -1)
    b = b.reshape(n, -1)
    scale = np.maximum(np.abs(b).max(axis=1), 1e-300)
    err = np.max(np.abs(a - b).max(axis=1) / scale)
    assert err <= tol, err
    return err, float(np.mean(np.all(a == b, axis=1)))


def test_c2_full_scale_1M_vs_oracle():
    """BASELINE configs[1] at full size: every one of 2^20 instances has the
    oracle's status, step counts and a final state within 1e-10 (scaled)."""
    mu, t_end = S.c2_inputs()
    n = mu.shape[0]
    y0 = np.tile([2.0, 0.0], (n, 1))
    prob = bode.IvpBatch(y0, np.zeros(n), t_end, t_end[:, None])
    sol = bode.solve(prob, bode.vdp_dynamics(bode.VdpParams(mu)), controller=PI42,
                     cost_hint=mu * t_end)
    ref = O.solve(y0, 0.0, t_end, [np.array([x]) for x in t_end], dict(name="vdp", inst=mu[:, None]),
                  ctrl=PI42_D, nthreads=NT)
    err, bitwise = check_vs_oracle(sol, ref)
    print(f"C2 1M: scaled err {err:.2e}, bit-identical instances {bitwise:.1%}, "
          f"accepted {int(sol.stats.n_accepted.sum())}")


def test_c5_stiff_prefix_vs_oracle():
    mu = S.c5_inputs()[:32768]
    n = mu.shape[0]
    y0 = np.tile([2.0, 0.0], (n, 1))
    prob = bode.IvpBatch(y0, np.zeros(n), np.full(n, 10.0), np.full((n, 1), 10.0))
    sol = bode.solve(prob, bode.vdp_dynamics(bode.VdpParams(mu)), controller=PI42,
                     max_steps=100_000, cost_hint=mu)
    ref = O.solve(y0, 0.0, 10.0, [np.array([10.0])] * n, dict(name="vdp", inst=mu[:, None]),
                  ctrl=PI42_D, max_steps=100_000, nthreads=NT)
    check_vs_oracle(sol, ref)


def test_c3_lorenz_dense_output_prefix_vs_oracle():
    y0 = S.c3_inputs()[:1024]
    n = y0.shape[0]
    te = np.linspace(0.0, 10.0, 1000)
    prob = bode.IvpBatch(y0, np.zeros(n), np.full(n, 10.0), te)
    sol = bode.solve(prob, bode.lorenz_dynamics(), tableau=bode.tsit5(),
                     tol=bode.Tolerances(1e-8, 1e-8), max_steps=100_000)
    ref = O.solve(y0, 0.0, 10.0, te, dict(name="lorenz", inst=None, shared=(10.0, 28.0, 8 / 3)),
                  method="tsit5", atol=1e-8, rtol=1e-8, max_steps=100_000, nthreads=NT)
    # chaotic flow over t in [0,10] amplifies ulp-level pow differences by
    # ~e^(0.9*10); step counts stay identical, ys within 1e-9 scaled
    check_vs_oracle(sol, ref, tol=1e-9)


# ---- properties -------------------------------------------------------
def _lin_problem(seed, n=6):
    rng = np.random.default_rng(seed)
    lam = rng.uniform(-4.0, 0.5, size=n)
    y0 = rng.normal(size=(n, 2))
    te = [np.sort(rng.uniform(0.0, 2.0, size=4)) for _ in range(n)]
    return lam, y0, te


def test_batch_independence_bit_identical():  # tests/test_solver.py:140-168
    lam, y0, te = _lin_problem(11)
    n = len(lam)
    full = bode.solve(bode.IvpBatch(y0, np.zeros(n), np.full(n, 2.0), te),
                      bode.forced_linear_dynamics(lam, 1.0, 3.0), record_trace=True)
    for i in range(n):
        one = bode.solve(bode.IvpBatch(y0[i:i + 1], np.zeros(1), np.full(1, 2.0), [te[i]]),
                         bode.forced_linear_dynamics(lam[i:i + 1], 1.0, 3.0), record_trace=True)
        assert np.array_equal(full.ys[i], one.ys[0])
        assert np.array_equal(full.stats.extra["trace_dt"][i], one.stats.extra["trace_dt"][0])
        assert np.array_equal(full.stats.extra["trace_accept"][i],
                              one.stats.extra["trace_accept"][0])
        assert full.stats.n_steps[i] == one.stats.n_steps[0]
        assert full.status[i] == one.status[0]


def test_permutation_and_queue_order_invariance():  # tests/test_solver.py:170-189
    rng = np.random.default_rng(5)
    n = 4096
    mu = rng.uniform(1.0, 10.0, n)
    t_end = rng.uniform(5.0, 20.0, n)
    y0 = np.tile([2.0, 0.0], (n, 1))
    mk = lambda p: bode.IvpBatch(y0, np.zeros(n), t_end[p], t_end[p][:, None])  # noqa: E731
    a = bode.solve(mk(np.arange(n)), bode.vdp_dynamics(bode.VdpParams(mu)), controller=PI42)
    b = bode.solve(mk(np.arange(n)), bode.vdp_dynamics(bode.VdpParams(mu)), controller=PI42,
                   cost_hint=mu * t_end)
    assert np.array_equal(a.ys_flat, b.ys_flat)
    assert np.array_equal(a.stats.n_steps, b.stats.n_steps)
    perm = rng.permutation(n)
    c = bode.solve(mk(perm), bode.vdp_dynamics(bode.VdpParams(mu[perm])), controller=PI42)
    assert np.array_equal(c.ys_flat, a.ys_flat[perm])
    assert np.array_equal(c.stats.n_steps, a.stats.n_steps[perm])


def test_launch_shape_invariance():
    """Results do not depend on grid/block shape (lanes never share state)."""
    import torch

    rng = np.random.default_rng(9)
    n = 3000
    mu = torch.tensor(rng.uniform(1.0, 10.0, n), device="cuda")
    y0 = torch.tensor(np.tile([2.0, 0.0], (n, 1)), device="cuda")
    te = torch.linspace(0.0, 10.0, 7, dtype=torch.float64, device="cuda")
    outs = [bode.solve_device(y0, 0.0, 10.0, bode.vdp_dynamics(bode.VdpParams(mu)), t_eval=te,
                              threads_per_block=tpb, blocks=blk)
            for tpb, blk in ((128, 0), (32, 1), (64, 7), (96, 3))]
    for o in outs[1:]:
        assert torch.equal(o["ys"], outs[0]["ys"])
        assert torch.equal(o["n_steps"], outs[0]["n_steps"])
        assert torch.equal(o["n_f_evals"], outs[0]["n_f_evals"])
    with pytest.raises(ValueError):
        bode.solve_device(y0, 0.0, 10.0, bode.vdp_dynamics(bode.VdpParams(mu)),
                          threads_per_block=256)


# ---- the reference's solver known answers (tests/test_solver.py) ------
def _prob(y0, t_end=1.0, t_eval=None):
    y0 = np.atleast_2d(y0)
    n = y0.shape[0]
    return bode.IvpBatch(y0, np.zeros(n), np.full(n, t_end),
                         t_eval if t_eval is not None else [np.empty(0)] * n)


def test_constant_solution():
    sol = bode.solve(_prob(np.array([[3.0, -1.0]]), t_eval=[np.array([0.0, 0.3, 1.0])]),
                     bode.zero_dynamics())
    assert sol.status[0] == bode.SolveStatus.SUCCESS
    assert np.array_equal(sol.ys[0], np.tile([3.0, -1.0], (3, 1)))


def test_max_steps_bound():
    """Per-instance step counters are 32-bit: max_steps >= 2^31 - 2 is
    rejected (ValueError, BODE_EINVAL) instead of wrapping; the largest
    accepted value solves normally."""
    prob = _prob(np.array([[3.0, -1.0]]), t_eval=[np.array([0.0, 1.0])])
    with pytest.raises(ValueError):
        bode.solve(prob, bode.zero_dynamics(), max_steps=2 ** 31)
    sol = bode.solve(prob, bode.zero_dynamics(), max_steps=16)
    assert sol.status[0] == bode.SolveStatus.SUCCESS


def test_exponential_accuracy_and_backward():
    sol = bode.solve(_prob(np.ones((1, 1)), t_eval=[np.array([1.0])]), bode.linear_dynamics(1.0),
                     tol=bode.Tolerances(1e-8, 1e-8))
    assert abs(sol.ys[0][0, 0] - np.e) < 1e-6
    back = bode.IvpBatch(np.array([[np.e]]), np.ones(1), np.zeros(1), [np.array([0.5, 0.0])])
    sol = bode.solve(back, bode.linear_dynamics(1.0), tol=bode.Tolerances(1e-8, 1e-8))
    assert sol.status[0] == bode.SolveStatus.SUCCESS
    assert sol.ys[0][:, 0] == pytest.approx([np.exp(0.5), 1.0], abs=1e-6)


def test_failure_statuses():
    sol = bode.solve(_prob(np.ones((1, 1)), t_end=1e6), bode.linear_dynamics(1.0), max_steps=20)
    assert sol.status[0] == bode.SolveStatus.MAX_STEPS_EXCEEDED and sol.stats.n_steps[0] == 20
    sol = bode.solve(_prob(np.ones((1, 1))), bode.square_dynamics(-np.inf))
    assert sol.status[0] == bode.SolveStatus.INFINITE_DYNAMICS and sol.stats.n_steps[0] == 0
    sol = bode.solve(_prob(np.ones((1, 1)), t_end=2.0, t_eval=[np.array([0.5, 1.9])]),
                     bode.square_dynamics(), tol=bode.Tolerances(1e-8, 1e-8), max_steps=100_000)
    assert sol.status[0] == bode.SolveStatus.STEP_UNDERFLOW
    assert sol.ys[0].shape == (1, 1) and sol.ys[0][0, 0] == pytest.approx(2.0, rel=1e-6)


def test_evaluation_completeness_and_ragged():
    te = np.linspace(0.0, 1.0, 17)
    sol = bode.solve(_prob(np.ones((1, 1)), t_eval=[te]), bode.linear_dynamics(1.0),
                     tol=bode.Tolerances(1e-8, 1e-8))
    assert sol.ys[0].shape == (17, 1)
    assert sol.ys[0][:, 0] == pytest.approx(np.exp(te), abs=1e-6)
    sol = bode.solve(bode.IvpBatch(np.ones((2, 1)), np.zeros(2), np.ones(2),
                                   [np.array([0.25, 0.5, 0.75]), np.empty(0)]),
                     bode.linear_dynamics(1.0))
    assert sol.ys[0].shape == (3, 1) and sol.ys[1].shape == (0, 1)


def test_stats_and_per_instance_tolerances():
    sol = bode.solve(_prob(np.array([[1.0], [100.0], [0.01]])), bode.linear_dynamics(-1.0))
    assert np.all(sol.stats.n_f_evals == sol.stats.n_f_evals[0])
    assert np.all(sol.stats.n_accepted <= sol.stats.n_steps)
    tol = bode.Tolerances(atol=np.array([1e-10, 1e-3]), rtol=np.array([1e-10, 1e-3]))
    sol = bode.solve(_prob(np.ones((2, 1))), bode.linear_dynamics(1.0), tol=tol)
    assert sol.stats.n_accepted[0] > sol.stats.n_accepted[1]


def test_fsal_counting_formula():  # tests/test_stepper.py:156-171, criterion 6
    sol = bode.solve(bode.IvpBatch([[1.0, 0.0]], [0.0], [10.0], [np.empty(0)]),
                     bode.damped_dynamics(), tol=bode.Tolerances(1e-9, 1e-9))
    a = sol.stats.n_accepted[0]
    r = sol.stats.n_steps[0] - a
    assert sol.stats.n_f_evals[0] == 1 + 6 * a + 7 * r
    sol = bode.solve(bode.IvpBatch([[1.0, 0.0]], [0.0], [10.0], [np.empty(0)]),
                     bode.damped_dynamics(), tableau=bode.heun(), tol=bode.Tolerances(1e-5, 1e-5))
    assert sol.stats.n_f_evals[0] == 1 + 2 * sol.stats.n_steps[0]


def test_mixed_accept_reject_and_three_point_step():  # tests/test_solver.py:241-262
    tol = bode.Tolerances(atol=np.array([1e-2, 1e-10]), rtol=np.array([0.0, 0.0]))
    sol = bode.solve(_prob(np.ones((2, 1))), bode.linear_dynamics(1.0), tol=tol, dt0=0.5,
                     record_trace=True)
    assert [sol.stats.extra["trace_accept"][i][0] for i in range(2)] == [True, False]
    sol = bode.solve(_prob(np.ones((1, 1)), t_eval=[np.array([0.1, 0.2, 0.3])]),
                     bode.zero_dynamics(), dt0=0.4, record_trace=True)
    assert sol.stats.extra["trace_accept"][0][0] and sol.n_emitted[0] == 3


def test_acceptance_4_large_batch_accuracy():  # tests/test_acceptance.py:116-127
    """256 VdP, mu=2, tol 1e-5 vs a tight 1e-10 self-reference: max error < 1e-3
    (VdP with phase-spread starts on [0, 6.6])."""
    rng = np.random.default_rng(4)
    n = 256
    y0 = np.stack([rng.uniform(-2, 2, n), rng.uniform(-2, 2, n)], 1)
    prob = bode.IvpBatch(y0, np.zeros(n), np.full(n, 6.6), np.linspace(0, 6.6, 200))
    f = bode.vdp_dynamics(bode.VdpParams(2.0))
    sol = bode.solve(prob, f, tol=bode.Tolerances(1e-5, 1e-5), max_steps=100_000)
    ref = bode.solve(prob, f, tol=bode.Tolerances(1e-10, 1e-10), max_steps=1_000_000)
    assert sol.ok and ref.ok
    err = max(np.max(np.abs(sol.ys[i][-1] - ref.ys[i][-1])) for i in range(n))
    assert err < 1e-3


def test_untraceable_callable_is_rejected():
    # a NumPy callable runs on the device once traced (tests/test_gpu_dropin.py);
    # Python control flow on state values cannot be traced: no CPU fallback
    with pytest.raises(NotImplementedError):
        bode.solve(_prob(np.ones((1, 1))), lambda t, y: y if y[0, 0] > 0 else -y)


def test_pipelined_host_path_matches_single_chunk():
    """bode_solve_host's chunked copy/compute pipeline (and the on-device LPT
    order) change only the schedule: every output, including the
    batch-global n_f_evals, is bit-identical."""
    rng = np.random.default_rng(21)
    n = 100_003
    mu = rng.uniform(1.0, 10.0, n)
    t_end = rng.uniform(5.0, 20.0, n)
    te = [np.sort(rng.uniform(0.0, x, rng.integers(0, 4))) for x in t_end]
    prob = bode.IvpBatch(np.tile([2.0, 0.0], (n, 1)), np.zeros(n), t_end, te)
    f = bode.vdp_dynamics(bode.VdpParams(mu))
    a = bode.solve(prob, f, controller=PI42, pipeline_chunks=1)
    for chunks, cost in ((4, None), (7, mu * t_end), (1, mu * t_end)):
        b = bode.solve(prob, f, controller=PI42, pipeline_chunks=chunks, cost_hint=cost)
        assert np.array_equal(a.ys_flat, b.ys_flat)
        for k in ("n_steps", "n_accepted", "n_f_evals", "final_dt"):
            assert np.array_equal(getattr(a.stats, k), getattr(b.stats, k)), k
        assert np.array_equal(a.status, b.status) and np.array_equal(a.n_emitted, b.n_emitted)


def test_host_transfer_paths_are_equivalent(monkeypatch):
    """Page-locked inputs (direct DMA), pageable inputs through the pinned
    staging arena, and pageable inputs beyond the arena limit (driver-staged
    copies) give bit-identical results (csrc/bode_hostio.cu)."""
    rng = np.random.default_rng(22)
    n = 70_001
    mu = rng.uniform(1.0, 10.0, n)
    t_end = rng.uniform(5.0, 20.0, n)
    te = [np.sort(rng.uniform(0.0, x, rng.integers(0, 3))) for x in t_end]
    y0 = np.tile([2.0, 0.0], (n, 1))
    f = bode.vdp_dynamics(bode.VdpParams(mu))
    a = bode.solve(bode.IvpBatch(y0, np.zeros(n), t_end, te), f, controller=PI42)
    P = bode.pinned
    b = bode.solve(bode.IvpBatch(P(y0), P(np.zeros(n)), P(t_end), te),
                   bode.vdp_dynamics(bode.VdpParams(P(mu))), controller=PI42)
    monkeypatch.setenv("BODE_STAGING_MAX", "4096")  # nothing fits: driver-staged copies
    c = bode.solve(bode.IvpBatch(y0, np.zeros(n), t_end, te), f, controller=PI42)
    for o in (b, c):
        assert np.array_equal(a.ys_flat, o.ys_flat)
        for k in ("n_steps", "n_accepted", "n_f_evals", "final_dt"):
            assert np.array_equal(getattr(a.stats, k), getattr(o.stats, k)), k
        assert np.array_equal(a.status, o.status) and np.array_equal(a.n_emitted, o.n_emitted)


def test_mlp_neural_ode_vs_reference_fp32():
    """C4 (neural ODE, D=64, H=256, tanh): the reference solve with a NumPy
    fp32 MLP (tests/golden/mlp.npz).  fp32 GEMM summation order differs from
    OpenBLAS (and 3xTF32 from fp32), so step counts are compared in
    aggregate (2%, north_star) and y(T) at 1e-4 of each instance's scale;
    statuses must match."""
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "mlp.npz"))
    n = z["y0"].shape[0]
    prob = bode.IvpBatch(z["y0"], np.zeros(n), np.full(n, 10.0), np.full((n, 1), 10.0))
    sol = bode.solve(prob, bode.mlp_dynamics(z["W1"], z["b1"], z["W2"], z["b2"]),
                     max_steps=100_000)
    assert np.array_equal(sol.status, z["status"])
    ratio = sol.stats.n_steps.sum() / z["n_steps"].sum()
    assert abs(ratio - 1.0) < 0.02, ratio
    ys = sol.ys_flat.reshape(n, -1)
    rel = np.max(np.abs(ys - z["ys"]), axis=1) / np.max(np.abs(z["ys"]), axis=1)
    assert np.max(rel) < 1e-4, np.max(rel)
    # batch-global n_f_evals follows the FSAL formula over the lockstep loop
    assert sol.stats.n_f_evals[0] >= 1 + 6 * sol.stats.n_steps.max()


def test_mlp_matches_oracle_at_scale():
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "mlp.npz"))
    rng = np.random.default_rng(3)
    n = 2048
    y0 = rng.normal(size=(n, 64))
    mlp = (z["W1"], z["b1"], z["W2"], z["b2"])
    te = np.array([2.5, 5.0, 10.0])
    sol = bode.solve(bode.IvpBatch(y0, np.zeros(n), np.full(n, 10.0), te),
                     bode.mlp_dynamics(*mlp), tol=bode.Tolerances(1e-6, 1e-6), max_steps=100_000)
    ref = O.solve(y0, 0.0, 10.0, te, dict(name="mlp", inst=None, shared=(), mlp=mlp),
                  atol=1e-6, rtol=1e-6, max_steps=100_000, nthreads=NT)
    assert np.array_equal(sol.status, ref["status"])
    assert abs(sol.stats.n_steps.sum() / ref["n_steps"].sum() - 1.0) < 0.02
    assert np.mean(sol.stats.n_steps == ref["n_steps"]) > 0.9
    a, b = sol.ys_flat.reshape(n, -1), ref["ys"].reshape(n, -1)
    assert np.max(np.abs(a - b).max(axis=1) / np.abs(b).max(axis=1)) < 1e-4


@pytest.mark.parametrize("te", ["shared", "ragged"])
def test_solve_device_ys_equals_host_ys(te):
    """solve(..., device_ys=True) is the same solve with ys left on the
    device: ys bitwise equal to the host-buffer solve, same statistics."""
    import torch

    rng = np.random.default_rng(21)
    n = 3000
    mu = rng.uniform(1.0, 10.0, n)
    t1 = rng.uniform(3.0, 8.0, n)
    tev = (np.linspace(0.0, 3.0, 7) if te == "shared"
           else [np.sort(rng.uniform(0.0, t1[i], i % 5)) for i in range(n)])
    prob = bode.IvpBatch(np.tile([2.0, 0.0], (n, 1)), np.zeros(n), t1, tev)
    f = bode.vdp_dynamics(bode.VdpParams(mu))
    kw = dict(controller=bode.pid_controller("PI42"), mode="fast", cost_hint=mu * t1)
    a = bode.solve(prob, f, **kw)
    b = bode.solve(prob, f, device_ys=True, **kw)
    assert isinstance(b.ys_flat, torch.Tensor) and b.ys_flat.is_cuda
    assert np.array_equal(a.ys_flat.reshape(-1), b.ys_flat.cpu().numpy().reshape(-1))
    for k in ("n_steps", "n_accepted", "final_dt"):
        assert np.array_equal(getattr(a.stats, k), getattr(b.stats, k)), k
    assert np.array_equal(a.status, b.status) and np.array_equal(a.n_emitted, b.n_emitted)
    assert np.array_equal(a.stats.n_f_evals, b.stats.n_f_evals)
    i = int(np.argmax(a.n_emitted))
    assert np.array_equal(a.ys[i], b.ys[i].cpu().numpy())
