"""Benchmark: accepted instance-steps/s of the batched independent ODE solve.

Headline workload (BASELINE.json metric, configs[1]):
Van der Pol, 2^20 instances per GPU, mu ~ U[1,10], t_end ~ U[5,20],
y0 = (2, 0), t_eval = {t_end_i}, dopri5, PI42 (0.6, -0.2, 0), atol = rtol =
1e-6, fp64, fast mode (FMA contraction, ~1-ulp controller pow; statuses and
step counts identical to the oracle at full scale; --mode exact replays the
reference's unfused operation order).  A "step" is one
complete solve of that batch: the persistent kernel runs every instance to
termination.  value = sum_i n_accepted_i / device time (max over ranks,
weak scaling: every rank solves its own 2^20-instance shard).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c5]
    python bench.py --impl reference ...   # CPU reference arm (oracle port)
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PI42 = dict(betas=(0.6, -0.2, 0.0), safety=0.9, factor_min=0.2, factor_max=10.0, hist=True)
ICTRL = dict(betas=(1.0, 0.0, 0.0), safety=0.9, factor_min=0.2, factor_max=10.0, hist=True)

# algorithmic flops: per attempted step 82d+20+6*F_f (FSAL,
# s=7), per emitted point 15d+51; pow counted separately (2 per step with PI42)
F_F = {"vdp": 5, "lorenz": 8, "mlp": 4 * 64 * 256 + 64 + 256}  # MLP: 2 GEMMs + biases


def flops_per_step(dyn, d):
    return 82 * d + 20 + 6 * F_F[dyn]


def flops_per_point(d):
    return 15 * d + 51


# ----------------------------------------------------------------- configs --
def make_config(name, rank, n_override=None):
    """Seeded synthetic inputs; rank r of a weak-scaling run draws shard r."""
    if name == "c2":
        n = n_override or 2 ** 20
        rng = np.random.default_rng(1000 + rank) if rank else np.random.default_rng(0)
        mu = rng.uniform(1.0, 10.0, n)
        t_end = rng.uniform(5.0, 20.0, n)
        return dict(workload="vdp_1M_dopri5_pi42_fp64", dyn="vdp", n=n, d=2,
                    y0=np.tile([2.0, 0.0], (n, 1)), t_start=np.zeros(n), t_end=t_end,
                    te2d=t_end[:, None].copy(), mu=mu, method="dopri5", ctrl=PI42,
                    tol=1e-6, max_steps=10_000, cost=mu * t_end)
    if name == "c1":
        n = n_override or 256
        rng = np.random.default_rng(0)
        mu = rng.uniform(1.0, 10.0, n)
        return dict(workload="vdp_256_dopri5_I_50pts_fp64", dyn="vdp", n=n, d=2,
                    y0=np.tile([2.0, 0.0], (n, 1)), t_start=np.zeros(n), t_end=np.full(n, 10.0),
                    te1d=np.linspace(0.0, 10.0, 50), mu=mu, method="dopri5", ctrl=ICTRL,
                    tol=1e-6, max_steps=100_000, cost=None)
    if name == "c5":
        n = n_override or 2 ** 20
        rng = np.random.default_rng(0 if rank == 0 else 1000 + rank)
        mu = np.exp(rng.uniform(0.0, np.log(1000.0), n))
        return dict(workload="vdp_1M_stiff_logmu_dopri5_pi42_fp64", dyn="vdp", n=n, d=2,
                    y0=np.tile([2.0, 0.0], (n, 1)), t_start=np.zeros(n), t_end=np.full(n, 10.0),
                    mu=mu, method="dopri5", ctrl=PI42, tol=1e-6, max_steps=100_000,
                    cost=mu)
    if name == "c4":  # neural ODE: SURVEY.md §8(d) C4 weights/inputs
        n = n_override or 65536
        rng = np.random.default_rng(0)
        D, H = 64, 256
        W1 = (rng.normal(size=(H, D)) / np.sqrt(D)).astype(np.float32)
        b1 = (0.1 * rng.normal(size=H)).astype(np.float32)
        W2 = (rng.normal(size=(D, H)) / np.sqrt(H)).astype(np.float32)
        b2 = (0.1 * rng.normal(size=D)).astype(np.float32)
        y0 = np.random.default_rng(1 + rank).normal(size=(n, D))
        return dict(workload="mlp64x256_tanh_64K_dopri5_fp32mlp_fp64state", dyn="mlp", n=n, d=D,
                    y0=y0, t_start=np.zeros(n), t_end=np.full(n, 10.0),
                    te2d=np.full((n, 1), 10.0), mu=None, mlp=(W1, b1, W2, b2),
                    method="dopri5", ctrl=ICTRL, tol=1e-6, max_steps=100_000, cost=None)
    if name == "c3":
        n = n_override or 2 ** 18
        rng = np.random.default_rng(0 if rank == 0 else 1000 + rank)
        y0 = 1.0 + 0.1 * rng.normal(size=(n, 3))
        return dict(workload="lorenz_256K_tsit5_1e-8_1000pts_fp64", dyn="lorenz", n=n, d=3,
                    y0=y0, t_start=np.zeros(n), t_end=np.full(n, 10.0),
                    te1d=np.linspace(0.0, 10.0, 1000), mu=None, method="tsit5", ctrl=ICTRL,
                    tol=1e-8, max_steps=100_000, cost=None)
    raise ValueError(name)


def n_points(cfg):
    if "te2d" in cfg:
        return cfg["te2d"].size
    if "te1d" in cfg:
        return cfg["n"] * cfg["te1d"].size
    return 0


# ------------------------------------------------------------ CPU legs ----
def cpu_run(cfg, sample, nthreads):
    """Oracle (C restatement of the reference, test infrastructure) on the
    first `sample` instances; returns (accepted, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    k = min(sample, cfg["n"])
    if "te2d" in cfg:
        te = [cfg["te2d"][i] for i in range(k)]
    else:
        te = cfg.get("te1d")
    dyn = (dict(name="vdp", inst=cfg["mu"][:k, None]) if cfg["dyn"] == "vdp"
           else dict(name="mlp", inst=None, shared=(), mlp=cfg["mlp"]) if cfg["dyn"] == "mlp"
           else dict(name="lorenz", inst=None, shared=(10.0, 28.0, 8.0 / 3.0)))
    t0 = time.perf_counter()
    r = O.solve(cfg["y0"][:k], cfg["t_start"][:k], cfg["t_end"][:k], te, dyn,
                method=cfg["method"], atol=cfg["tol"], rtol=cfg["tol"], ctrl=cfg["ctrl"],
                max_steps=cfg["max_steps"], nthreads=nthreads)
    dt = time.perf_counter() - t0
    return int(r["n_accepted"].sum()), dt, k


def cpu_sample_size(cfg):
    # BASELINE.md §3 / SURVEY §8(d): C1 and C2 at full size, C3 >= 16K and
    # C5 >= 64K seeded prefixes (the rate is intensive); C4's fp32-MLP oracle
    # is ~1e5 steps/s, so a 1024-instance prefix
    return {"c2": 2 ** 20, "c5": 65_536, "c3": 16_384, "c1": 256, "c4": 1024}[cfg["_name"]]


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


CPU_NOTE = ("C oracle (bode_oracle.c, gcc -O2 -ffp-contract=off, libm pow; no NumPy, so "
            "NPY_DISABLE_CPU_FEATURES does not apply), one pthread per host core")


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on host cores (oracle port,
    all threads), rank 0 only."""
    if rank != 0:
        return
    cfg = make_config(args.config, 0)
    cfg["_name"] = args.config
    nthreads = os.cpu_count() or 1
    sample = cpu_sample_size(cfg)
    for _ in range(args.warmup):
        cpu_run(cfg, sample, nthreads)
    acc, secs = 0, 0.0
    for _ in range(args.steps):
        a, s, k = cpu_run(cfg, sample, nthreads)
        acc += a
        secs += s
    value = acc / secs
    line = dict(metric="accepted instance-steps/sec", value=value,
                unit="instance-steps/s", n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=1e3 * secs / args.steps, higher_is_better=True,
                scaling="strong" if world > 1 else "weak", vs_baseline=None, dtype="f64",
                data="synthetic", impl="reference",
                config=dict(workload=cfg["workload"], instances_per_gpu=cfg["n"],
                            global_instances=cfg["n"], method=cfg["method"],
                            controller="PI42" if cfg["ctrl"] is PI42 else "I", tol=cfg["tol"],
                            sample_instances=min(sample, cfg["n"]),
                            parallelism=f"host threads ({nthreads})"),
                cpu_baseline=dict(value=value, unit="instance-steps/s", cores=nthreads,
                                  kind="port", cpu_model=cpu_model(), note=CPU_NOTE,
                                  sample=f"first {min(sample, cfg['n'])} of the {cfg['n']} "
                                         f"instances of the seeded {cfg['workload']} batch "
                                         "per step"),
                e2e=dict(value=value, unit="instance-steps/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU leg -----
class ClockSampler:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        if os.environ.get("BODE_NO_CLOCKS"):  # diagnosis only: no nvidia-smi polling
            return self
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self, gpu_index):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except Exception:
            return None
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 9 and r[0].strip() == str(gpu_index)]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return dict(sm_mhz=float(np.median(sm)) if sm else None, sm_max_mhz=mx,
                    reasons=reasons, samples=len(rows))


def measured_peak(key):
    """Driver-measured roofline denominators (MEASURED_PEAKS.json); fallback
    per /opt/skills/guides/B200_PROFILING.md when the file is absent."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))[key])
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}[key]


def fp64_peak(torch, lib, dev):
    """Measured DFMA throughput (bode_probe_fp64), TFLOP/s."""
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, iters = sms * 8, 20000
    st = torch.cuda.current_stream(dev)
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        lib.bode_probe_fp64(iters, blocks, out.data_ptr(), st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        secs = e0.elapsed_time(e1) / 1e3
        best = max(best, 2.0 * 8 * 256 * blocks * iters / secs / 1e12)
    return best


def tf32_peak(torch, lib, dev):
    """Measured tcgen05 kind::tf32 throughput (bode_probe_tf32), TFLOP/s."""
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    reps = 4000
    st = torch.cuda.current_stream(dev)
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        lib.bode_probe_tf32(reps, sms, st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        secs = e0.elapsed_time(e1) / 1e3
        best = max(best, 2.0 * 128 * 256 * 8 * 8 * reps * sms / secs / 1e12)
    return best


def run_bode(args, rank, world, local_rank):
    import torch

    import paper_2210_12375_b200 as bode
    from paper_2210_12375_b200 import _abi

    # BODE_BENCH_SHARED_GPU=1 (tests only): every rank on cuda:0 with gloo
    # collectives, to exercise the multi-rank path on a one-GPU box
    shared_gpu = os.environ.get("BODE_BENCH_SHARED_GPU") == "1"
    dev = torch.device("cuda", 0 if shared_gpu else local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    lib = _abi.load()
    # strong scaling (default for N > 1): every rank holds the same seeded
    # batch and solves its cost-balanced shard of it; weak: rank r solves its
    # own full-size batch (seed 1000 + r)
    strong = world > 1 and args.scaling == "strong"
    cfg = make_config(args.config, 0 if strong else rank)
    cfg["_name"] = args.config
    n, d = cfg["n"], cfg["d"]
    f64 = dict(dtype=torch.float64, device=dev)
    y0 = torch.tensor(cfg["y0"], **f64)
    ts = torch.tensor(cfg["t_start"], **f64)
    tn = torch.tensor(cfg["t_end"], **f64)
    dyn = (bode.vdp_dynamics(bode.VdpParams(torch.tensor(cfg["mu"], **f64)))
           if cfg["dyn"] == "vdp" else bode.mlp_dynamics(*cfg["mlp"]) if cfg["dyn"] == "mlp"
           else bode.lorenz_dynamics())
    ctrl = bode.PidCoefficients(*cfg["ctrl"]["betas"])
    te_kw = {}
    if "te2d" in cfg:
        te_kw["t_eval"] = torch.tensor(cfg["te2d"], **f64)
    elif "te1d" in cfg:
        te_kw["t_eval"] = torch.tensor(cfg["te1d"], **f64)
    cost = torch.tensor(cfg["cost"], **f64) if (cfg["cost"] is not None and args.lpt) else None
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    st = torch.cuda.current_stream(dev)

    is_mlp = cfg["dyn"] == "mlp"

    from paper_2210_12375_b200 import distributed as bdist

    def one_step(prof=None):
        if strong:
            # the whole sharded job: device shard plan (cost-aware), shard
            # row gathers, persistent solve of the shard, the n_f_evals
            # all-reduce and the NCCL gather of every instance's results to
            # rank 0 in batch order (distributed.solve_sharded_device)
            out = bdist.solve_sharded_device(
                y0, ts, tn, dyn, method=cfg["method"], atol=cfg["tol"], rtol=cfg["tol"],
                controller=ctrl, max_steps=cfg["max_steps"], mode=args.mode,
                cost_hint=torch.tensor(cfg["cost"], **f64) if cfg["cost"] is not None else None,
                prof_events=prof, gather_to=0, **te_kw)
            if out is None:  # ranks other than 0 hold no results after the gather
                z = torch.zeros(1, dtype=torch.int64, device=dev)
                out = dict(n_accepted=z, n_steps=z, launches=0)
            return out
        out = bode.solve_device(y0, ts, tn, dyn, method=cfg["method"], atol=cfg["tol"],
                                rtol=cfg["tol"], controller=ctrl, max_steps=cfg["max_steps"],
                                mode=args.mode, cost_hint=cost, prof_events=prof,
                                with_refresh_map=world > 1, **te_kw)
        if world > 1:
            # the sharded batch's one real exchange: the batch-global n_f_evals
            # (MAX all-reduce of iteration counts and refresh maps, NCCL)
            out["n_f_evals"] = bdist.global_f_evals_device(
                out, stages=2 if cfg["method"] == "heun" else 7, fsal=cfg["method"] != "heun")
            if args.gather:  # optional: gather ys/stats to rank 0 over NVLink
                bdist.gather_device(out, dst=0)
        return out

    times, kern_times, accepted, attempted = [], [], 0, 0
    kern_ms = 0.0
    clock_path = os.path.join(tempfile.gettempdir(), f"bode_clocks_rank{rank}_{os.getpid()}.csv")
    # the clock sampler runs from the warm-up through the timed steps
    def run_steps(k):
        # k steps enqueued back to back (L2 flush, then the solve between its
        # two events), so host launch latency overlaps the previous step's
        # device work; the caller synchronises once after the last step
        pend = []
        for _ in range(k):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(st)  # materialise the cudaEvent_t handles (torch creates them lazily);
            k1.record(st)  # bode_solve re-records both around the persistent launch
            e0.record(st)
            out = one_step((k0, k1))
            e1.record(st)
            # device-side reductions only; the step's buffers go back to the
            # caching allocator (holding them would force fresh cudaMallocs,
            # which synchronise, inside later timed steps)
            pend.append((e0, e1, k0, k1, out["n_accepted"].sum(), out["n_steps"].sum(),
                         out["launches"]))

            del out
        return pend

    with ClockSampler(clock_path) as clk:
        # warm-up: the identical loop body (lazy module loads, allocator pools)
        run_steps(args.warmup)
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        pending = run_steps(args.steps)
        torch.cuda.synchronize(dev)
        time.sleep(0.25)
    for e0, e1, k0, k1, acc_d, att_d, nl in pending:
        times.append(e0.elapsed_time(e1))
        # the dominant kernel alone (persistent integrator), same stream
        kern_times.append(k0.elapsed_time(k1))
        accepted += int(acc_d)
        attempted += int(att_d)
        launches_per_step = nl  # kernels of ours in this solve
    del pending
    torch.cuda.synchronize(dev)
    total_ms = float(np.sum(times))
    # max over ranks of device time; sum of accepted over ranks
    if dist:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        aa = torch.tensor([accepted, attempted], dtype=torch.float64, device=dev)
        dist.all_reduce(aa)
        accepted, attempted = int(aa[0].item()), int(aa[1].item())
    value = accepted / (total_ms / 1e3)

    # ---- roofline of the dominant kernel, timed with events inside the timed
    # steps above (bode_solve records them around the persistent launch)
    pts = n_points(cfg)
    kern_ms = float(np.mean(kern_times))
    # attempted steps per persistent launch (one launch per rank per step)
    att_launch = attempted / args.steps / max(world, 1)
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[args.config]
        traffic = tj["dram_read_bytes"] + tj["dram_write_bytes"]
    except Exception:
        pass
    ncu_pipes = None  # pipe utilisation of the same kernel from the committed ncu capture
    try:
        ncu_pipes = json.load(open(os.path.join(ROOT, "profiles", "ncu_pipes.json")))[args.config]
    except Exception:
        pass
    if is_mlp:
        # tensor-pipe bound: algorithmic MLP GEMM flops (4*D*H per f-eval, 6 FSAL
        # stages per attempted step) of the fused persistent kernel (the init
        # pass's two evaluations per instance run before it); peak = TF32
        # tcgen05 throughput measured in-run by bode_probe_tf32
        D_, H_ = cfg["mlp"][0].shape[1], cfg["mlp"][0].shape[0]
        flops_launch = 4.0 * D_ * H_ * 6 * att_launch
        peak = tf32_peak(torch, lib, dev)
        achieved = flops_launch / (kern_ms / 1e3) / 1e12
        roof = dict(bound="tensor", achieved=achieved, peak=peak, unit="TFLOP/s",
                    frac=achieved / peak, traffic=traffic, kernel="mlp_fused_kernel",
                    note="algorithmic GEMM flops of the fp32 MLP (3xTF32 issues 3x the MMAs: "
                         "tensor-pipe work = 3 x achieved) / fused-kernel time (CUDA events "
                         "around its launch); peak = tcgen05 kind::tf32 M=128 N=256 throughput "
                         "measured in-run by bode_probe_tf32",
                    mma_issue_frac=3 * achieved / peak, kernel_ms=kern_ms, ncu=ncu_pipes)
    else:
        peak_fp64 = fp64_peak(torch, lib, dev)
        flops_launch = flops_per_step(cfg["dyn"], d) * att_launch + flops_per_point(d) * pts
        achieved = flops_launch / (kern_ms / 1e3) / 1e12
        roof = dict(bound="fp64", achieved=achieved, peak=peak_fp64, unit="TFLOP/s",
                    frac=achieved / peak_fp64, traffic=traffic, kernel="bode_persistent_kernel",
                    note="algorithmic flops (SURVEY §8(a): 82d+20+6F_f per attempted step, "
                         "15d+51 per point; pow, div, sqrt not counted) / persistent-kernel time "
                         "(CUDA events around its launch); peak = DFMA throughput measured in-run "
                         "by bode_probe_fp64 (2 flops/DFMA); traffic = ncu dram bytes/launch "
                         "(profiles/traffic.json); ncu = FP64-pipe / issue utilisation of the "
                         "same kernel (profiles/ncu_pipes.json)",
                    kernel_ms=kern_ms, ncu=ncu_pipes)

    # ---- end to end through the reference-facing solve() with host buffers
    e2e = None
    if not args.no_e2e:
        # the caller stages its inputs in page-locked host memory (bode.pinned),
        # so the uploads inside the timed call are DMA copies
        P = bode.pinned
        te_h = cfg.get("te2d", cfg.get("te1d"))
        prob = bode.IvpBatch(P(cfg["y0"]), P(cfg["t_start"]), P(cfg["t_end"]),
                             P(te_h) if te_h is not None else [np.empty(0)] * n)
        dyn_h = (bode.vdp_dynamics(bode.VdpParams(P(cfg["mu"]))) if cfg["dyn"] == "vdp"
                 else bode.mlp_dynamics(*cfg["mlp"]) if cfg["dyn"] == "mlp"
                 else bode.lorenz_dynamics())
        tab = {"dopri5": bode.dopri5, "tsit5": bode.tsit5}[cfg["method"]]()
        kw = dict(tableau=tab, tol=bode.Tolerances(cfg["tol"], cfg["tol"]), controller=ctrl,
                  max_steps=cfg["max_steps"], mode=args.mode,
                  cost_hint=P(cfg["cost"]) if (args.lpt and cfg["cost"] is not None) else None)
        def e2e_solve():
            if strong:  # host arrays in, the full Solution on rank 0
                return bdist.solve_sharded(prob, dyn_h, **kw)
            return bode.solve(prob, dyn_h, **kw)

        for _ in range(max(3, args.warmup)):  # untimed warm-up calls, as for `value`
            del_sol = e2e_solve()
            del del_sol
        if dist:
            dist.barrier()
        e2e_t, e2e_acc = [], 0
        for _ in range(max(1, min(args.steps, 5))):
            flush.zero_()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            sol = e2e_solve()
            e2e_t.append(time.perf_counter() - t0)
            e2e_acc += int(sol.stats.n_accepted.sum()) if sol is not None else 0
            del sol  # result consumed: its page-locked buffers return to the host cache
        tot = float(np.sum(e2e_t))
        if dist:
            tt = torch.tensor([tot, e2e_acc], dtype=torch.float64, device=dev)
            dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
            acc_t = torch.tensor([float(e2e_acc)], dtype=torch.float64, device=dev)
            dist.all_reduce(acc_t)
            tot, e2e_acc = float(tt[0].item()), int(acc_t.item())
        h2d = (prob.y0.nbytes + prob.t_start.nbytes + prob.t_end.nbytes + prob.te_values.nbytes
               + (0 if prob.te_shared else prob.te_offsets.nbytes)
               + (cfg["mu"].nbytes if cfg["mu"] is not None else 0)
               + (sum(w.nbytes for w in cfg["mlp"]) if cfg.get("mlp") else 0)
               + (8 * n if args.lpt and cfg["cost"] is not None else 0))
        d2h = 8 * pts * d + n * (8 + 8 + 8 + 8 + 8) + 8  # ys + 5 int64/f64 stats + n_f_evals
        e2e = dict(value=e2e_acc / tot, unit="instance-steps/s", h2d_bytes_per_step=int(h2d),
                   d2h_bytes_per_step=int(d2h), ms_per_step=1e3 * tot / len(e2e_t),
                   path="paper_2210_12375_b200.solve -> bode_solve_host (NumPy arrays in "
                        "page-locked host memory, outputs page-locked)")
        if not strong and 8 * pts * d > 1e9:
            # the same call with ys left on the device (solve(..., device_ys=True)):
            # inputs up, statistics down -- for callers that consume the dense
            # output on the GPU (C3: 6.3 GB of ys otherwise cross PCIe)
            dv_t = []
            for _ in range(max(1, min(args.steps, 3))):
                flush.zero_()
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                sol = bode.solve(prob, dyn_h, device_ys=True, **kw)
                acc_dv = int(sol.stats.n_accepted.sum())
                dv_t.append(time.perf_counter() - t0)
                del sol
            e2e["device_ys"] = dict(value=acc_dv / float(np.mean(dv_t)), unit="instance-steps/s",
                                    ms_per_step=1e3 * float(np.mean(dv_t)),
                                    h2d_bytes_per_step=int(h2d),
                                    d2h_bytes_per_step=int(n * 40 + 8),
                                    path="paper_2210_12375_b200.solve(device_ys=True) -> "
                                         "solve_device (ys stay in HBM)")

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        nthreads = os.cpu_count() or 1
        sample = cpu_sample_size(cfg)
        a, s, k = cpu_run(cfg, sample, nthreads)
        cpu = dict(value=a / s, unit="instance-steps/s", cores=nthreads, kind="port",
                   cpu_model=cpu_model(), note=CPU_NOTE,
                   sample=f"first {k} of the {cfg['n']} instances of the seeded batch, one "
                          f"solve ({s:.2f} s wall)")

    clocks = clk.summary(dev.index)
    if rank == 0:
        line = dict(
            metric="accepted instance-steps/sec", value=value, unit="instance-steps/s",
            n_gpus=world, steps=args.steps, warmup=args.warmup,
            ms_per_step=total_ms / args.steps, higher_is_better=True,
            scaling="strong" if strong else "weak",
            vs_baseline=None, dtype="f64", data="synthetic",
            config=dict(workload=cfg["workload"],
                        instances_per_gpu=n if not strong else n / world,
                        global_instances=n if strong else n * world, method=cfg["method"],
                        controller="PI42" if cfg["ctrl"] is PI42 else "I",
                        tol=cfg["tol"],
                        mode=args.mode,
                        lpt_order=bool(args.lpt),
                        parallelism=(f"shard{world}: one {n}-instance batch, cost-balanced "
                                     "device partition, NCCL gather of all results to rank 0 "
                                     "inside every step") if strong else
                                    (f"shard{world}: independent {n}-instance batch per GPU"
                                     if world > 1 else "shard1"),
                        l2="flushed (256 MiB write) between steps",
                        accepted_per_step=accepted / args.steps,
                        attempted_per_step=attempted / args.steps),
            roofline=roof,
            cpu_baseline=cpu, e2e=e2e, gpu_launches=launches_per_step * args.steps,
            clocks=clocks)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="bode", choices=["bode", "reference"])
    p.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    # fast = FMA-contracted arithmetic + ~1-ulp controller pow; at full scale
    # (C2/C3/C5) every status and step count equals the oracle's and ys are
    # within 1e-10 (tests/test_gpu_parity.py, tools/parity_report.py); exact =
    # the reference's unfused operation order (85% of C2 bit-identical)
    p.add_argument("--mode", default="fast", choices=["exact", "fast"])
    p.add_argument("--lpt", type=int, default=1, help="cost-sorted (LPT) instance queue")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--gather", action="store_true",
                   help="N>1 weak scaling: also gather every shard's ys/stats to rank 0 "
                        "inside the timed step")
    p.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                   help="N>1: strong = shard ONE batch over the ranks (cost-aware device "
                        "partition, NCCL gather to rank 0 in every step); weak = an "
                        "independent full batch per rank")
    args = p.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_bode(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
