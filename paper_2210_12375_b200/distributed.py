"""Sharding one batch over the GPUs of a box (one process per GPU).

The solve path has no data-path exchange: instances are independent and a
shard's results are bitwise equal to its rows of the full batch (reference
tests/test_solver.py:140-168).  What a sharded solve needs is

  * a partition that balances *work*, not instance counts -- step counts are
    heavy-tailed, so instances are dealt in decreasing
    ``cost_hint`` order in a snake pattern (an LPT approximation);
  * the one genuinely global statistic, ``n_f_evals``: the reference
    counts full-batch dynamics evaluations of the lockstep loop
    (solver.py:184,224,239), i.e. 1 + (S-1)*max_i n_steps_i + #{loop
    iterations j >= 1 at which some running instance had rejected at j-1}.
    Each shard exports its max iteration count and its per-iteration refresh
    map (``bode_solve`` ``max_iterations_out`` / ``refresh_map_out``); ranks
    combine them with a MAX all-reduce (a byte per iteration, so MAX == OR);
  * a gather of ys/stats to one rank (or none: results can stay sharded).

Collectives go through ``torch.distributed`` (NCCL over NVLink on the GPU
box, gloo in the CPU tests).
"""

import numpy as np

from .solver import IvpBatch, Solution, SolveStats

__all__ = ["partition", "combine_f_evals", "subset_problem", "solve_sharded",
           "global_f_evals_device", "gather_device", "gather_rows", "shard_plan",
           "solve_sharded_device"]


def partition(n: int, world: int, cost=None) -> list:
    """Instance indices per rank.  Without costs: contiguous equal blocks.
    With costs: deal instances in decreasing cost in a snake pattern
    (0..W-1, W-1..0, ...), which keeps per-rank cost sums within one
    instance's cost of each other for sorted inputs (LPT-like)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if cost is None:
        bounds = [n * r // world for r in range(world + 1)]
        return [np.arange(bounds[r], bounds[r + 1]) for r in range(world)]
    order = np.argsort(-np.asarray(cost, dtype=np.float64), kind="stable")
    pos = np.arange(n)
    lap, k = pos // world, pos % world
    rank = np.where(lap % 2 == 0, k, world - 1 - k)
    return [np.sort(order[rank == r]) for r in range(world)]


def combine_f_evals(max_iterations, refresh_maps, stages: int, fsal: bool) -> int:
    """Global n_f_evals from per-shard (max iterations, refresh maps)."""
    mx = int(max(max_iterations)) if len(max_iterations) else 0
    if not fsal:
        return 1 + stages * mx
    union = np.zeros(max(len(m) for m in refresh_maps), dtype=bool)
    for m in refresh_maps:
        union[:len(m)] |= np.asarray(m, dtype=bool)
    return int(1 + (stages - 1) * mx + union[1:mx].sum())


def _csr_rows(offs: np.ndarray, idx: np.ndarray):
    """Row indices (into a CSR array with offsets ``offs``) of instances
    ``idx`` in that order, and the shard's own offsets -- vectorised."""
    counts = offs[idx + 1] - offs[idx]
    sub = np.zeros(len(idx) + 1, np.int64)
    np.cumsum(counts, out=sub[1:])
    rows = np.repeat(offs[idx] - sub[:-1], counts) + np.arange(int(sub[-1]), dtype=np.int64)
    return rows, sub


def subset_problem(problem: IvpBatch, idx) -> IvpBatch:
    """The instances ``idx`` of a validated batch (no per-instance Python
    work: the evaluation points are sliced as CSR rows)."""
    idx = np.asarray(idx, dtype=np.int64)
    sub = IvpBatch.__new__(IvpBatch)
    sub.y0 = problem.y0[idx]
    sub.t_start, sub.t_end = problem.t_start[idx], problem.t_end[idx]
    sub._te_list = None
    sub.te_shared = problem.te_shared
    if problem.te_shared:
        sub.te_values, sub.te_offsets = problem.te_values, None
    else:
        rows, offs = _csr_rows(problem.te_offsets, idx)
        sub.te_values, sub.te_offsets = problem.te_values[rows], offs
    return sub


def solve_sharded(problem: IvpBatch, f, *, group=None, cost_hint=None, gather_to: int | None = 0,
                  shard_solve=None, tableau=None, **solve_kw):
    """Solve ``problem`` split over the ranks of ``group``; every rank passes
    the same full problem description.  Returns the full Solution on rank
    ``gather_to`` (None elsewhere); with ``gather_to=None`` every rank gets
    (its indices, its shard Solution) with the global n_f_evals filled in."""
    import torch
    import torch.distributed as dist

    from .solver import solve
    from .tableau import method_of

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n = problem.batch_size
    parts = partition(n, world, cost_hint)
    idx = parts[rank]
    shard_solve = shard_solve or solve
    sub = subset_problem(problem, idx)
    sub_f = f.subset(idx) if hasattr(f, "subset") else f
    kw = dict(solve_kw)
    if cost_hint is not None and shard_solve is solve:
        kw["cost_hint"] = np.asarray(cost_hint)[idx]
    sol = shard_solve(sub, sub_f, tableau=tableau, with_refresh_map=True, **kw)
    method = method_of(tableau)
    stages, fsal = (2, False) if method == "heun" else (7, True)
    # the one exchange: global loop-iteration count and refresh iterations
    dev = torch.device("cuda", torch.cuda.current_device()) if (
        dist.is_initialized() and dist.get_backend(group) == "nccl") else torch.device("cpu")
    mx = torch.tensor([sol.stats.extra["max_iterations"]], dtype=torch.int64, device=dev)
    rmap = torch.from_numpy(np.ascontiguousarray(sol.stats.extra["refresh_map"])).to(dev)
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(rmap, op=dist.ReduceOp.MAX, group=group)
    nfe = combine_f_evals([int(mx.item())], [rmap.cpu().numpy()], stages, fsal)
    sol.stats.n_f_evals = np.full(len(idx), nfe, dtype=np.int64)
    if gather_to is None:
        return idx, sol
    # results travel as tensors (NCCL on the GPU box, gloo on CPU): one
    # (rows, 6) record per instance and the shard's flat ys rows (its CSR
    # layout; rows past an instance's n_emitted are never read)
    k, d = len(idx), problem.n_features
    rec = np.empty((k, 6), np.int64)
    rec[:, 0] = idx
    rec[:, 1], rec[:, 2] = sol.stats.n_steps, sol.stats.n_accepted
    rec[:, 3] = np.asarray(sol.stats.final_dt, np.float64).view(np.int64)
    rec[:, 4], rec[:, 5] = sol.status, sol.n_emitted
    flat = np.ascontiguousarray(np.asarray(sol.ys_flat, np.float64).reshape(-1, d))
    recs = gather_rows(torch.from_numpy(rec).to(dev), gather_to, group)
    ys_all = gather_rows(torch.from_numpy(flat).to(dev), gather_to, group)
    if rank != gather_to:
        return None
    counts = problem.eval_counts()
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=offs[1:])
    out = np.empty((int(offs[-1]), d))
    n_steps = np.zeros(n, np.int64)
    n_acc = np.zeros(n, np.int64)
    fdt = np.zeros(n)
    status = np.zeros(n, np.int64)
    n_emit = np.zeros(n, np.int64)
    for r, y in zip(recs, ys_all):  # one vectorised scatter per rank
        r, y = r.cpu().numpy(), y.cpu().numpy()
        ids = r[:, 0]
        n_steps[ids], n_acc[ids], status[ids], n_emit[ids] = r[:, 1], r[:, 2], r[:, 4], r[:, 5]
        fdt[ids] = r[:, 3].view(np.float64)
        if problem.te_shared:
            m = counts[0] if n else 0
            out.reshape(n, m, d)[ids] = y.reshape(len(ids), m, d)
        elif len(ids):
            rows, _ = _csr_rows(offs, ids)
            out[rows] = y[:len(rows)]
    stats = SolveStats(n_steps=n_steps, n_accepted=n_acc,
                       n_f_evals=np.full(n, nfe, dtype=np.int64), final_dt=fdt)
    if problem.te_shared:
        return Solution(out.reshape(-1), None, int(counts[0]) if n else 0, n_emit, stats, status, d)
    return Solution(out, offs, 0, n_emit, stats, status, d)


def gather_rows(t, dst: int = 0, group=None):
    """Gather tensors whose first dimension differs per rank to rank ``dst``
    (list in rank order there, None elsewhere): row counts are exchanged
    first, then every rank sends its rows padded to the longest shard."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [t]
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    rows = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(rows) for _ in range(world)]
    dist.all_gather(sizes, rows, group=group)
    sizes = [int(x.item()) for x in sizes]
    return _gather_padded(t, sizes, dst, group)


def _gather_padded(t, sizes, dst, group):
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    mrow = max(sizes)
    home = t.device
    t = _on_backend(t.contiguous(), group)
    if t.shape[0] != mrow:
        pad = torch.zeros((mrow,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        t = pad
    bufs = [torch.empty_like(t) for _ in sizes] if rank == dst else None
    dist.gather(t, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return [b[:s_].to(home) for b, s_ in zip(bufs, sizes)]


def _on_backend(t, group):
    """Collectives run on device tensors under NCCL; a gloo group (the CPU
    tests, or several ranks sharing one GPU) takes host copies."""
    import torch.distributed as dist

    if t.is_cuda and dist.get_backend(group) == "gloo":
        return t.cpu()
    return t


# ------------------------------------------------- device-side (NCCL) path --
def global_f_evals_device(out, stages: int = 7, fsal: bool = True, group=None):
    """The sharded solve's one real exchange, on device tensors: MAX
    all-reduce of the shards' loop-iteration counts and refresh maps (a byte
    per iteration, so MAX == OR), then n_f_evals = 1 + (S-1) max + #refresh
    iterations in [1, max) (FSAL) -- the reference's batch-global count
    (solver.py:184,224,239).  ``out`` is a ``solve_device(...,
    with_refresh_map=True)`` result; returns a 0-d int64 device tensor, no
    host sync."""
    import torch
    import torch.distributed as dist

    mx = out["max_iterations"].clone()
    rmap = out["refresh_map"].clone()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        mx, rmap = _on_backend(mx, group), _on_backend(rmap, group)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(rmap, op=dist.ReduceOp.MAX, group=group)
        mx, rmap = mx.to(out["max_iterations"].device), rmap.to(out["max_iterations"].device)
    if not fsal:
        return 1 + stages * mx[0]
    it = torch.arange(rmap.numel(), device=rmap.device)
    refresh = ((rmap != 0) & (it >= 1) & (it < mx[0])).sum()
    return 1 + (stages - 1) * mx[0] + refresh


def gather_device(out, dst: int = 0, group=None, keys=("n_steps", "n_accepted", "final_dt",
                                                        "status", "n_emitted", "ys")):
    """Gather the shards' per-instance results to rank ``dst`` with device
    collectives (NCCL over NVLink on the GPU box): returns a dict of
    concatenated tensors in rank order on ``dst``, None elsewhere.  Shards
    may differ in length (each rank's row count is exchanged first)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    res = {} if rank == dst else None
    for k in keys:
        t = out[k].contiguous()
        rows = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        sizes = [torch.zeros_like(rows) for _ in range(world)]
        dist.all_gather(sizes, rows, group=group)
        sizes = [int(x.item()) for x in sizes]
        mrow = max(sizes)
        pad = torch.zeros((mrow,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
        dist.gather(pad, bufs, dst=dst, group=group)
        if rank == dst:
            res[k] = torch.cat([b[:s_] for b, s_ in zip(bufs, sizes)])
    return res


def shard_plan(n: int, world: int, cost=None, device=None, group=None):
    """Device shard plan (``bode_partition``): returns (perm, sizes) with
    perm an (n,) int64 device tensor = shard 0's instance indices, then
    shard 1's, ... -- with ``cost`` dealt longest-first in a snake pattern
    (each shard stays longest-first, i.e. in its own queue order), without
    it contiguous blocks -- and sizes the per-shard counts (host ints, they
    depend on n and world only).  The longest-first order ranks equal cost
    buckets in arrival order (shared-memory atomics), so with several
    ranks, rank 0's plan is broadcast (8 bytes per instance over NVLink)
    and every rank works from the same permutation.  No host sync."""
    import torch

    from . import _abi

    lib = _abi.load()
    perm = torch.empty(n, dtype=torch.int64, device=device)
    sizes = (_abi.C.c_int64 * world)()
    st = torch.cuda.current_stream(device)
    keep = []
    if cost is not None:
        c = torch.as_tensor(cost, dtype=torch.float64, device=device).expand(n).contiguous()
        wsb = lib.bode_partition_workspace_size(n)
        ws = torch.empty(wsb, dtype=torch.uint8, device=device)
        keep += [c, ws]
        rc = lib.bode_partition(c.data_ptr(), n, world, perm.data_ptr(), sizes, ws.data_ptr(),
                                wsb, st.cuda_stream)
    else:
        rc = lib.bode_partition(None, n, world, perm.data_ptr(), sizes, None, 0, st.cuda_stream)
    _abi.check(rc)
    for t in keep:
        t.record_stream(st)
    import torch.distributed as dist
    if cost is not None and world > 1 and dist.is_initialized():
        p = _on_backend(perm, group)
        dist.broadcast(p, src=dist.get_global_rank(group, 0) if group is not None else 0,
                       group=group)
        perm = p.to(perm.device)
    return perm, [int(v) for v in sizes]


def solve_sharded_device(y0, t_start, t_end, f, *, t_eval=None, cost_hint=None, method="dopri5",
                         atol=1e-6, rtol=1e-6, dt0=None, group=None, gather_to: int | None = 0,
                         **solve_kw):
    """One batch solved across the ranks of ``group`` (one GPU each), device
    tensors in and out, no host sync until the gather.

    Every rank passes the same full batch description (resident on its
    device).  The batch is partitioned on the device (``shard_plan``:
    cost-aware when ``cost_hint`` is given), each rank gathers its shard's
    rows and solves them with the persistent kernel (queue order = the
    shard's longest-first row order), the batch-global ``n_f_evals`` is
    combined with two MAX all-reduces, and the per-instance results are
    gathered to rank ``gather_to`` over NCCL and put back in batch order.
    Returns the solve_device-style dict for the whole batch on
    ``gather_to`` (None on the other ranks); ``gather_to=None`` returns each
    rank's shard dict (with ``idx``) instead.  ``t_eval``: None, a 1-D tensor
    shared by every instance or an (n, m) tensor."""
    import torch
    import torch.distributed as dist

    from .solver import solve_device
    from .tableau import method_of

    on = dist.is_initialized()
    world = dist.get_world_size(group) if on else 1
    rank = dist.get_rank(group) if on else 0
    dev = y0.device
    n, d = y0.shape
    perm, sizes = shard_plan(n, world, cost_hint, dev, group)
    off = int(np.sum(sizes[:rank]))
    idx = perm[off:off + sizes[rank]]

    def rows(x):
        if isinstance(x, torch.Tensor) and x.dim() > 0 and x.shape[0] == n:
            return x.index_select(0, idx)
        return x

    te = t_eval if (t_eval is None or t_eval.dim() == 1) else rows(t_eval)
    sub_f = f.subset(idx) if hasattr(f, "subset") else f
    m = method_of(method)
    out = solve_device(rows(y0), rows(torch.as_tensor(t_start, dtype=torch.float64, device=dev)
                                      .expand(n)),
                       rows(torch.as_tensor(t_end, dtype=torch.float64, device=dev).expand(n)),
                       sub_f, t_eval=te, method=m, atol=rows(atol), rtol=rows(rtol),
                       dt0=rows(dt0), with_refresh_map=world > 1, **solve_kw)
    stages, fsal = (2, False) if m == "heun" else (7, True)
    nfe = global_f_evals_device(out, stages=stages, fsal=fsal, group=group) if world > 1 \
        else out["n_f_evals"][0]
    if gather_to is None:
        out["idx"], out["n_f_evals"] = idx, nfe.reshape(1)
        return out
    k = sizes[rank]
    rec = torch.stack([out["n_steps"], out["n_accepted"], out["final_dt"].view(torch.int64),
                       out["status"], out["n_emitted"]], dim=1)
    mpts = 0 if t_eval is None else (t_eval.numel() if t_eval.dim() == 1 else t_eval.shape[1])
    ys = out["ys"].reshape(k, mpts * d) if mpts else None
    if world > 1:
        recs = _gather_padded(rec, sizes, gather_to, group)
        yss = _gather_padded(ys, sizes, gather_to, group) if mpts else None
        if rank != gather_to:
            return None
        rec = torch.cat(recs)
        ys = torch.cat(yss) if mpts else None
    full = torch.empty_like(rec).index_copy_(0, perm, rec)
    res = dict(n_steps=full[:, 0], n_accepted=full[:, 1], final_dt=full[:, 2].view(torch.float64),
               status=full[:, 3], n_emitted=full[:, 4], n_f_evals=nfe.reshape(1),
               launches=out["launches"] + (4 if cost_hint is not None else 1))  # + the plan (LPT histogram, scan, scatter; permutation)
    res["ys"] = (torch.empty_like(ys).index_copy_(0, perm, ys).reshape(n * mpts, d) if mpts
                 else out["ys"][:0])
    return res


def solve_multi(y0, t_start, t_end, f, *, devices, t_eval=None, cost_hint=None,
                method="dopri5", atol=1e-6, rtol=1e-6, dt0=None, comms=None, gather: bool = True,
                **solve_kw):
    """One batch across several GPUs of THIS process through the C ABI's
    ``bode_solve_multi`` (no torch.distributed, no extra processes): the
    device shard plan (``shard_plan``, cost-aware with ``cost_hint``), each
    shard's rows copied to its device, the shard solves launched
    concurrently and the batch-global ``n_f_evals`` combined by the library
    (peer access, or NCCL when ``comms`` holds one ncclComm_t per shard, as
    integers, of a communicator over exactly these devices).  ``devices``
    lists CUDA device indices, one per shard (repeats allowed: several
    shards on one GPU).  Returns the solve_device-style dict in batch order
    on ``devices[0]`` (``gather=True``) or the list of shard dicts (each
    with ``idx``, its rows of the batch)."""
    import torch

    from . import _abi
    from .solver import solve_device
    from .tableau import method_of

    lib = _abi.load()
    ndev = len(devices)
    n, d = y0.shape
    if ndev < 1 or n < ndev:
        raise ValueError("solve_multi needs 1 <= len(devices) <= n")
    home = y0.device
    perm, sizes = shard_plan(n, ndev, cost_hint, home)
    m = method_of(method)
    shards, off = [], 0
    for k, dv in enumerate(devices):
        idx = perm[off:off + sizes[k]]
        off += sizes[k]
        dev = torch.device("cuda", int(dv))

        def rows(x, idx=idx, dev=dev):
            if isinstance(x, torch.Tensor) and x.dim() > 0 and x.shape[0] == n:
                return x.index_select(0, idx.to(x.device)).to(dev)
            if isinstance(x, torch.Tensor):
                return x.to(dev)
            return x

        ts = torch.as_tensor(t_start, dtype=torch.float64, device=home).expand(n)
        tn = torch.as_tensor(t_end, dtype=torch.float64, device=home).expand(n)
        te = None if t_eval is None else (t_eval.to(dev) if t_eval.dim() == 1 else rows(t_eval))
        sub_f = f.subset(idx.cpu().numpy()) if hasattr(f, "subset") else f
        with torch.cuda.device(dev):
            o = solve_device(rows(y0), rows(ts), rows(tn), sub_f, t_eval=te, method=m,
                             atol=rows(atol), rtol=rows(rtol), dt0=rows(dt0),
                             with_refresh_map=True, _launch=False, **solve_kw)
        o["idx"] = idx
        shards.append(o)
    arr = (_abi.SolveArgs * ndev)(*[o["_args"] for o in shards])
    cm = None if comms is None else (_abi.C.c_void_p * ndev)(*comms)
    _abi.check(lib.bode_solve_multi(arr, ndev, cm))
    for o in shards:
        o["launches"] = 3  # init pass, persistent integrator, finalize (+ the combine below)
    shards[0]["launches"] += 1
    if not gather:
        return shards
    # results back in batch order on the first device
    dev0 = torch.device("cuda", int(devices[0]))
    for dv in set(int(x) for x in devices):
        torch.cuda.synchronize(dv)  # (every shard's stream has seen the combine)
    keys = ("n_steps", "n_accepted", "final_dt", "status", "n_emitted")
    rec = torch.cat([torch.stack([o[k].view(torch.int64) if o[k].dtype == torch.float64 else o[k]
                                  for k in keys], dim=1).to(dev0) for o in shards])
    full = torch.empty_like(rec).index_copy_(0, perm.to(dev0), rec)
    res = {k: full[:, j] for j, k in enumerate(keys)}
    res["final_dt"] = res["final_dt"].contiguous().view(torch.float64)
    res["n_f_evals"] = shards[0]["n_f_evals"].to(dev0)
    mpts = 0 if t_eval is None else (t_eval.numel() if t_eval.dim() == 1 else t_eval.shape[1])
    if mpts:
        ys = torch.cat([o["ys"].reshape(-1, mpts * d).to(dev0) for o in shards])
        res["ys"] = torch.empty_like(ys).index_copy_(0, perm.to(dev0), ys).reshape(n * mpts, d)
    else:
        res["ys"] = shards[0]["ys"][:0].to(dev0)
    res["launches"] = sum(o["launches"] for o in shards)
    return res
