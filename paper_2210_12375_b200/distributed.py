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
           "global_f_evals_device", "gather_device"]


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


def subset_problem(problem: IvpBatch, idx) -> IvpBatch:
    idx = np.asarray(idx)
    if problem.te_shared:
        te = problem.te_values
    else:
        o = problem.te_offsets
        te = [problem.te_values[o[i]:o[i + 1]] for i in idx]
    return IvpBatch(problem.y0[idx], problem.t_start[idx], problem.t_end[idx], te)


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
    payload = (idx, [np.asarray(y) for y in sol.ys], sol.stats.n_steps, sol.stats.n_accepted,
               sol.stats.final_dt, sol.status, sol.n_emitted)
    if world > 1:
        objs = [None] * world if rank == gather_to else None
        dist.gather_object(payload, objs, dst=gather_to, group=group)
    else:
        objs = [payload]
    if rank != gather_to:
        return None
    d = problem.n_features
    ys = [None] * n
    n_steps = np.zeros(n, np.int64)
    n_acc = np.zeros(n, np.int64)
    fdt = np.zeros(n)
    status = np.zeros(n, np.int64)
    n_emit = np.zeros(n, np.int64)
    for ids, y, ns, na, fd, st, ne in objs:
        for j, i in enumerate(ids):
            ys[i] = y[j]
        n_steps[ids], n_acc[ids], fdt[ids], status[ids], n_emit[ids] = ns, na, fd, st, ne
    counts = problem.eval_counts()
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=offs[1:])
    flat = np.full((int(offs[-1]), d), np.nan)
    for i in range(n):
        flat[offs[i]:offs[i] + len(ys[i])] = ys[i]
    stats = SolveStats(n_steps=n_steps, n_accepted=n_acc,
                       n_f_evals=np.full(n, nfe, dtype=np.int64), final_dt=fdt)
    return Solution(flat, offs, 0, n_emit, stats, status, d)


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
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(rmap, op=dist.ReduceOp.MAX, group=group)
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
