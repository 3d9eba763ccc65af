"""Summarise ncu captures for profiles/ (run here, on the CPU side).

    python tools/ncu_summary.py launches <launches.csv>        # share per kernel
    python tools/ncu_summary.py full <report.ncu-rep>          # key metrics
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(list)
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) > vi and r[vi]:
            tot[r[ki]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    # the roofline probes (bench.py's in-run peak measurement) are not part of
    # the solve: listed, but excluded from the shares
    grand = sum(sum(v) for k, v in tot.items() if "probe" not in k)
    print("| kernel | launches | total us | mean us | share of solve |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
        share = "probe (excluded)" if "probe" in k else f"{sum(v)/grand:.1%}"
        print(f"| `{k[:90]}` | {len(v)} | {sum(v):.1f} | {sum(v)/len(v):.1f} | {share} |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"### {name[:120]}")
        print("| metric | value | unit |")
        print("|---|---|---|")
        for k in KEYS:
            if k in h:
                print(f"| {k} | {v[h.index(k)]} | {u[h.index(k)]} |")
        stall = [(c, v[i]) for i, c in enumerate(h)
                 if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
        stall = sorted(((c.split("stalled_")[1].split("_per_issue")[0], float(x or 0)) for c, x in stall),
                       key=lambda t: -t[1])[:8]
        print("\nTop warp stall reasons (warps per issue-active cycle): " +
              ", ".join(f"{c} {x:.2f}" for c, x in stall))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
