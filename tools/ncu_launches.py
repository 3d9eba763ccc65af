"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel:
launches, total / mean us, share.   python tools/ncu_launches.py launches.csv"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        tot[r[ki][:90]] += us
        cnt[r[ki][:90]] += 1
    s = sum(tot.values())
    print(f"| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.1f} | {100 * tot[k] / s:.1f}% |")
    print(f"total {s / 1e3:.2f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
