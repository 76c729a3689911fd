"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel.

usage: python scripts/launch_summary.py launches.csv [--steps S]
Per-launch ncu times are cold-cache and serialised: compare SHARES, not absolutes.
"""
import collections
import csv
import re
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def summarise(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).strip()
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        tot[name] += us
        cnt[name] += 1
    return tot, cnt


if __name__ == "__main__":
    tot, cnt = summarise(sys.argv[1])
    T = sum(tot.values())
    print(f"# {sys.argv[1]}: {sum(cnt.values())} launches, {T:.1f} us total (ncu, serialised)")
    print(f"{'share':>7} {'total_us':>11} {'launches':>8} {'avg_us':>8}  kernel")
    for k, v in tot.most_common():
        print(f"{100 * v / T:6.2f}% {v:11.1f} {cnt[k]:8d} {v / cnt[k]:8.2f}  {k}")
