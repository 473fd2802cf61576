#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, time, share.

    python tools/ncu_launch_summary.py gpurun_out/launches.csv [--skip N] > profiles/rNN_launches_summary.txt
"""
import collections
import csv
import re
import sys


def main() -> int:
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1 + skip:]:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else v * 1e3 if r[ui] == "ms" else v
        agg[name][0] += 1
        agg[name][1] += v
    total = sum(v for _, v in agg.values())
    print(f"# {path}: {len(rows) - 1 - skip} launches, {total / 1e3:.3f} ms of kernel time (cold-cache, serialised under ncu)")
    print(f"{'kernel':64s} {'launches':>8s} {'us':>12s} {'share':>7s}")
    for name, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:64s} {c:8d} {v:12.1f} {100 * v / total:6.1f}%")
    return 0


if __name__ == "__main__":
    sys.exit(main())
