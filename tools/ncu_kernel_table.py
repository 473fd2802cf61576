#!/usr/bin/env python3
"""One line per launch from an `ncu --metrics ... --csv` log: kernel, grid, and the requested metrics."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii, gi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ii], {"k": r[ki].replace("void ", "")[:34], "g": r[gi]})[r[mi]] = r[vi]
for i, e in d.items():
    t = float(e.get("gpu__time_duration.sum", "0").replace(",", "")) / 1e3
    rd = float(e.get("dram__bytes_read.sum", "0").replace(",", "")) / 1e6
    wr = float(e.get("dram__bytes_write.sum", "0").replace(",", "")) / 1e6
    inst = float(e.get("smsp__inst_executed.sum", "0").replace(",", "")) / 1e6
    print(f"{i:>4s} {e['k']:34s} {e['g']:>12s} {t:9.1f} us  rd {rd:8.1f} MB  wr {wr:8.1f} MB  inst {inst:7.1f} M")
