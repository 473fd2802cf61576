#!/usr/bin/env python3
"""Hot source lines of each kernel in an `ncu -i X.ncu-rep --page source --csv --print-source sass,cuda` dump.

Aggregates warp-stall samples per CUDA source line (file:line) and prints the top N per kernel with
the dominant stall reason.  Usage: ncu_source_hot.py dump.csv [N]
"""
import collections
import csv
import sys


def main() -> int:
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
    kernel, hdr = None, None
    per_kernel = collections.OrderedDict()
    cur_src = ""
    for row in csv.reader(open(path, errors="replace")):
        if not row:
            continue
        if row[0] == "File Path":
            cur_src = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Function Name":
            kernel = row[1].replace("ltlb200::", "").replace("(int)", "")[:70]
            per_kernel.setdefault(kernel, collections.defaultdict(lambda: collections.Counter()))
            hdr = None
            continue
        if row[0] in ("Line No", "Address") or (len(row) > 3 and "Warp Stall Sampling (All Samples)" in row):
            hdr = row
            continue
        if hdr is None or kernel is None or len(row) != len(hdr):
            continue
        rec = dict(zip(hdr, row))
        # the merged view repeats the CUDA source line in the first "Source" column
        line_no = row[0]
        if not line_no:  # a SASS row; the CUDA line above it already carries the aggregate
            continue
        src = row[1]
        key = f"{cur_src}:{line_no}: {src.strip()[:90]}"
        c = per_kernel[kernel][key]
        try:
            c["samples"] += int(rec.get("# Samples") or 0)
            c["inst"] += int(rec.get("Instructions Executed") or 0)
        except ValueError:
            continue
        for k, v in rec.items():
            if k.startswith("stall_") and "Not Issued" not in k and v:
                try:
                    c[k] += int(v)
                except ValueError:
                    pass
    for kernel, lines in per_kernel.items():
        total = sum(c["samples"] for c in lines.values()) or 1
        tot_inst = sum(c["inst"] for c in lines.values()) or 1
        print(f"== {kernel}: {total} samples, {tot_inst} warp instructions")
        for key, c in sorted(lines.items(), key=lambda kv: -kv[1]["samples"])[:top]:
            stalls = sorted(((v, k) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:2]
            why = ", ".join(f"{k[6:]} {100 * v // max(c['samples'], 1)}%" for v, k in stalls)
            print(f"  {100 * c['samples'] / total:5.1f}%  inst {100 * c['inst'] / tot_inst:5.1f}%  {key}   [{why}]")
    return 0


if __name__ == "__main__":
    sys.exit(main())
