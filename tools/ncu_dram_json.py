#!/usr/bin/env python3
"""Per-kernel DRAM traffic of one search from an ncu metrics pass, as the JSON bench.py reads.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
        --clock-control none --csv --log-file gpurun_out/x.csv python tools/run_workload.py spec2
    python tools/ncu_dram_json.py gpurun_out/x.csv "<command>" > profiles/rNN_dram_spec2.json

`enumerate_*` sums the construction + dedup launches (every kernel whose name contains "level_kernel").
"""
import collections
import csv
import json
import re
import sys


def main() -> int:
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        launches.setdefault(r[ii], {"kernel": re.sub(r"\(.*", "", r[ki]).replace("void ", "")})[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.OrderedDict()
    for e in launches.values():
        a = agg.setdefault(e["kernel"], {"kernel": e["kernel"], "launches": 0, "us": 0.0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0})
        a["launches"] += 1
        a["us"] += e.get("gpu__time_duration.sum", 0.0) / 1e3
        a["dram_read_bytes"] += e.get("dram__bytes_read.sum", 0.0)
        a["dram_write_bytes"] += e.get("dram__bytes_write.sum", 0.0)
    total = sum(a["us"] for a in agg.values()) or 1.0
    kernels = sorted(agg.values(), key=lambda a: -a["us"])
    for a in kernels:
        a["us"] = round(a["us"], 1)
        a["share"] = round(a["us"] / total, 4)
    enum = [a for a in kernels if "level_kernel" in a["kernel"]]
    out = {
        "command": sys.argv[2] if len(sys.argv) > 2 else "",
        "kernels": kernels,
        "enumerate_launches": sum(a["launches"] for a in enum),
        "enumerate_us": round(sum(a["us"] for a in enum), 1),
        "enumerate_dram_bytes": sum(a["dram_read_bytes"] + a["dram_write_bytes"] for a in enum),
    }
    json.dump(out, sys.stdout, indent=1)
    print()
    return 0


if __name__ == "__main__":
    sys.exit(main())
