#!/usr/bin/env python3
"""One short line per bench.py JSON line on stdin (workload, ms/step, enumerate / finalise ms, roofline, e2e)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline", {})
    print(" ".join(sys.argv[1:]), d["config"]["workload"], "ms/step", round(d["ms_per_step"], 3),
          "enum", round(r.get("kernel_ms_per_step", 0), 3), "fin", round(r.get("finalize_ms_per_step", 0), 3),
          "frac", round(r.get("frac", 0), 4), "e2e_ms", round(d["e2e"].get("time_to_solution_ms", 0), 3),
          "unique/s", f"{d['value']:.4g}", "e2e unique/s", f"{d['e2e']['value']:.4g}")
