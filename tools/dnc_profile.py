#!/usr/bin/env python3
"""Divide-and-conquer on the GPU: sequential leaves (the reference's order of execution) against
concurrent leaves, on the golden cases of tests/golden_callers/dnc_cases.json and a larger spec."""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2504_18943_b200 import dnc, parse_specification, workloads
from paper_2504_18943_b200.engine import EngineConfig

cases = json.loads((pathlib.Path(__file__).resolve().parent.parent / "tests" / "golden_callers" / "dnc_cases.json").read_text())
todo = [(c["name"], parse_specification(c["trc"]), EngineConfig(**c["config"])) for c in cases if c["name"].startswith(("random_s105", "random_s102", "spec2_threshold4"))]
todo.append(("synthetic 32+32 x len 6, threshold 8", workloads.synthetic_spec(7, 2, 32, 32, 6, False), EngineConfig(max_cost=12)))
for name, spec, cfg in todo:
    row = []
    for workers in (1, 4, 16):
        dnc.synthesize_dnc(spec, cfg, workers=workers)
        t0 = time.perf_counter()
        for _ in range(3):
            res = dnc.synthesize_dnc(spec, cfg, workers=workers)
        row.append((workers, round(1e3 * (time.perf_counter() - t0) / 3, 2)))
    leaves = []
    dnc._unfold(spec, cfg, "root", leaves)
    print(f"{name}: {len(leaves)} leaves, outcome {res.outcome}, cost {res.cost}, ms by workers {row}", flush=True)
