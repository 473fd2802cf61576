#!/usr/bin/env python3
"""Golden fixtures for expand_level SCHEDULES (operators / exhaustive flag changing from level to level),
generated from the UNMODIFIED reference.  Build container only (/root/reference does not travel):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden_schedules/make_schedule_golden.py

The reference API lets a caller pass a different operator set and a different `exhaustive` flag to every
`expand_level` call (reference engine.py:367-375).  tests/golden/ holds uniform runs; this file pins the mixed
ones: operator sets that change between levels, exhaustive levels on top of a level that was cut at its
separator, and non-exhaustive levels on top of such a level (where the reference truncates every chunk at its
first separating candidate, fresh or not -- engine.py:334-335 -- which the CUDA engine reproduces
with a scan pass and dead ordinal ranges; "engine_exact": false marks those cases).
"""
import hashlib
import json
import pathlib
import sys

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from ltlsynth import engine as ref_engine  # noqa: E402
from ltlsynth.traces import parse_specification as ref_parse  # noqa: E402

from paper_2504_18943_b200 import workloads  # noqa: E402
from paper_2504_18943_b200.traces import serialize_specification  # noqa: E402

FULL = ["not", "next", "future", "and", "until"]


def sched(*parts):
    out = []
    for ops, exhaustive, count in parts:
        out += [[list(ops), bool(exhaustive)]] * count
    return out


CASES = []
for wl, seed in (("c3", 1), ("c1", 3), ("spec2", 0)):
    CASES += [
        dict(name=f"{wl}_s{seed}_ops_a", workload=wl, seed=seed, engine_exact=True,
             schedule=sched((FULL, True, 6), (["not", "and", "until"], True, 2), (FULL, True, 2))),
        dict(name=f"{wl}_s{seed}_ops_b", workload=wl, seed=seed, engine_exact=True,
             schedule=sched((["not", "next", "until"], True, 5), (FULL, True, 4))),
        dict(name=f"{wl}_s{seed}_ops_c", workload=wl, seed=seed, engine_exact=True,
             schedule=sched((FULL, True, 5), (["future", "and", "until", "or"], True, 3))),
    ]
for seed, found in ((0, 4), (2, 5), (3, 6), (4, 8)):
    CASES += [
        dict(name=f"c1_s{seed}_cut_then_exhaustive", workload="c1", seed=seed, engine_exact=True,
             schedule=sched((FULL, False, found), (FULL, True, 3))),
        dict(name=f"c1_s{seed}_cut_then_nonexhaustive", workload="c1", seed=seed, engine_exact=False,
             schedule=sched((FULL, False, found + 2), (FULL, True, 1))),
    ]
for seed, found in ((0, 5), (1, 5)):  # 24-byte CMs: the wide path
    CASES += [
        dict(name=f"w32_s{seed}_cut_then_exhaustive", workload="w32", seed=seed, engine_exact=True,
             schedule=sched((FULL, False, found), (FULL, True, 3))),
        dict(name=f"w32_s{seed}_cut_then_nonexhaustive", workload="w32", seed=seed, engine_exact=False,
             schedule=sched((FULL, False, found + 2), (FULL, True, 1))),
    ]
CASES.append(dict(name="c3_s2_exh11", workload="c3", seed=2, engine_exact=True, schedule=sched((FULL, True, 11))))
# exhaustive levels that record a separating CM, then a NON-exhaustive level: chunk truncation over complete levels
# (the associativity pruning of AND blocks must be off there: the dead ranges delete the witnesses it relies on)
NAN = ["not", "and", "next"]
for batch in (64, 65536):
    CASES.append(dict(name=f"c1_s3_nan_exh7_then_nonexhaustive_b{batch}", workload="c1", seed=3, engine_exact=False,
                      batch_size=batch, schedule=sched((NAN, True, 7), (NAN, False, 2), (NAN, True, 1))))
for seed in (0, 2, 4):
    CASES.append(dict(name=f"c1_s{seed}_exh_then_nonexhaustive_b256", workload="c1", seed=seed, engine_exact=False,
                      batch_size=256, schedule=sched((FULL, True, 7), (FULL, False, 2))))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = []
    for case in CASES:
        spec = workloads.named_workload(case["workload"], case["seed"])
        rspec = ref_parse(serialize_specification(spec))
        store = ref_engine.CandidateStore(rspec)
        levels = []
        for cost, (ops, exhaustive) in enumerate(case["schedule"], 1):
            cfg = ref_engine.EngineConfig(exhaustive=exhaustive, threads=1, batch_size=case.get("batch_size", 65536))
            stats = ref_engine.RunStats()
            n, sep = ref_engine.expand_level(store, cost, tuple(ops), config=cfg, stats=stats)
            lv = store.level(cost)
            levels.append(dict(cost=cost, n=int(n), sep_gid=None if sep is None else int(sep),
                               constructed=int(stats.constructed), cms_sha256=sha(lv.cms), op_sha256=sha(lv.op),
                               left_sha256=sha(lv.left), right_sha256=sha(lv.right)))
        out.append(dict(case, levels=levels))
        print(case["name"], [(l["n"], l["sep_gid"]) for l in levels])
    (HERE / "schedules.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
