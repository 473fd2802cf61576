#!/usr/bin/env python3
"""Generate the golden fixtures in this directory from the UNMODIFIED reference.

Run in the build container only (the reference lives at /root/reference, which
does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--only NAME] [--slow]

For every case it runs the reference's own ``CandidateStore`` / ``expand_level``
(or ``synthesize``) on a specification produced by this repo's workload
generator (handed over as ``.trc`` text, so the reference parses it itself) and
records, per cost level: entry count, base id, the ``constructed`` delta, the
returned separator id and sha256 digests of the level's ``cms`` / ``op`` /
``left`` / ``right`` arrays exactly as numpy lays them out.  The parity tests
compare the C oracle (CPU) and the CUDA engine (GPU) with these files.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import pathlib
import sys
import time

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import ltlsynth  # noqa: E402  (the reference)
from ltlsynth import engine as ref_engine  # noqa: E402
from ltlsynth.formulas import to_text as ref_to_text  # noqa: E402

from paper_2504_18943_b200 import workloads  # noqa: E402
from paper_2504_18943_b200.traces import serialize_specification  # noqa: E402

DEFAULT_OPS = ("not", "next", "future", "and", "until")

# name, workload, seed, kind, options
#   kind "levels": expand_level for cost 1..max_cost (no executor), record every level
#   kind "synth" : synthesize(), record the result (+ levels are not visible, so only stats)
CASES = [
    dict(name="spec1_exh10", workload="spec1", max_cost=10, exhaustive=True),
    dict(name="spec1_found", workload="spec1", max_cost=6, exhaustive=False),
    dict(name="spec1_found_b1", workload="spec1", max_cost=6, exhaustive=False, batch_size=1),
    dict(name="spec1_found_b3", workload="spec1", max_cost=6, exhaustive=False, batch_size=3),
    dict(name="spec1_found_b7", workload="spec1", max_cost=6, exhaustive=False, batch_size=7),
    dict(name="spec1_or_exh7", workload="spec1", max_cost=7, exhaustive=True, ops=DEFAULT_OPS + ("or",)),
    dict(name="spec1_or_found", workload="spec1", max_cost=6, exhaustive=False, ops=DEFAULT_OPS + ("or",)),
    dict(name="spec1_fuo_exh7", workload="spec1", max_cost=7, exhaustive=True, ops=("future", "until", "or")),
    dict(name="spec2_exh11", workload="spec2", max_cost=11, exhaustive=True),
    dict(name="spec2_fuo_exh8", workload="spec2", max_cost=8, exhaustive=True, ops=("future", "until", "or")),
    dict(name="spec2_b5_exh7", workload="spec2", max_cost=7, exhaustive=True, batch_size=5),
    dict(name="c1_s0", workload="c1", seed=0, max_cost=14, exhaustive=False),
    dict(name="c1_s1", workload="c1", seed=1, max_cost=14, exhaustive=False),
    dict(name="c1_s2", workload="c1", seed=2, max_cost=14, exhaustive=False),
    dict(name="c1_s3", workload="c1", seed=3, max_cost=14, exhaustive=False),
    dict(name="c1_s4", workload="c1", seed=4, max_cost=14, exhaustive=False),
    dict(name="c1_s1_exh9", workload="c1", seed=1, max_cost=9, exhaustive=True),
    dict(name="c3_s0_exh10", workload="c3", seed=0, max_cost=10, exhaustive=True),
    dict(name="c3wide_s0_exh8", workload="c3wide", seed=0, max_cost=8, exhaustive=True),
    dict(name="c4-512_s0_exh8", workload="c4-512", seed=0, max_cost=8, exhaustive=True),
    dict(name="c4-1024_s0_exh8", workload="c4-1024", seed=0, max_cost=8, exhaustive=True),
    dict(name="c4xl_s0_exh7", workload="c4xl", seed=0, max_cost=7, exhaustive=True),
    dict(name="c5_s0_exh8", workload="c5", seed=0, max_cost=8, exhaustive=True),
    dict(name="c5_s0_or_exh7", workload="c5", seed=0, max_cost=7, exhaustive=True, ops=DEFAULT_OPS + ("or",)),
    dict(name="w32_s0_exh8", workload="w32", seed=0, max_cost=8, exhaustive=True),
    dict(name="w32_s1_found", workload="w32", seed=1, max_cost=12, exhaustive=False),
    dict(name="w64_s0_exh8", workload="w64", seed=0, max_cost=8, exhaustive=True),
    dict(name="w64_s1_found", workload="w64", seed=1, max_cost=12, exhaustive=False),
    dict(name="w32n_s0_exh9", workload="w32n", seed=0, max_cost=9, exhaustive=True),
    dict(name="w32n_s2_found", workload="w32n", seed=2, max_cost=12, exhaustive=False),
    dict(name="w64n_s0_exh9", workload="w64n", seed=0, max_cost=9, exhaustive=True),
    dict(name="w64n_s3_found", workload="w64n", seed=3, max_cost=12, exhaustive=False),
    dict(name="c3_s1_found", workload="c3", seed=1, max_cost=12, exhaustive=False),
    dict(name="c3_s0_b1000_found", workload="c3", seed=2, max_cost=12, exhaustive=False, batch_size=1000),
]
SLOW_CASES = [
    # the paper's 7+7 example to its cost-16 solution (about a minute of reference time)
    dict(name="spec2_found", workload="spec2", max_cost=16, exhaustive=False),
    dict(name="c3_s0_exh12", workload="c3", seed=0, max_cost=12, exhaustive=True),
    dict(name="c5_s0_exh10", workload="c5", seed=0, max_cost=10, exhaustive=True),
    dict(name="c5_s0_exh11", workload="c5", seed=0, max_cost=11, exhaustive=True),          # 19.0 M CMs of 128 bytes
    dict(name="c4-1024_s0_exh10", workload="c4-1024", seed=0, max_cost=10, exhaustive=True),  # 0.98 M CMs of 128 bytes
]


def digest(arr) -> str:
    return hashlib.sha256(arr.tobytes()).hexdigest()


def run_case(case: dict) -> dict:
    spec_mine = workloads.named_workload(case["workload"], case.get("seed", 0))
    trc = serialize_specification(spec_mine)
    spec = ltlsynth.parse_specification(trc)
    ops = ref_engine.normalize_operators(case.get("ops", DEFAULT_OPS))
    cfg = ref_engine.EngineConfig(
        operators=ops,
        max_cost=case["max_cost"],
        exhaustive=case["exhaustive"],
        batch_size=case.get("batch_size", 1 << 16),
        threads=1,
        time_budget_s=36000.0,
        memory_budget_mb=48000,
    )
    store = ref_engine.CandidateStore(spec)
    stats = ref_engine.RunStats()
    levels = []
    found = None
    t0 = time.perf_counter()
    for cost in range(1, cfg.max_cost + 1):
        before = stats.constructed
        n_new, sep = ref_engine.expand_level(store, cost, ops, config=cfg, stats=stats)
        lv = store.level(cost)
        levels.append(
            dict(
                cost=cost,
                n=int(lv.n),
                base=int(lv.base),
                constructed=int(stats.constructed - before),
                sep_gid=None if sep is None else int(sep),
                cms_sha256=digest(lv.cms),
                op_sha256=digest(lv.op),
                left_sha256=digest(lv.left),
                right_sha256=digest(lv.right),
            )
        )
        assert n_new == lv.n
        if sep is not None and found is None:
            found = (int(sep), cost)
            if not cfg.exhaustive:
                break
    elapsed = time.perf_counter() - t0
    out = dict(
        name=case["name"],
        workload=case["workload"],
        seed=case.get("seed", 0),
        operators=list(ops),
        max_cost=cfg.max_cost,
        exhaustive=cfg.exhaustive,
        batch_size=cfg.batch_size,
        trace_count=spec.trace_count,
        lane_bits=int(store.dtype.itemsize * 8),
        spec_trc_sha256=hashlib.sha256(trc.encode()).hexdigest(),
        levels=levels,
        constructed=int(stats.constructed),
        unique=int(store.total),
        found_gid=None if found is None else found[0],
        found_cost=None if found is None else found[1],
        formula=None if found is None else ref_to_text(ref_engine.reconstruct(store, found[0]), spec.alphabet),
        reference_elapsed_s=round(elapsed, 3),
        generator="tests/golden/make_golden.py on ltlsynth " + ltlsynth.__version__,
    )
    # cross-check the reference's own top-level entry point on the cheap cases
    if elapsed < 5.0:
        res = ref_engine.synthesize(spec, cfg)
        assert res.stats.constructed == out["constructed"], (res.stats, out["constructed"])
        assert res.stats.unique == out["unique"]
        if found is not None:
            assert ref_to_text(res.formula, spec.alphabet) == out["formula"] and res.cost == out["found_cost"]
    return out


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--slow", action="store_true", help="also run the minute-long cases")
    args = ap.parse_args()
    cases = CASES + (SLOW_CASES if args.slow else [])
    if args.only:
        cases = [c for c in CASES + SLOW_CASES if c["name"] == args.only]
    for case in cases:
        t0 = time.perf_counter()
        out = run_case(case)
        path = HERE / (case["name"] + ".json")
        path.write_text(json.dumps(out, indent=1) + "\n")
        print(f"{case['name']}: unique={out['unique']} constructed={out['constructed']} "
              f"formula={out['formula']!r} ({time.perf_counter() - t0:.1f}s)", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
