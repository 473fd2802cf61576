"""expand_level schedules on the CUDA engine, against fixtures of the unmodified reference.

The reference API takes a different operator set and exhaustive flag on every expand_level call
(reference engine.py:367-375).  The associativity pruning of the narrow path is sound only
while every stored level is complete and all levels were built with one operator set, so these cases break
that on purpose -- the operator set changes between levels, exhaustive levels are built on top of a level that
was cut at its separator -- and every level must still be the reference's, bit for bit
(tests/golden_schedules/schedules.json; the same file pins the CPU oracle in test_oracle_schedules.py).

Cases with "engine_exact": false are NON-exhaustive levels over a store that already holds a separating CM,
where the reference truncates every chunk at its first separating candidate, fresh or not; the engine
reproduces that with a scan pass and dead ordinal ranges (c1 = narrow path, w32 = wide path),
so they must match as well.
"""

import json
import pathlib

import pytest

from helpers import assert_level_matches_golden
from paper_2504_18943_b200 import engine, workloads

pytestmark = pytest.mark.gpu

SCHEDULES = json.loads((pathlib.Path(__file__).resolve().parent / "golden_schedules" / "schedules.json").read_text())


@pytest.mark.parametrize("case", SCHEDULES, ids=lambda c: c["name"])
def test_engine_reproduces_reference_schedule(case):
    spec = workloads.named_workload(case["workload"], case["seed"])
    store = engine.CandidateStore(spec)
    try:
        for (ops, exhaustive), gl in zip(case["schedule"], case["levels"]):
            cfg = engine.EngineConfig(exhaustive=exhaustive, batch_size=case.get("batch_size", 65536))
            stats = engine.RunStats()
            n_new, sep = engine.expand_level(store, gl["cost"], tuple(ops), config=cfg, stats=stats)
            where = f"{case['name']} cost {gl['cost']}"
            assert (n_new, sep, stats.constructed) == (gl["n"], gl["sep_gid"], gl["constructed"]), where
            gold = dict(gl, base=store.level(gl["cost"]).base)
            assert_level_matches_golden(store.level(gl["cost"]), gold, where)
    finally:
        store.close()
