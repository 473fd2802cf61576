"""EXTENSION on the CUDA engine: G and per-operator cost weights against the CPU oracle's extension (which
tests/test_extension_oracle.py pins to semantic identities and brute force; the reference has neither, so parity
with the reference is unpinned here and stays pinned everywhere else because the extension is off by default)."""

import pytest

import oracle
from helpers import assert_levels_equal
from paper_2504_18943_b200 import engine, to_text, workloads

pytestmark = pytest.mark.gpu
EXT_OPS = ("not", "next", "future", "globally", "and", "until")


@pytest.mark.parametrize("workload,seed,max_cost,ops,weights", [
    ("spec1", 0, 8, EXT_OPS, None),
    ("c1", 2, 9, EXT_OPS + ("or",), None),
    ("spec2", 0, 10, EXT_OPS, {"until": 2}),
    ("c3", 0, 11, ("not", "next", "future", "and", "until"), {"atom": 2, "and": 2, "next": 3}),
    ("c5", 0, 8, EXT_OPS, {"globally": 2}),      # 128-byte CMs: the wide kernels
    ("w64n", 0, 9, EXT_OPS, {"future": 2}),      # 64-bit lanes
])
def test_engine_levels_equal_the_oracle_extension(workload, seed, max_cost, ops, weights):
    spec = workloads.named_workload(workload, seed)
    store = engine.CandidateStore(spec, operator_weights=weights)
    ref = oracle.OracleStore(spec, operator_weights=weights)
    cfg = engine.EngineConfig(operators=ops, exhaustive=True, extended_grammar=True, operator_weights=weights, memory_budget_mb=1 << 20)
    try:
        stats = engine.RunStats()
        for cost in range(1, max_cost + 1):
            before = stats.constructed
            n_new, sep = engine.expand_level(store, cost, ops, config=cfg, stats=stats)
            o_new, o_sep, o_delta, _ = ref.expand_level(cost, ops, True, cfg.batch_size, memory_budget_mb=1 << 20)
            where = f"{workload} cost {cost} weights {weights}"
            assert (n_new, sep, stats.constructed - before) == (o_new, o_sep, o_delta), where
            assert_levels_equal(store.level(cost), ref.level(cost), where)
    finally:
        store.close()


@pytest.mark.parametrize("workload,seed,weights", [("spec1", 0, {"until": 3}), ("c1", 1, {"globally": 1, "not": 2}),
                                                    ("c1", 4, {"atom": 2}), ("w32", 1, {"and": 2})])
def test_synthesize_with_extension_returns_the_oracles_witness(workload, seed, weights):
    spec = workloads.named_workload(workload, seed)
    cfg = engine.EngineConfig(operators=EXT_OPS, extended_grammar=True, operator_weights=weights, max_cost=14)
    res = engine.synthesize(spec, cfg)
    want = oracle.synthesize(spec, operators=EXT_OPS, max_cost=14, operator_weights=weights)
    assert (res.outcome, res.cost, res.stats.unique, res.stats.constructed) == (want.outcome, want.cost, want.unique, want.constructed)
    if want.formula is not None:
        assert to_text(res.formula, spec.alphabet) == to_text(want.formula, spec.alphabet)
