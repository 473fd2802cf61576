"""The reference's behavioural known answers, checked on the CUDA engine through the public API."""

import types

import pytest

import behaviour
from paper_2504_18943_b200 import engine
from paper_2504_18943_b200.formulas import DEFAULT_OPERATORS

pytestmark = pytest.mark.gpu


class EngineBackend:
    name = "b200"

    def store(self, spec):
        return engine.CandidateStore(spec)

    def expand(self, store, level, ops=DEFAULT_OPERATORS, exhaustive=False, batch=1 << 16, memory_mb=1 << 20):
        cfg = engine.EngineConfig(exhaustive=exhaustive, batch_size=batch, memory_budget_mb=memory_mb)
        stats = engine.RunStats()
        n_new, sep = engine.expand_level(store, level, ops, config=cfg, stats=stats)
        return n_new, sep, stats.constructed

    def close(self, store):
        store.close()

    def reconstruct(self, store, gid):
        return engine.reconstruct(store, gid)

    def synth(self, spec, **kw):
        r = engine.synthesize(spec, engine.EngineConfig(**kw))
        return types.SimpleNamespace(outcome=r.outcome, cost=r.cost, formula=r.formula, constructed=r.stats.constructed,
                                     unique=r.stats.unique, failure=r.failure, max_cost_reached=r.stats.max_cost_reached)


@pytest.mark.parametrize("check", behaviour.ALL_CHECKS, ids=lambda f: f.__name__)
def test_engine(check):
    check(EngineBackend())
