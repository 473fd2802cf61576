"""EXTENSION beyond the reference grammar: the operator G and per-operator cost weights.

The reference has neither (formulas.py:59,65-71), so no golden output exists: PARITY
UNPINNED.  What pins the CPU oracle's extension instead:

  * G's bit semantics equal the reference connectives' reading of !F!x on every stored CM (the reference-pinned
    kernels k_not / k_future of the same oracle), and the naive finite-trace semantics of `Globally`;
  * minimality under weights: oracle.synthesize == dedup-free brute force over weighted formula trees (the
    reference's oracle.py:96-109 pattern) on random small specifications;
  * with all weights 1 and G disabled nothing changes (the goldens of test_oracle_golden.py).
The CUDA engine is then compared with this oracle in test_gpu_extension.py.
"""

import random

import numpy as np
import pytest

import oracle
from behaviour import random_spec, truth_cm
from paper_2504_18943_b200 import formulas as F
from paper_2504_18943_b200 import semantics, to_text, workloads
from paper_2504_18943_b200.engine import EngineConfig, normalize_operators

EXT_OPS = ("not", "next", "future", "globally", "and", "until")


def test_reference_behaviour_is_the_default():
    with pytest.raises(ValueError, match="unknown operators"):
        normalize_operators(("not", "globally"))
    with pytest.raises(ValueError, match="unknown operators"):
        EngineConfig(operators=("globally", "and"))
    with pytest.raises(ValueError, match="extension"):
        EngineConfig(operator_weights={"until": 3})
    cfg = EngineConfig(operators=EXT_OPS, extended_grammar=True, operator_weights={"until": 3, "atom": 1})
    assert cfg.weights == {"until": 3, "atom": 1} and hash(cfg) is not None
    assert normalize_operators(EXT_OPS, extended=True) == EXT_OPS


def test_globally_parses_prints_and_means_not_future_not():
    spec = workloads.spec1()
    f = F.parse_formula("G (a | X b) U !G c", spec.alphabet)
    assert to_text(f, spec.alphabet) == "G (a | X b) U !G c"
    assert F.weighted_cost(f, {"globally": 4, "atom": 2}) == 3 * 2 + 2 * 4 + 4
    rng = random.Random(7)
    for _ in range(50):
        sp = random_spec(rng, 2, 4, 6)
        g = F.Atom(rng.randrange(2))
        for _ in range(rng.randrange(4)):
            g = rng.choice([F.Not, F.Next, F.Future, F.Globally])(g)
        lhs, rhs = F.Globally(g), F.Not(F.Future(F.Not(g)))
        for tr in sp.positives + sp.negatives:
            assert semantics._truth_table(tr, lhs) == semantics._truth_table(tr, rhs) == semantics._truth_table_fast(tr, lhs)


def test_oracle_globally_rows_are_the_truth_tables_of_their_formulas():
    spec = workloads.named_workload("c1", 2)
    store = oracle.OracleStore(spec)
    for cost in range(1, 6):
        store.expand_level(cost, EXT_OPS, True)
    seen_g = 0
    for cost in range(2, 6):
        lv = store.level(cost)
        for k in range(lv.n):
            formula = oracle.reconstruct(store, lv.base + k)
            seen_g += isinstance(formula, F.Globally)
            assert np.array_equal(lv.cms[k], truth_cm(spec, formula, store.dtype)), to_text(formula, spec.alphabet)
    assert seen_g > 0


@pytest.mark.parametrize("weights", [{"until": 3}, {"atom": 2, "not": 1, "and": 2}, {"globally": 1, "future": 2, "next": 3}])
def test_oracle_minimality_under_weights_against_bruteforce(weights):
    rng = random.Random(hash(tuple(sorted(weights.items()))) & 0xFFFF)
    checked = 0
    for _ in range(25):
        spec = random_spec(rng, 2, 3, 4)
        brute = oracle.min_cost_bruteforce(spec, EXT_OPS, max_cost=7, operator_weights=weights)
        res = oracle.synthesize(spec, operators=EXT_OPS, max_cost=7, operator_weights=weights)
        if brute is None:
            assert res.formula is None
            continue
        checked += 1
        assert res.cost == brute[0] == F.weighted_cost(res.formula, weights), (to_text(brute[1], spec.alphabet), weights)
        assert semantics.separates_by_sat(spec, res.formula)
    assert checked >= 10
