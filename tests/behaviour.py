"""Behaviour checks shared by the CPU oracle and the CUDA engine.

Each check restates, in this repo's own words, something the reference's test-suite pins
(file:line cited per check) and is run twice: against ``oracle/`` in the CPU suite
(tests/test_behaviour_oracle.py) and against the CUDA engine through the C ABI in the GPU
suite (tests/test_behaviour_gpu.py).  A backend is a tiny adaptor with the methods of
``OracleBackend`` below."""

from __future__ import annotations

import random
import types

import numpy as np
import pytest

import oracle
from paper_2504_18943_b200 import (
    And,
    Atom,
    Future,
    InfeasibleSpecificationError,
    Next,
    Not,
    Or,
    Until,
    cost,
    parse_formula,
    semantics,
    spec_from_steps,
    to_text,
    workloads,
)
from paper_2504_18943_b200.formulas import DEFAULT_OPERATORS
from paper_2504_18943_b200.traces import Alphabet, Specification, Trace

UNARY = {1: Not, 2: Next, 3: Future}
BINARY = {4: And, 5: Until, 6: Or}


class OracleBackend:
    name = "oracle"

    def store(self, spec):
        return oracle.OracleStore(spec)

    def expand(self, store, level, ops=DEFAULT_OPERATORS, exhaustive=False, batch=1 << 16, memory_mb=1 << 20):
        n_new, sep, delta, failure = store.expand_level(level, ops, exhaustive, batch, memory_mb)
        assert failure is None
        return n_new, sep, delta

    def close(self, store):
        pass

    def reconstruct(self, store, gid):
        return oracle.reconstruct(store, gid)

    def synth(self, spec, **kw):
        r = oracle.synthesize(spec, **kw)
        return types.SimpleNamespace(outcome=r.outcome, cost=r.cost, formula=r.formula, constructed=r.constructed,
                                     unique=r.unique, failure=r.failure, max_cost_reached=r.max_cost_reached)


def truth_cm(spec, formula, dtype):
    """CM of a formula from the naive position-by-position semantics."""
    return np.array([sum(int(semantics.sat(tr, i, formula)) << i for i in range(tr.length)) for tr in spec.traces],
                    dtype=dtype)


def random_spec(rng, n_atoms, max_side, max_len):
    """reference tests/strategies.py:81-100"""
    def trace():
        return Trace(tuple(frozenset(p for p in range(n_atoms) if rng.random() < 0.5)
                           for _ in range(rng.randint(1, max_len))))
    while True:
        pos = [trace() for _ in range(rng.randint(1, max_side))]
        neg = [trace() for _ in range(rng.randint(1, max_side))]
        if not {t.steps for t in pos} & {t.steps for t in neg}:
            return Specification(Alphabet.default(n_atoms), tuple(pos), tuple(neg))


# ---- checks ---------------------------------------------------------------------------------

def check_bit_fixtures(b):
    """reference tests/test_kernels.py:43-45,70-72,88-90 and test_acceptance.py:63-69:
    atom a over the word abcaa is 10011; !a = 01100, X a = 00110, F a = 11111 (position 0 leftmost)."""
    alphabet = Alphabet.of("abc")
    spec = Specification(alphabet, (Trace(tuple(frozenset({alphabet.index(c)}) for c in "abcaa")),), ())
    store = b.store(spec)
    try:
        ops = ("not", "next", "future")
        b.expand(store, 1, ops, exhaustive=True)
        b.expand(store, 2, ops, exhaustive=True)
        l1, l2 = store.level(1), store.level(2)
        render = lambda word: "".join("1" if (int(word) >> j) & 1 else "0" for j in range(5))
        assert render(l1.cms[0][0]) == "10011"
        got = {(int(o), int(l)): render(row[0]) for row, o, l in zip(l2.cms, l2.op, l2.left)}
        assert got[(1, 0)] == "01100"  # !a
        assert got[(2, 0)] == "00110"  # X a
        assert got[(3, 0)] == "11111"  # F a
    finally:
        b.close(store)


def check_until_fixture(b):
    """reference tests/test_kernels.py:122-129: b U a over <b, a> holds at both positions."""
    spec = spec_from_steps([["b", "a"]], [], "ab")
    store = b.store(spec)
    try:
        for level in (1, 2, 3):
            b.expand(store, level, ("not", "until"), exhaustive=True)
        want = truth_cm(spec, parse_formula("b U a", spec.alphabet), store.dtype)
        assert int(want[0]) == 0b11
        l3 = store.level(3)
        hits = [k for k in range(l3.n) if l3.op[k] == 5 and store.entry(int(l3.left[k]))[0] == 0]
        assert any(np.array_equal(l3.cms[k], want) for k in range(l3.n)) or np.any((store.all_cms() == want).all(axis=1))
    finally:
        b.close(store)


def check_cost_two_known_answer(b):
    """reference tests/test_engine.py:65-78: n1 = 2, sep = 0, n2 = 1, constructed = 2 + 6."""
    spec = spec_from_steps([["a"]], [["b"]], "ab")
    store = b.store(spec)
    try:
        ops = ("not", "next", "future")
        n1, sep, d1 = b.expand(store, 1, ops, exhaustive=True)
        n2, _, d2 = b.expand(store, 2, ops, exhaustive=True)
        assert (n1, sep, n2, d1 + d2) == (2, 0, 1, 8)
    finally:
        b.close(store)


def check_store_invariants(b):
    """reference tests/test_engine.py:81-117: CMs pairwise distinct, children strictly below
    their level, every stored CM equals the naive semantics of its reconstructed formula and
    the formula's node count is the level."""
    spec = workloads.spec1()
    store = b.store(spec)
    try:
        for level in range(1, 6):
            b.expand(store, level, exhaustive=True)
            lv = store.level(level)
            if lv.n:
                assert lv.left[lv.op != 0].max(initial=-1) < lv.base
                assert lv.right.max(initial=-1) < lv.base
        cms = store.all_cms()
        assert len(np.unique(cms, axis=0)) == len(cms) == store.total
        rng = random.Random(7)
        for gid in rng.sample(range(store.total), min(100, store.total)):
            f = b.reconstruct(store, gid)
            level = next(c for c in range(1, 6) if store.level(c).base <= gid < store.level(c).base + store.level(c).n)
            assert cost(f) == level
            lv = store.level(level)
            assert np.array_equal(truth_cm(spec, f, store.dtype), lv.cms[gid - lv.base]), to_text(f, spec.alphabet)
    finally:
        b.close(store)


def check_completeness(b):
    """reference tests/test_engine.py:209-224: the CM set of costs <= 4 equals the CM set of
    every formula tree of cost <= 4 (no dedup, both argument orders)."""
    spec = workloads.spec1()
    store = b.store(spec)
    try:
        for level in range(1, 5):
            b.expand(store, level, exhaustive=True)
        engine_cms = {tuple(int(w) for w in row) for row in store.all_cms()}
        tree_cms = {tuple(int(w) for w in truth_cm(spec, f, np.uint64))
                    for _, f in oracle.enumerate_formulas(spec.alphabet.n, DEFAULT_OPERATORS, 4)}
        assert engine_cms == tree_cms
    finally:
        b.close(store)


def check_synthesize_outcomes(b):
    """reference tests/test_engine.py:26-62,149-206."""
    spec1 = workloads.spec1()
    r = b.synth(spec1)
    assert (r.outcome, r.cost) == ("found", 4) and semantics.separates_by_sat(spec1, r.formula)
    assert to_text(r.formula, spec1.alphabet) == "!(b U a)"
    assert (r.constructed, r.unique) == (65, 33)

    trivial = spec_from_steps([["a"]], [["b"]], "ab")
    r = b.synth(trivial)
    assert (r.cost, r.formula) == (1, Atom(0))

    with pytest.raises(InfeasibleSpecificationError):
        b.synth(spec_from_steps([["a"]], [["a"]], "ab"))

    only_neg = spec_from_steps([], [["a", "b"], ["ab", ""]], "ab")
    r = b.synth(only_neg)
    assert r.cost == 2 and semantics.separates_by_sat(only_neg, r.formula)
    only_pos = spec_from_steps([["", "a"], ["", "b"]], [], "ab")
    r = b.synth(only_pos)
    assert r.cost == 2 and semantics.separates_by_sat(only_pos, r.formula)

    disj = spec_from_steps([["a", ""], ["b", ""]], [["", ""]], "ab")
    r = b.synth(disj, operators=("or",))
    assert (r.outcome, r.cost) == ("found", 3) and semantics.separates_by_sat(disj, r.formula)

    with pytest.raises(ValueError, match="unknown operators"):
        b.synth(trivial, operators=("xor",))

    r = b.synth(spec1, max_cost=3)
    assert (r.outcome, r.formula, r.cost, r.max_cost_reached) == ("exhausted", None, None, 3) and r.unique > 0

    r = b.synth(spec1, time_budget_s=0.0)
    assert r.outcome == "exhausted" and "time budget" in r.failure

    r = b.synth(workloads.spec2(), memory_budget_mb=1)
    assert r.outcome == "exhausted" and "memory budget" in r.failure and r.unique > 0

    r = b.synth(spec1, max_cost=5, exhaustive=True)
    assert (r.outcome, r.cost) == ("found", 4) and semantics.separates_by_sat(spec1, r.formula)

    small, big = b.synth(spec1, batch_size=3), b.synth(spec1, batch_size=1 << 16)
    assert small.formula == big.formula and small.unique == big.unique

    r = b.synth(trivial, exhaustive=True, max_cost=3)
    assert r.constructed >= 2 and r.unique <= r.constructed


def check_minimality_against_bruteforce(b, cases=15):
    """reference tests/test_engine.py:135-146 (seed 2024): the found cost equals the cost of the
    first separating tree in a dedup-free enumeration checked with the naive semantics."""
    rng = random.Random(2024)
    checked = 0
    while checked < cases:
        spec = random_spec(rng, 2, 2, 4)
        brute = oracle.min_cost_bruteforce(spec, max_cost=6)
        if brute is None:
            continue
        r = b.synth(spec, max_cost=6)
        assert r.outcome == "found" and r.cost == brute[0], to_text(brute[1], spec.alphabet)
        checked += 1


ALL_CHECKS = [check_bit_fixtures, check_until_fixture, check_cost_two_known_answer, check_store_invariants,
              check_completeness, check_synthesize_outcomes, check_minimality_against_bruteforce]
