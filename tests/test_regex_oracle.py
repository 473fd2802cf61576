"""Regex front-end, first slice: host model and CPU oracle.  PARITY UNPINNED -- the reference has
no regex synthesiser -- so the oracle is pinned to Python's `re` instead: membership of every stored
characteristic sequence, and minimality against a dedup-free brute force over expression trees."""

import random
import re

import pytest

from oracle import regex_oracle as ro
from paper_2504_18943_b200 import regex as rx
from paper_2504_18943_b200.traces import InfeasibleSpecificationError

EMAIL_P = ("geon@ex.io", "test@gmail.com", "mail@test.org", "mail@testing.com")
EMAIL_N = ("hello@", "@test", "email@gmail", "t@test@gmail.com", "mail with@space.com")


def random_binary_spec(rng, n_pos=4, n_neg=4, max_len=5):
    """BASELINE configs[0]: alphabet {0,1}, 4 positive / 4 negative strings of length <= 5."""
    while True:
        draw = lambda: "".join(rng.choice("01") for _ in range(rng.randint(0, max_len)))
        pos, neg = {draw() for _ in range(n_pos)}, {draw() for _ in range(n_neg)}
        if len(pos) == n_pos and len(neg) == n_neg and not pos & neg:
            return rx.RegexSpecification(tuple(sorted(pos)), tuple(sorted(neg)))


def test_infix_closure_and_guide_table():
    ix = rx.InfixIndex(rx.RegexSpecification(("ab", "b"), ("a",)))
    assert ix.infixes == ["", "a", "b", "ab"] and ix.n_bits == 4
    assert ix.splits[ix.offsets[3]:ix.offsets[4]] == [(0, 3), (1, 2), (3, 0)]  # ab = ()ab | a b | ab()
    assert ix.positive_bits == 0b1100 and ix.example_bits == 0b1110
    assert ix.separates(ix.cs_of_pattern("a?b")) and not ix.separates(ix.cs_of_pattern("a|b"))
    with pytest.raises(InfeasibleSpecificationError):
        rx.RegexSpecification(("x",), ("x",))


def test_patterns_costs_and_printing():
    r = rx.Concat(rx.Star(rx.Union(rx.Lit("a"), rx.Lit("."))), rx.Question(rx.Concat(rx.Lit("b"), rx.Eps())))
    assert rx.to_pattern(r) == r"(a|\.)*(b())?"
    assert rx.regex_cost(r) == 9 and rx.regex_cost(r, rx.CostFunction(literal=2, star=5, union=3)) == 2 * 4 + 5 + 3 + 1 + 2
    assert re.fullmatch(rx.to_pattern(r), "a.a.b") and not re.fullmatch(rx.to_pattern(r), "ba")


def test_operators_agree_with_re_on_every_stored_expression():
    rng = random.Random(5)
    total = 0
    for _ in range(6):
        store = ro.RegexOracle(random_binary_spec(rng))
        for c in range(1, 6):
            store.expand_level(c, exhaustive=True)
        total += ro.check_store_against_re(store)
    assert total > 300


def test_email_example_characteristic_sequences():
    """The paper's running example: 528 infixes, so host model / oracle only in this slice."""
    spec = rx.RegexSpecification(EMAIL_P, EMAIL_N)
    ix = rx.InfixIndex(spec)
    assert (ix.n_bits, len(ix.splits), len(spec.alphabet)) == (528, 4103, 19)
    intended = r"[^@ \s]+@[^@ \s]+\.[^@ \s]+"          # the expression the paper expects
    overfit = "|".join(re.escape(w) for w in EMAIL_P)   # ... and the one it does not want
    assert ix.separates(ix.cs_of_pattern(intended)) and ix.separates(ix.cs_of_pattern(overfit))
    # the guide-table operators reproduce re's concatenation / star on this space
    word = ix.cs_of_pattern(r"[^@ \s]+")
    at, dot = 1 << ix.index["@"], 1 << ix.index["."]
    built = ro.cs_concat(ix, ro.cs_concat(ix, ro.cs_concat(ix, ro.cs_concat(ix, word, at), word), dot), word)
    assert built == ix.cs_of_pattern(intended)
    assert ro.cs_star(ix, ix.cs_of_pattern("m|a|i|l")) == ix.cs_of_pattern("(m|a|i|l)*")
    # a bounded search: no expression of cost <= 3 separates, and every level is correct against re
    store = ro.RegexOracle(spec)
    for c in range(1, 4):
        _, sep, _ = store.expand_level(c)
        assert sep is None
    assert ro.check_store_against_re(store) == store.total == 262


@pytest.mark.parametrize("cost", [rx.CostFunction(), rx.CostFunction(literal=1, question=2, star=2, concat=1, union=3),
                                  rx.CostFunction(literal=2, star=1, concat=2)])
def test_minimality_against_bruteforce(cost):
    rng = random.Random(11)
    solved = 0
    for _ in range(12):
        spec = random_binary_spec(rng, 2, 2, 3)
        brute = ro.min_cost_bruteforce(spec, cost, max_cost=7)
        res = ro.synthesize(spec, cost, max_cost=7)
        if brute is None:
            assert res.regex is None
            continue
        solved += 1
        assert res.cost == brute[0] == rx.regex_cost(res.regex, cost), (rx.to_pattern(brute[1]), res.pattern)
        assert all(re.fullmatch(res.pattern, w) for w in spec.positives) and not any(re.fullmatch(res.pattern, w) for w in spec.negatives)
    assert solved >= 4


def test_example_file_of_the_regex_command():
    from paper_2504_18943_b200 import cli

    assert cli.parse_examples("ab\n<eps>\n\n---\nb\r\na b\n") == (("ab", ""), ("b", "a b"))
    for bad in ("ab\n", "a\n---\nb\n---\nc\n"):
        with pytest.raises(ValueError):
            cli.parse_examples(bad)
    args = cli.make_parser().parse_args(["regex", "--input", "x.txt", "--cost", "1,2,2,1,3"])
    assert (args.command, args.cost, args.max_cost, args.format) == ("regex", "1,2,2,1,3", 12, "text")
