"""Regex front-end on the CUDA engine (characteristic sequences of up to 4096 bits) against the CPU oracle
(oracle/regex_oracle.py, pinned to Python's `re` by tests/test_regex_oracle.py).  PARITY UNPINNED with respect to the
reference, which has no regex synthesiser."""

import random
import re

import numpy as np
import pytest

from oracle import regex_oracle as ro
from paper_2504_18943_b200 import _native
from paper_2504_18943_b200 import regex as rx
from test_regex_oracle import EMAIL_N, EMAIL_P, random_binary_spec

pytestmark = pytest.mark.gpu


def _assert_level_equal(store, oracle_store, cost, where):
    a, b = store.level(cost), oracle_store.level(cost)
    assert (a.n, a.base) == (b.n, b.base), where
    want = np.frombuffer(b"".join(store.ix.row_bytes(cs) for cs in b.cs), dtype=np.uint8).reshape(b.n, store.ix.n_bytes) \
        if b.n else np.empty((0, store.ix.n_bytes), dtype=np.uint8)
    assert np.array_equal(a.cms, want), where + ": characteristic sequences differ"
    assert list(a.op) == b.op and list(a.left) == b.left and list(a.right) == b.right, where + ": provenance differs"


@pytest.mark.parametrize("seed,cost,max_cost", [
    (0, rx.CostFunction(), 7), (1, rx.CostFunction(), 7), (2, rx.CostFunction(), 6),
    (3, rx.CostFunction(literal=1, question=2, star=2, concat=1, union=3), 8),
    (4, rx.CostFunction(literal=2, star=1, concat=2), 9),
])
def test_levels_equal_the_oracle_on_baseline_config_0(seed, cost, max_cost):
    """BASELINE configs[0]: alphabet {0,1}, 4 positive / 4 negative strings of length <= 5; exhaustive levels."""
    spec = random_binary_spec(random.Random(seed))
    store, ref = rx.RegexStore(spec, cost), ro.RegexOracle(spec, cost)
    try:
        for c in range(1, max_cost + 1):
            status, n_new, sep, constructed = store.expand(c, exhaustive=True)
            o_new, o_sep, o_constructed = ref.expand_level(c, exhaustive=True)
            assert (status, n_new, constructed) == (0, o_new, o_constructed), f"seed {seed} cost {c}"
            _assert_level_equal(store, ref, c, f"seed {seed} cost {c}")
        for lv_cost in (2, max_cost):  # every stored expression means what re says it means
            lv = store.level(lv_cost)
            for k in range(0, lv.n, max(1, lv.n // 50)):
                pattern = rx.to_pattern(store.regex_of(lv.base + k))
                assert store.ix.row_bytes(store.ix.cs_of_pattern(pattern)) == lv.cms[k].tobytes(), pattern
    finally:
        store.close()


@pytest.mark.parametrize("seed", range(8))
def test_synthesize_regex_returns_the_oracles_expression(seed):
    spec = random_binary_spec(random.Random(100 + seed))
    res = rx.synthesize_regex(spec, rx.RegexConfig(max_cost=9))
    want = ro.synthesize(spec, max_cost=9)
    assert (res.pattern, res.cost, res.stats.unique, res.stats.constructed) == (want.pattern, want.cost, want.unique, want.constructed)
    if res.pattern is not None:
        assert all(re.fullmatch(res.pattern, w) for w in spec.positives) and not any(re.fullmatch(res.pattern, w) for w in spec.negatives)


def test_three_letter_alphabet_and_wider_sequences():
    words = ['aacca', 'acacbcab', 'bbccba', 'bcaaaaac', 'bcaabbca', 'bcacbbac', 'cbcbba', 'ccaaca']
    spec = rx.RegexSpecification(tuple(words[:4]), tuple(words[4:]))
    ix = rx.InfixIndex(spec)
    assert ix.n_bits == 111
    store, ref = rx.RegexStore(spec), ro.RegexOracle(spec)
    try:
        for c in range(1, 6):
            _, n_new, _, constructed = store.expand(c, exhaustive=True)
            o_new, _, o_constructed = ref.expand_level(c, exhaustive=True)
            assert (n_new, constructed) == (o_new, o_constructed)
            _assert_level_equal(store, ref, c, f"abc cost {c}")
    finally:
        store.close()


def _wide_words(seed, n_words=8, length=(9, 13), letters="abc"):
    rng = random.Random(seed)
    words = set()
    while len(words) < n_words:
        words.add("".join(rng.choice(letters) for _ in range(rng.randint(*length))))
    return sorted(words)


@pytest.mark.parametrize("seed,cost,max_cost", [
    (0, rx.CostFunction(), 5), (1, rx.CostFunction(literal=1, question=2, star=1, concat=1, union=2), 6),
])
def test_sequences_wider_than_128_bits_equal_the_oracle(seed, cost, max_cost):
    """CSs of three vectors."""
    words = _wide_words(seed)
    spec = rx.RegexSpecification(tuple(words[:4]), tuple(words[4:]))
    store, ref = rx.RegexStore(spec, cost), ro.RegexOracle(spec, cost)
    assert 128 < store.ix.n_bits <= 1024
    try:
        for c in range(1, max_cost + 1):
            status, n_new, sep, constructed = store.expand(c, exhaustive=True)
            o_new, o_sep, o_constructed = ref.expand_level(c, exhaustive=True)
            assert (status, n_new, constructed) == (0, o_new, o_constructed), f"seed {seed} cost {c}"
            _assert_level_equal(store, ref, c, f"wide seed {seed} cost {c}")
    finally:
        store.close()


def _build_levels(store, max_cost):
    for c in range(1, max_cost + 1):
        status, n_new, sep, constructed = store.expand(c, exhaustive=True)
        assert status == 0
    return [store.level(c) for c in range(1, max_cost + 1)]


def test_email_example_on_the_gpu():
    """528 infixes (five uint4 vectors per CS), 4103 guide entries, 20 literals.  Levels 1-6 against the
    oracle; levels 7-8 (10^5..10^6 candidates: the per-operator kernels, the estimate-and-redo path) against `re` on a
    sample, pairwise distinct over the whole store, and identical on a second run."""
    spec = rx.RegexSpecification(EMAIL_P, EMAIL_N)
    store, ref = rx.RegexStore(spec), ro.RegexOracle(spec)
    assert (store.ix.n_bits, len(store.ix.splits)) == (528, 4103)
    try:
        for c in range(1, 7):
            status, n_new, sep, constructed = store.expand(c, exhaustive=True)
            o_new, o_sep, o_constructed = ref.expand_level(c, exhaustive=True)
            assert (status, n_new, constructed) == (0, o_new, o_constructed), f"cost {c}"
            _assert_level_equal(store, ref, c, f"e-mail cost {c}")
        seen = set()
        for c in range(1, 9):
            if c > 6:
                status, n_new, sep, constructed = store.expand(c, exhaustive=True)
                assert status == 0 and sep is None
            lv = store.level(c)
            rows = {lv.cms[k].tobytes() for k in range(lv.n)}
            assert len(rows) == lv.n and not (rows & seen), f"cost {c}: a sequence is stored twice"
            seen |= rows
            for k in range(0, lv.n, max(1, lv.n // 25)):
                pattern = rx.to_pattern(store.regex_of(lv.base + k))
                assert store.ix.row_bytes(store.ix.cs_of_pattern(pattern)) == lv.cms[k].tobytes(), pattern
        assert store.level(8).n > 50_000
        again = rx.RegexStore(spec)
        try:
            for lv, lv2 in zip([store.level(c) for c in (7, 8)], _build_levels(again, 8)[6:]):
                assert np.array_equal(lv.cms, lv2.cms) and np.array_equal(lv.op, lv2.op)
                assert np.array_equal(lv.left, lv2.left) and np.array_equal(lv.right, lv2.right)
        finally:
            again.close()
    finally:
        store.close()


def test_synthesize_regex_on_wide_sequences():
    """Searches that end with a separator cut on sequences of two / three vectors: same expression, cost and counters as
    the oracle."""
    cases = [
        (("abcabcabcabc", "abcabc", "abc"), ("cacbaccbabacab", "bccabbabcbbaca", "cbabcaacbcabbb", "abcab", "bca", "acb"), 9),
        (("abaabaaba", "abab", "ab", "abaab"), ("aabbaaaabbabbaababba", "babbbbbabbaababbabbb", "abaaaaabbbbbabbabaab", "a", "bb", "aab"), 10),
    ]
    for pos, neg, max_cost in cases:
        spec = rx.RegexSpecification(pos, neg)
        assert rx.InfixIndex(spec).n_bits > 128
        res = rx.synthesize_regex(spec, rx.RegexConfig(max_cost=max_cost))
        want = ro.synthesize(spec, max_cost=max_cost)
        assert want.pattern is not None
        assert (res.pattern, res.cost, res.stats.unique, res.stats.constructed) == (want.pattern, want.cost, want.unique, want.constructed)


@pytest.mark.parametrize("name,max_cost,bits", [("re-c2", 10, 207), ("re-c3", 7, 2709)])
def test_baseline_shaped_example_sets_equal_the_oracle(name, max_cost, bits):
    """BASELINE configs[2] / configs[3] as literally worded (binary alphabet 20 + 20 strings of length <= 10; three
    letters, 64 + 64 strings of length <= 16: 22 uint4 per sequence, 24912 guide entries)."""
    from paper_2504_18943_b200.workloads import regex_workload

    spec = regex_workload(name)
    store, ref = rx.RegexStore(spec), ro.RegexOracle(spec)
    assert store.ix.n_bits == bits
    try:
        for c in range(1, max_cost + 1):
            status, n_new, sep, constructed = store.expand(c, exhaustive=True)
            o_new, o_sep, o_constructed = ref.expand_level(c, exhaustive=True)
            assert (status, n_new, constructed) == (0, o_new, o_constructed), f"{name} cost {c}"
            _assert_level_equal(store, ref, c, f"{name} cost {c}")
    finally:
        store.close()


@pytest.mark.parametrize("name,seed,max_cost,world", [("re-c0", 0, 8, 2), ("re-c0", 3, 7, 3), ("re-c2", 0, 11, 2), ("re-email", 0, 6, 3)])
def test_sharded_search_of_regex_stores(name, seed, max_cost, world):
    """One regex search over several ranks (stores on one GPU play them, the exchange done by hand as in
    tests/test_gpu_sharded.py): candidates routed to their hash owners by the bit-sliced tiles in route mode, and every rank ends every level equal to the oracle."""
    from paper_2504_18943_b200 import engine
    from paper_2504_18943_b200.workloads import regex_workload
    from test_gpu_sharded import _exchange_level

    spec = regex_workload(name, seed)
    stores, ref = [rx.RegexStore(spec) for _ in range(world)], ro.RegexOracle(spec)
    cfg = engine.EngineConfig(exhaustive=True, batch_size=1)
    try:
        for c in range(1, max_cost + 1):
            results = _exchange_level(stores, c, cfg, mask=rx._OP_MASK)
            o_new, o_sep, o_constructed = ref.expand_level(c, exhaustive=True)
            for r, (status, n_new, sep, delta) in enumerate(results):
                assert (status, n_new, delta) == (0, o_new, o_constructed), f"{name} cost {c} rank {r}"
                _assert_level_equal(stores[r], ref, c, f"{name} cost {c} rank {r}")
    finally:
        for s in stores:
            s.close()


def test_synthesize_regex_over_a_process_group():
    """The real protocol code (dist.sharded_expand_level over NCCL) with one rank: every level through the exchange,
    small levels built locally, and the default threshold; same expression and counters as the oracle."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2504_18943_b200 import dist as pdist

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    default_threshold = pdist.REPLICATE_BELOW
    try:
        cases = [(rx.RegexSpecification(("abcabcabcabc", "abcabc", "abc"), ("cacbaccbabacab", "bccabbabcbbaca", "cbabcaacbcabbb", "abcab", "bca", "acb")), 9),
                 (random_binary_spec(random.Random(101)), 9)]
        for spec, max_cost in cases:
            want = ro.synthesize(spec, max_cost=max_cost)
            for replicate_below in (0, 500, default_threshold):
                pdist.REPLICATE_BELOW = replicate_below
                res = rx.synthesize_regex(spec, rx.RegexConfig(max_cost=max_cost), group=dist.group.WORLD)
                assert (res.pattern, res.cost, res.stats.unique, res.stats.constructed) == (want.pattern, want.cost, want.unique, want.constructed)
    finally:
        pdist.REPLICATE_BELOW = default_threshold
        dist.destroy_process_group()


def test_regex_command_line(tmp_path, capsys):
    import json

    from paper_2504_18943_b200 import cli

    path = tmp_path / "examples.txt"
    path.write_text("abcabcabcabc\nabcabc\nabc\n<eps>\n---\nabcab\nbca\nacb\nab\n")
    assert cli.main(["regex", "--input", str(path), "--format", "json"]) == 0
    report = json.loads(capsys.readouterr().out)
    want = ro.synthesize(rx.RegexSpecification(("abcabcabcabc", "abcabc", "abc", ""), ("abcab", "bca", "acb", "ab")), max_cost=12)
    assert (report["regex"], report["cost"], report["constructed"], report["unique"], report["outcome"]) == \
        (want.pattern, want.cost, want.constructed, want.unique, "found")
    assert cli.main(["regex", "--input", str(path), "--max-cost", "3"]) == 2     # budget exhausted
    assert "no expression found" in capsys.readouterr().out
    path.write_text("ab\n---\nab\n")
    assert cli.main(["regex", "--input", str(path)]) == 1                         # infeasible
    assert "error:" in capsys.readouterr().err


@pytest.mark.parametrize("seed", [207, 210])
def test_cut_levels_on_top_of_a_store_that_holds_a_solution(seed):
    """Exhaustive levels up to and including the first solution, then non-exhaustive ones: the guarded kernel with the
    regex tiles (the LTL engine's chunk truncation at batch size 1)."""
    spec = random_binary_spec(random.Random(seed))
    first = ro.synthesize(spec, max_cost=10).cost
    assert first == 8
    store, ref = rx.RegexStore(spec), ro.RegexOracle(spec)
    try:
        for c in range(1, first + 3):
            exhaustive = c <= first
            status, n_new, sep, constructed = store.expand(c, exhaustive=exhaustive)
            assert (status, n_new, sep, constructed) == (0,) + tuple(ref.expand_level(c, exhaustive=exhaustive)), f"seed {seed} cost {c}"
            _assert_level_equal(store, ref, c, f"seed {seed} cost {c}")
    finally:
        store.close()


def test_sequences_beyond_4096_bits_are_refused():
    words = _wide_words(7, n_words=12, length=(28, 30), letters="abcdefgh")
    with pytest.raises(_native.NativeEngineError, match="4096 bits"):
        rx.RegexStore(rx.RegexSpecification(tuple(words[:6]), tuple(words[6:])))


def test_email_example_at_scale():
    """The e-mail example to cost 10 (16.1 M candidates, 992 K stored sequences of 528 bits; levels 8-10 take the
    per-operator launches and the estimate-and-redo path): pairwise distinct over the whole store, every sampled entry
    is the operator of its provenance applied to its children (oracle operators on Python integers), the closed-form
    candidate counts, and a second run gives the same arrays."""
    spec = rx.RegexSpecification(EMAIL_P, EMAIL_N)
    store = rx.RegexStore(spec)
    ix = store.ix
    try:
        sizes, constructed = [], []
        for c in range(1, 11):
            status, n_new, sep, built = store.expand(c, exhaustive=True)
            assert status == 0 and sep is None
            sizes.append(n_new)
            constructed.append(built)
        n = lambda c: sizes[c - 1] if c >= 1 else 0
        for c in range(2, 11):  # unit costs: ? and * over level c-1, concatenation over all splits of c-1, union over c1 <= c2
            want = 2 * n(c - 1) + sum(n(a) * n(c - 1 - a) for a in range(1, c - 1))
            want += sum(n(a) * n(c - 1 - a) if a < c - 1 - a else n(a) * (n(a) + 1) // 2 for a in range(1, c - 1) if a <= c - 1 - a)
            assert constructed[c - 1] == want, f"cost {c}"
        assert store.total == sum(sizes) == 992_008 and sum(constructed) == 16_139_866
        rows = store.all_cms()
        keys = {rows[k].tobytes() for k in range(len(rows))}
        assert len(keys) == store.total
        as_int = lambda k: int.from_bytes(rows[k].tobytes(), "little")
        rng = random.Random(5)
        lv10 = store.level(10)
        for k in [rng.randrange(lv10.n) for _ in range(1500)] + list(range(40)) + list(range(lv10.n - 40, lv10.n)):
            tag, left, right = int(lv10.op[k]), int(lv10.left[k]), int(lv10.right[k])
            if tag == rx.OP_QUESTION:
                want = ro.cs_question(ix, as_int(left))
            elif tag == rx.OP_STAR:
                want = ro.cs_star(ix, as_int(left))
            elif tag == rx.OP_CONCAT:
                want = ro.cs_concat(ix, as_int(left), as_int(right))
            else:
                want = ro.cs_union(ix, as_int(left), as_int(right))
            assert as_int(lv10.base + k) == want, (k, tag, left, right)
        again = rx.RegexStore(spec)
        try:
            for c in range(1, 11):
                again.expand(c, exhaustive=True)
            lv = again.level(10)
            assert np.array_equal(lv.cms, lv10.cms) and np.array_equal(lv.op, lv10.op)
            assert np.array_equal(lv.left, lv10.left) and np.array_equal(lv.right, lv10.right)
        finally:
            again.close()
    finally:
        store.close()
