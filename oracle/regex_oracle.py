"""CPU oracle of the regex front-end -- TEST INFRASTRUCTURE, not product code.

There is NO reference implementation of regular-expression inference under /root/reference (SPEC.md:11 scopes it
out; the arithmetic lives in the work cited at PAPER.md:45), so this file restates nothing: PARITY UNPINNED.  It is
an independent, deliberately naive statement of the semantics that ``paper_2504_18943_b200/regex.py`` and
``csrc/regex_ops.cuh`` implement -- characteristic sequences as Python integers, operators straight from their
definitions, candidates visited strictly in canonical order, first construction wins -- modelled on how the
reference backs its LTL engine with ``oracle.py:67-109`` (naive semantics + dedup-free brute force).  It is pinned
to ground truth that does not depend on this repository:

  * membership: the CS of every stored expression equals ``re.fullmatch`` of its pattern on every infix
    (``check_store_against_re``);
  * minimality: ``min_cost_bruteforce`` enumerates expression TREES by cost without any dedup and tests them with
    ``re.fullmatch`` on the examples only.

Only tests/ may import this module.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field
from itertools import product

from paper_2504_18943_b200.regex import (
    OP_CONCAT, OP_LITERAL, OP_QUESTION, OP_STAR, OP_UNION, Concat, CostFunction, Eps, InfixIndex, Lit, Question,
    RegexSpecification, Star, Union, to_pattern,
)


def cs_question(ix: InfixIndex, a: int) -> int:
    return a | 1


def cs_union(ix: InfixIndex, a: int, b: int) -> int:
    return a | b


def cs_concat(ix: InfixIndex, a: int, b: int) -> int:
    """bit w = some split w = u v has u in a and v in b"""
    out = 0
    for w in range(ix.n_bits):
        for u, v in ix.splits[ix.offsets[w]:ix.offsets[w + 1]]:
            if (a >> u) & 1 and (b >> v) & 1:
                out |= 1 << w
                break
    return out


def cs_star(ix: InfixIndex, a: int) -> int:
    """least fixpoint of  s = {empty word} | a s  restricted to the infixes (shorter infixes first)"""
    out = 1
    for w in range(1, ix.n_bits):
        for u, v in ix.splits[ix.offsets[w]:ix.offsets[w + 1]]:
            if u != 0 and (a >> u) & 1 and (out >> v) & 1:
                out |= 1 << w
                break
    return out


@dataclass
class OracleLevel:
    base: int
    cs: list = field(default_factory=list)      # characteristic sequences (int)
    op: list = field(default_factory=list)
    left: list = field(default_factory=list)
    right: list = field(default_factory=list)

    @property
    def n(self) -> int:
        return len(self.cs)


class RegexOracle:
    """Level-wise enumeration in the engine's canonical order (csrc/engine.cu: plan_level with the regex tags):
    literals (the empty word, then the letters) at cost `literal`; r? over level c - question; r* over level
    c - star; r s over all (c1, c2) with c1 + c2 = c - concat, left operand outer; r | s over c1 <= c2 with
    c1 + c2 = c - union, pairs i <= j when c1 == c2."""

    def __init__(self, spec: RegexSpecification, cost: CostFunction = CostFunction()):
        self.spec, self.cost, self.ix = spec, cost, InfixIndex(spec)
        self.levels: list[OracleLevel] = []
        self.seen: set[int] = set()
        self.total = 0

    def level(self, c: int) -> OracleLevel:
        return self.levels[c - 1]

    def _candidates(self, c: int):
        ix, k = self.ix, self.cost
        lv = lambda cc: self.levels[cc - 1]
        if c == k.literal:
            for a, bits in enumerate(ix.atom_bits):
                yield bits, OP_LITERAL, a, -1
        if c - k.question >= 1:
            src = lv(c - k.question)
            for i in range(src.n):
                yield cs_question(ix, src.cs[i]), OP_QUESTION, src.base + i, -1
        if c - k.star >= 1:
            src = lv(c - k.star)
            for i in range(src.n):
                yield cs_star(ix, src.cs[i]), OP_STAR, src.base + i, -1
        for c1 in range(1, c - k.concat):
            la, lb = lv(c1), lv(c - k.concat - c1)
            for i, j in product(range(la.n), range(lb.n)):
                yield cs_concat(ix, la.cs[i], lb.cs[j]), OP_CONCAT, la.base + i, lb.base + j
        for c1 in range(1, c - k.union):
            c2 = c - k.union - c1
            if c1 > c2:
                break
            la, lb = lv(c1), lv(c2)
            for i in range(la.n):
                for j in range(i if c1 == c2 else 0, lb.n):
                    yield cs_union(ix, la.cs[i], lb.cs[j]), OP_UNION, la.base + i, lb.base + j

    def expand_level(self, c: int, exhaustive: bool = False):
        """-> (new entries, separator id or None, candidates constructed); a non-exhaustive level ends at its
        first separating candidate (which is new: an older separating CS would have ended the search before)"""
        assert c == len(self.levels) + 1
        level, constructed, sep_gid = OracleLevel(self.total), 0, None
        for cs, op, left, right in self._candidates(c):
            constructed += 1
            fresh = cs not in self.seen
            if fresh:
                self.seen.add(cs)
                level.cs.append(cs)
                level.op.append(op)
                level.left.append(left)
                level.right.append(right)
            if self.ix.separates(cs) and sep_gid is None and fresh:
                sep_gid = level.base + level.n - 1
                if not exhaustive:
                    break
        self.levels.append(level)
        self.total += level.n
        return level.n, sep_gid, constructed

    def entry(self, gid: int):
        for lv in self.levels:
            if lv.base <= gid < lv.base + lv.n:
                k = gid - lv.base
                return lv.op[k], lv.left[k], lv.right[k]
        raise IndexError(gid)

    def regex_of(self, gid: int):
        op, left, right = self.entry(gid)
        if op == OP_LITERAL:
            return self.ix.atoms[left]
        if op == OP_QUESTION:
            return Question(self.regex_of(left))
        if op == OP_STAR:
            return Star(self.regex_of(left))
        return (Concat if op == OP_CONCAT else Union)(self.regex_of(left), self.regex_of(right))


@dataclass
class OracleResult:
    regex: object
    pattern: str | None
    cost: int | None
    constructed: int
    unique: int
    store: RegexOracle


def synthesize(spec: RegexSpecification, cost: CostFunction = CostFunction(), max_cost: int = 12, exhaustive: bool = False) -> OracleResult:
    store, constructed, found = RegexOracle(spec, cost), 0, None
    for c in range(1, max_cost + 1):
        _, sep, delta = store.expand_level(c, exhaustive)
        constructed += delta
        if sep is not None and found is None:
            found = (sep, c)
            if not exhaustive:
                break
    if found is None:
        return OracleResult(None, None, None, constructed, store.total, store)
    regex = store.regex_of(found[0])
    return OracleResult(regex, to_pattern(regex), found[1], constructed, store.total, store)


def check_store_against_re(store: RegexOracle) -> int:
    """Every stored CS equals re.fullmatch of the expression's pattern on every infix; returns how many were checked."""
    checked = 0
    for lv in store.levels:
        for k in range(lv.n):
            pattern = to_pattern(store.regex_of(lv.base + k))
            assert store.ix.cs_of_pattern(pattern) == lv.cs[k], pattern
            checked += 1
    return checked


def enumerate_trees(alphabet, cost: CostFunction, max_cost: int):
    """Every expression tree by ascending cost, no dedup (the pattern of the reference's oracle.py:67-93)."""
    by_cost = [[]]
    for c in range(1, max_cost + 1):
        here = []
        if c == cost.literal:
            here += [Eps()] + [Lit(ch) for ch in alphabet]
        if c - cost.question >= 1:
            here += [Question(g) for g in by_cost[c - cost.question]]
        if c - cost.star >= 1:
            here += [Star(g) for g in by_cost[c - cost.star]]
        for c1 in range(1, c - cost.concat):
            here += [Concat(a, b) for a, b in product(by_cost[c1], by_cost[c - cost.concat - c1])]
        for c1 in range(1, c - cost.union):
            here += [Union(a, b) for a, b in product(by_cost[c1], by_cost[c - cost.union - c1])]
        yield from ((c, g) for g in here)
        by_cost.append(here)


def min_cost_bruteforce(spec: RegexSpecification, cost: CostFunction = CostFunction(), max_cost: int = 6):
    for c, g in enumerate_trees(spec.alphabet, cost, max_cost):
        compiled = re.compile(to_pattern(g))
        if all(compiled.fullmatch(w) for w in spec.positives) and not any(compiled.fullmatch(w) for w in spec.negatives):
            return c, g
    return None
