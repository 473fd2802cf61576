"""Regular-expression inference on the same engine -- first slice (BASELINE configs 1-4 as worded).

NOT part of the reference: ``SPEC.md:11`` scopes regular-expression synthesis out and ``PAPER.md:81-113`` only
motivates it (the e-mail example), so nothing here restates reference code and PARITY IS UNPINNED.  The semantics
are pinned instead to Python's ``re.fullmatch`` through the CPU oracle ``oracle/regex_oracle.py``.

The idea is the paper's "enumerate semantics, not syntax" applied to regular expressions:

* the examples' **infix closure** -- every substring of every example string, sorted by (length, text), the empty
  word first -- is the observation space; the **characteristic sequence** (CS) of a regular expression has one bit
  per infix: "this infix is in the language".  Two expressions with equal CSs are indistinguishable on the examples
  and on everything the constructions below look at, so only the first (cheapest, then first in canonical order) is
  kept: the engine's observational-equivalence dedup, unchanged;
* on CSs, union is OR, ``r?`` is OR with the empty-word bit, and concatenation and star go through the
  **guide table**: for every infix ``w`` the pairs (index of ``u``, index of ``v``) of its splits ``w = u v``;
* an expression is a solution when its CS agrees with the positives on the bits of the example strings;
* cost levels, canonical order inside a level, first-construction-wins and the separator cut are the engine's
  (``csrc/engine.cu: plan_level`` with the regex operator tags); the **cost function has five parameters** --
  literal, ``?``, ``*``, concatenation, union -- which are the engine's per-operator weights.

CSs of up to 4096 bits (BASELINE configs[0]-sized example sets have a few dozen infixes, the e-mail example 528)
run through the multi-vector kernels (``csrc/wide2.cuh`` with the tiles of ``csrc/wide2_regex.cuh``: row log, 8-byte
slot words, concatenation and star on bit-sliced rows, 32 candidates per word operation); wider example sets are
handled by the host model and the CPU oracle only and raise ``NativeEngineError`` on the GPU path.
"""

from __future__ import annotations

import ctypes
import re
import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .engine import OUTCOME_EXHAUSTED, OUTCOME_FOUND, CandidateStore, RunStats, _BudgetExceeded, _FAILURE_TEXT, _Level, _monotonic
from .traces import InfeasibleSpecificationError

OP_LITERAL, OP_UNION, OP_QUESTION, OP_STAR, OP_CONCAT = 0, 6, 8, 9, 10  # operator tags of include/ltlsynth_b200.h
_OP_MASK = (1 << OP_UNION) | (1 << OP_QUESTION) | (1 << OP_STAR) | (1 << OP_CONCAT)
MAX_GPU_BITS = 4096  # csrc/engine.cu: Engine::set_regex
MIN_ROW_BYTES = 17


# ---- expressions ------------------------------------------------------------------------------------------------

class Regex:
    __slots__ = ()


@dataclass(frozen=True)
class Eps(Regex):
    pass


@dataclass(frozen=True)
class Lit(Regex):
    char: str


@dataclass(frozen=True)
class Question(Regex):
    child: Regex


@dataclass(frozen=True)
class Star(Regex):
    child: Regex


@dataclass(frozen=True)
class Concat(Regex):
    left: Regex
    right: Regex


@dataclass(frozen=True)
class Union(Regex):
    left: Regex
    right: Regex


@dataclass(frozen=True)
class CostFunction:
    """The five parameters of the cost of an expression: one literal (or the empty word), ``?``, ``*``, one
    concatenation, one union.  The default is the unit cost of BASELINE configs[0]."""

    literal: int = 1
    question: int = 1
    star: int = 1
    concat: int = 1
    union: int = 1

    def __post_init__(self):
        if min(self.literal, self.question, self.star, self.concat, self.union) < 1:
            raise ValueError("cost parameters must be >= 1")

    def weight_vector(self) -> list[int]:
        vec = [1] * 16
        vec[OP_LITERAL], vec[OP_QUESTION], vec[OP_STAR], vec[OP_CONCAT], vec[OP_UNION] = (
            self.literal, self.question, self.star, self.concat, self.union)
        return vec


def regex_cost(r: Regex, cost: CostFunction = CostFunction()) -> int:
    if isinstance(r, (Eps, Lit)):
        return cost.literal
    if isinstance(r, Question):
        return cost.question + regex_cost(r.child, cost)
    if isinstance(r, Star):
        return cost.star + regex_cost(r.child, cost)
    if isinstance(r, Concat):
        return cost.concat + regex_cost(r.left, cost) + regex_cost(r.right, cost)
    if isinstance(r, Union):
        return cost.union + regex_cost(r.left, cost) + regex_cost(r.right, cost)
    raise TypeError(f"not a regex node: {r!r}")


def to_pattern(r: Regex) -> str:
    """Python ``re`` syntax (binding: postfix > concatenation > union; only the parentheses that needs)."""
    def show(g: Regex, need: int) -> str:  # need: 0 union context, 1 concatenation operand, 2 postfix operand
        if isinstance(g, Eps):
            return "()"
        if isinstance(g, Lit):
            return re.escape(g.char)
        if isinstance(g, (Question, Star)):
            inner = show(g.child, 2)
            if isinstance(g.child, (Question, Star)):  # `a??` / `a*?` would be re's lazy quantifiers, `a**` an error
                inner = "(" + inner + ")"
            return inner + ("?" if isinstance(g, Question) else "*")
        if isinstance(g, Concat):
            body = show(g.left, 1) + show(g.right, 1)
            return body if need <= 1 else "(" + body + ")"
        if isinstance(g, Union):
            body = show(g.left, 0) + "|" + show(g.right, 0)
            return body if need == 0 else "(" + body + ")"
        raise TypeError(f"not a regex node: {g!r}")

    return show(r, 0)


# ---- examples, infix closure, guide table -------------------------------------------------------------------------

@dataclass(frozen=True)
class RegexSpecification:
    positives: tuple[str, ...]
    negatives: tuple[str, ...]

    def __post_init__(self):
        object.__setattr__(self, "positives", tuple(self.positives))
        object.__setattr__(self, "negatives", tuple(self.negatives))
        both = set(self.positives) & set(self.negatives)
        if both:
            raise InfeasibleSpecificationError(f"string {sorted(both)[0]!r} is both a positive and a negative example")

    @property
    def alphabet(self) -> tuple[str, ...]:
        return tuple(sorted(set("".join(self.positives + self.negatives))))


def infix_closure(strings) -> list[str]:
    """Every substring of every string, the empty word included, sorted by (length, text)."""
    out = {""}
    for w in strings:
        for i in range(len(w)):
            for j in range(i + 1, len(w) + 1):
                out.add(w[i:j])
    return sorted(out, key=lambda x: (len(x), x))


class InfixIndex:
    """Observation space of a specification: the infixes, the guide table and the bitsets the engine needs."""

    def __init__(self, spec: RegexSpecification):
        self.spec = spec
        self.infixes = infix_closure(spec.positives + spec.negatives)
        self.index = {w: k for k, w in enumerate(self.infixes)}
        self.n_bits = len(self.infixes)
        # (rows wider than one uint4 select the engine's multi-vector kernels, where the regex operators live)
        self.n_bytes = max(MIN_ROW_BYTES, -(-self.n_bits // 8))
        # guide table: splits of infix w are entries offsets[w] .. offsets[w+1]-1, each (u, v) with w = u v
        self.offsets, self.splits = [0], []
        for w in self.infixes:
            for cut in range(len(w) + 1):
                self.splits.append((self.index[w[:cut]], self.index[w[cut:]]))
            self.offsets.append(len(self.splits))
        self.positive_bits = self.bitset(spec.positives)
        self.example_bits = self.bitset(spec.positives + spec.negatives)
        # atoms in canonical order: the empty word, then the letters
        self.atoms = [Eps()] + [Lit(c) for c in spec.alphabet]
        self.atom_bits = [1] + [1 << self.index[c] for c in spec.alphabet]

    def bitset(self, words) -> int:
        return sum(1 << self.index[w] for w in set(words))

    def separates(self, cs: int) -> bool:
        return (cs & self.example_bits) == self.positive_bits

    def cs_of_pattern(self, pattern: str) -> int:
        """CS of a Python regular expression by ``re.fullmatch`` on every infix (the membership ground truth)."""
        compiled = re.compile(pattern)
        return sum(1 << k for k, w in enumerate(self.infixes) if compiled.fullmatch(w) is not None)

    def row_bytes(self, cs: int) -> bytes:
        return cs.to_bytes(self.n_bytes, "little")


# ---- the GPU store ------------------------------------------------------------------------------------------------

class RegexStore(CandidateStore):
    """Language cache of regular expressions on the GPU: the LTL store's handle with the regex grammar set."""

    def __init__(self, spec: RegexSpecification, cost: CostFunction = CostFunction(), device: int = 0, hbm_budget_mb: int = 0, stream=None):
        self.spec = spec
        self.ix = InfixIndex(spec)
        self.cost_function = cost
        self.dtype = np.dtype(np.uint8)
        self.trace_count = self.ix.n_bytes
        self.key_words = -(-self.ix.n_bytes // 8)
        self.levels: list[_Level] = []
        self._device, self._stream = int(device), int(stream or 0)
        lib = _native.load()
        if lib.ltlb200_device_count() < 1:
            raise _native.NativeEngineError("no usable B200: " + _native.last_error())
        if self.ix.n_bits > MAX_GPU_BITS:
            raise _native.NativeEngineError(
                f"regex front-end: the GPU path takes characteristic sequences of up to {MAX_GPU_BITS} bits; these examples "
                f"have {self.ix.n_bits} infixes (the host model and oracle/regex_oracle.py handle any width)")
        lanes = lambda cs: np.frombuffer(self.ix.row_bytes(cs), dtype=np.uint8).astype(np.uint64)
        masks, target = lanes(self.ix.example_bits), lanes(self.ix.positive_bits)
        atoms = np.ascontiguousarray(np.stack([lanes(b) for b in self.ix.atom_bits]))
        self._handle = lib.ltlb200_create(self.ix.n_bytes, 8, masks.ctypes.data, target.ctypes.data, atoms.ctypes.data,
                                          len(self.ix.atom_bits), int(device), int(hbm_budget_mb) << 20, ctypes.c_void_p(stream or 0))
        if not self._handle:
            raise _native.NativeEngineError("ltlb200_create failed: " + _native.last_error())
        offsets = np.asarray(self.ix.offsets, dtype=np.uint32)
        entries = np.asarray([u | (v << 16) for u, v in self.ix.splits], dtype=np.uint32)
        _native.check(lib.ltlb200_set_regex(self._handle, self.ix.n_bits, offsets.ctypes.data, entries.ctypes.data, len(entries)), "set_regex")
        _native.check(lib.ltlb200_set_weights(self._handle, (ctypes.c_int32 * 16)(*cost.weight_vector())), "set_weights")

    def expand(self, cost: int, exhaustive: bool = False, deadline=None, memory_budget_bytes: int = 0):
        """Build cost level ``cost``: (status, new entries, separator id or None, candidates constructed).  In a cut
        level ``constructed`` counts the candidates up to and including the separator (batch size 1)."""
        return self._expand(cost, _OP_MASK, exhaustive, 1, memory_budget_bytes, deadline)

    def regex_of(self, gid: int) -> Regex:
        tag, left, right = self.entry(gid)
        if tag == OP_LITERAL:
            return self.ix.atoms[left]
        if tag == OP_QUESTION:
            return Question(self.regex_of(left))
        if tag == OP_STAR:
            return Star(self.regex_of(left))
        node = Concat if tag == OP_CONCAT else Union
        return node(self.regex_of(left), self.regex_of(right))


@dataclass(frozen=True)
class RegexConfig:
    cost: CostFunction = CostFunction()
    max_cost: int = 12
    time_budget_s: float = 300.0
    exhaustive: bool = False
    device: int = 0
    hbm_budget_mb: int = 0


@dataclass
class RegexResult:
    regex: Regex | None
    pattern: str | None
    cost: int | None
    outcome: str
    stats: RunStats
    failure: str | None = None


def synthesize_regex(spec: RegexSpecification, config: RegexConfig = RegexConfig(), group=None) -> RegexResult:
    """Minimum-cost regular expression that accepts every positive and rejects every negative example, by level-wise
    enumeration of characteristic sequences on the GPU.  The result is re-checked with ``re.fullmatch``.

    ``group``: a ``torch.distributed`` process group (one rank per GPU, every rank calls this with the same
    arguments and ``config.device`` = its own GPU): the search is sharded over the ranks with the LTL engine's protocol
    (``dist.sharded_expand_level``: candidates routed to their hash owners, winners published to every rank) and every
    rank returns the same result as a single-GPU run."""
    t0 = time.perf_counter()
    store = RegexStore(spec, config.cost, device=config.device, hbm_budget_mb=config.hbm_budget_mb)
    try:
        stats, found, failure = RunStats(), None, None
        deadline = _monotonic() + config.time_budget_s
        for cost in range(1, config.max_cost + 1):
            stats.max_cost_reached = cost
            if group is not None:
                from . import dist as _dist
                from .engine import EngineConfig

                try:
                    _, sep_gid = _dist.sharded_expand_level(
                        store, cost, _OP_MASK, EngineConfig(exhaustive=config.exhaustive, batch_size=1, memory_budget_mb=1 << 30),
                        stats, deadline, group)
                except _BudgetExceeded as stop:
                    failure = str(stop)
                    break
                status = 0
            else:
                status, _, sep_gid, delta = store.expand(cost, config.exhaustive, deadline)
                stats.constructed += delta
                stats.unique = store.total
            if status in _FAILURE_TEXT:
                failure = _FAILURE_TEXT[status]
                break
            if sep_gid is not None and found is None:
                found = (sep_gid, cost)
                if not config.exhaustive:
                    break
        stats.elapsed_s = time.perf_counter() - t0
        if found is None:
            return RegexResult(None, None, None, OUTCOME_EXHAUSTED, stats, failure)
        regex = store.regex_of(found[0])
    finally:
        store.close()
    pattern = to_pattern(regex)
    compiled = re.compile(pattern)
    if not all(compiled.fullmatch(w) for w in spec.positives) or any(compiled.fullmatch(w) for w in spec.negatives):
        raise RuntimeError("internal error: synthesized expression fails re.fullmatch on the examples")
    return RegexResult(regex, pattern, found[1], OUTCOME_FOUND, stats)


__all__ = ["Regex", "Eps", "Lit", "Question", "Star", "Concat", "Union", "CostFunction", "regex_cost", "to_pattern",
           "RegexSpecification", "InfixIndex", "infix_closure", "RegexStore", "RegexConfig", "RegexResult", "synthesize_regex",
           "_BudgetExceeded"]
