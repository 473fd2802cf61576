"""LTLf formula trees, node-count cost and text syntax.

Same public names and text syntax as the reference's
``pkg/src/ltlsynth/formulas.py`` (node classes :20-52, OPERATOR_NAMES :59,
DEFAULT_OPERATORS :62, cost :65, to_text :80, parse_formula :136) so that the
witness returned by the CUDA engine prints exactly like the reference's.
Binding strength, tightest first: ``! X F``  >  ``U`` (right-assoc)  >  ``&``
>  ``|``.  The printer writes only the parentheses the parser needs.
"""

from __future__ import annotations

import re
from dataclasses import dataclass

from .traces import Alphabet


class Formula:
    __slots__ = ()


@dataclass(frozen=True)
class Atom(Formula):
    index: int


@dataclass(frozen=True)
class Not(Formula):
    child: Formula


@dataclass(frozen=True)
class Next(Formula):
    child: Formula


@dataclass(frozen=True)
class Future(Formula):
    child: Formula


@dataclass(frozen=True)
class Globally(Formula):
    """EXTENSION (not in the reference grammar): G child = child at every position to the end."""

    child: Formula


@dataclass(frozen=True)
class And(Formula):
    left: Formula
    right: Formula


@dataclass(frozen=True)
class Or(Formula):
    left: Formula
    right: Formula


@dataclass(frozen=True)
class Until(Formula):
    left: Formula
    right: Formula


OPERATOR_NAMES = ("not", "next", "future", "and", "until", "or")
DEFAULT_OPERATORS = ("not", "next", "future", "and", "until")
# EXTENSION: operators beyond the reference grammar, accepted only by an EngineConfig with
# extended_grammar=True, and the names a cost-weight table may use ("atom" = one atomic proposition)
EXTENDED_OPERATOR_NAMES = ("not", "next", "future", "globally", "and", "until", "or")
WEIGHT_NAMES = ("atom",) + EXTENDED_OPERATOR_NAMES

_UNARY_PREFIX = {Not: "!", Next: "X ", Future: "F ", Globally: "G "}
# binary node -> (symbol, own level, level required of left child, of right child)
_BINARY_SHAPE = {
    Until: (" U ", 3, 4, 3),  # right-associative
    And: (" & ", 2, 2, 3),  # left-associative
    Or: (" | ", 1, 1, 2),
}
_LEVEL_UNARY = 4


def cost(f: Formula) -> int:
    """Number of nodes."""
    total, todo = 0, [f]
    while todo:
        g = todo.pop()
        total += 1
        if isinstance(g, Atom):
            continue
        if type(g) in _UNARY_PREFIX:
            todo.append(g.child)
        elif type(g) in _BINARY_SHAPE:
            todo.extend((g.left, g.right))
        else:
            raise TypeError(f"not a formula node: {g!r}")
    return total


_WEIGHT_KEY = {Atom: "atom", Not: "not", Next: "next", Future: "future", Globally: "globally", And: "and", Until: "until", Or: "or"}


def weighted_cost(f: Formula, weights: dict | None = None) -> int:
    """EXTENSION: sum of the node weights (``weights[name]``, default 1 each); ``cost`` when no weights are given."""
    weights = weights or {}
    total, todo = 0, [f]
    while todo:
        g = todo.pop()
        total += int(weights.get(_WEIGHT_KEY[type(g)], 1))
        if type(g) in _UNARY_PREFIX:
            todo.append(g.child)
        elif type(g) in _BINARY_SHAPE:
            todo.extend((g.left, g.right))
    return total


def to_text(f: Formula, alphabet: Alphabet) -> str:
    def show(g: Formula, need: int) -> str:
        if isinstance(g, Atom):
            return alphabet.names[g.index]
        kind = type(g)
        if kind in _UNARY_PREFIX:
            return _UNARY_PREFIX[kind] + show(g.child, _LEVEL_UNARY)
        if kind in _BINARY_SHAPE:
            symbol, own, need_left, need_right = _BINARY_SHAPE[kind]
            body = show(g.left, need_left) + symbol + show(g.right, need_right)
            return body if own >= need else "(" + body + ")"
        raise TypeError(f"not a formula node: {g!r}")

    return show(f, 0)


class FormulaSyntaxError(ValueError):
    def __init__(self, message: str, position: int):
        self.position = position
        super().__init__(f"{message} at offset {position}")


_LEX = re.compile(r"\s*(?:(?P<sym>[!&|()])|(?P<word>[A-Za-z_][A-Za-z0-9_]*))")
_KEYWORDS = {"X": Next, "F": Future, "G": Globally}  # (G: extension; an alphabet with an atom named G keeps the reference reading)


def _lex(text: str):
    out, at = [], 0
    while at < len(text):
        m = _LEX.match(text, at)
        if not m:
            rest = text[at:].lstrip()
            if not rest:
                break
            raise FormulaSyntaxError(f"unexpected character {rest[0]!r}", len(text) - len(rest))
        if m.group("sym"):
            out.append((m.group("sym"), m.start("sym")))
        else:
            out.append((m.group("word"), m.start("word")))
        at = m.end()
    out.append((None, len(text)))
    return out


def parse_formula(text: str, alphabet: Alphabet) -> Formula:
    toks = _lex(text)
    pos = 0

    def unary() -> Formula:
        nonlocal pos
        tok, where = toks[pos]
        if tok == "!":
            pos += 1
            return Not(unary())
        if tok in _KEYWORDS and not (tok == "G" and "G" in alphabet.names):
            pos += 1
            return _KEYWORDS[tok](unary())
        if tok == "(":
            pos += 1
            inner = disjunction()
            tok2, where2 = toks[pos]
            if tok2 != ")":
                raise FormulaSyntaxError("expected ')'", where2)
            pos += 1
            return inner
        if tok is None:
            raise FormulaSyntaxError("expected formula, found end of input", where)
        if tok in "&|)" or tok == "U":
            raise FormulaSyntaxError(f"expected formula, found {tok!r}", where)
        pos += 1
        try:
            return Atom(alphabet.index(tok))
        except Exception:
            raise FormulaSyntaxError(f"unknown atom {tok!r}", where) from None

    def until() -> Formula:
        nonlocal pos
        head = unary()
        if toks[pos][0] == "U":
            pos += 1
            return Until(head, until())
        return head

    def conjunction() -> Formula:
        nonlocal pos
        node = until()
        while toks[pos][0] == "&":
            pos += 1
            node = And(node, until())
        return node

    def disjunction() -> Formula:
        nonlocal pos
        node = conjunction()
        while toks[pos][0] == "|":
            pos += 1
            node = Or(node, conjunction())
        return node

    tree = disjunction()
    tok, where = toks[pos]
    if tok is not None:
        raise FormulaSyntaxError(f"unexpected {tok!r}", where)
    return tree
