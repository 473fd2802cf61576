"""Plain finite-trace semantics of LTLf, used only to re-check a witness.

``synthesize`` re-validates the formula it returns against this definition
before handing it to the caller, exactly as the reference does through
``oracle.separates_by_sat`` (reference ``engine.py:502``, ``oracle.py:27-63``).
It shares nothing with the CUDA kernels: ``sat`` is a position-by-position
evaluation with the quantifiers of F and U written out, and the witness check
``separates_by_sat`` evaluates the same definition by its expansion laws
(``F p = p | X F p``, ``p U q = q | (p & X (p U q))``, X false at the last
position) -- ``_truth_table_fast`` in one backward pass per node over lists,
``_truth_mask`` (what ``separates_by_sat`` calls) with one Python integer per
table and the passes run by doubling shifts; the quantifier loops, then the
list passes, were a third of a millisecond of every ``synthesize`` call.
``tests/test_host_model.py`` checks that all three agree on random formulas
and traces.  None is ever part of enumeration.
"""

from __future__ import annotations

from .formulas import And, Atom, Formula, Future, Globally, Next, Not, Or, Until
from .traces import Specification, Trace


def _truth_table(trace: Trace, f: Formula) -> list[bool]:
    """Truth value of ``f`` at every position of ``trace``."""
    n = trace.length
    if isinstance(f, Atom):
        return [f.index in step for step in trace.steps]
    if isinstance(f, Not):
        return [not v for v in _truth_table(trace, f.child)]
    if isinstance(f, Next):
        inner = _truth_table(trace, f.child)
        return [inner[i + 1] if i + 1 < n else False for i in range(n)]
    if isinstance(f, Future):
        inner = _truth_table(trace, f.child)
        return [any(inner[i:]) for i in range(n)]
    if isinstance(f, Globally):  # extension
        inner = _truth_table(trace, f.child)
        return [all(inner[i:]) for i in range(n)]
    if isinstance(f, (And, Or, Until)):
        lhs, rhs = _truth_table(trace, f.left), _truth_table(trace, f.right)
        if isinstance(f, And):
            return [a and b for a, b in zip(lhs, rhs)]
        if isinstance(f, Or):
            return [a or b for a, b in zip(lhs, rhs)]
        return [any(rhs[k] and all(lhs[i:k]) for k in range(i, n)) for i in range(n)]
    raise TypeError(f"not a formula node: {f!r}")


def _truth_table_fast(trace: Trace, f: Formula) -> list[bool]:
    """``_truth_table`` by the expansion laws: one backward pass per temporal node."""
    n = trace.length
    if isinstance(f, Atom):
        return [f.index in step for step in trace.steps]
    if isinstance(f, Not):
        return [not v for v in _truth_table_fast(trace, f.child)]
    if isinstance(f, Next):
        inner = _truth_table_fast(trace, f.child)
        return inner[1:] + [False] if n else []
    if isinstance(f, Future):
        out = _truth_table_fast(trace, f.child)
        for i in range(n - 2, -1, -1):
            out[i] = out[i] or out[i + 1]
        return out
    if isinstance(f, Globally):  # extension: G p = p & X G p, with G p = p at the last position
        out = _truth_table_fast(trace, f.child)
        for i in range(n - 2, -1, -1):
            out[i] = out[i] and out[i + 1]
        return out
    if isinstance(f, (And, Or, Until)):
        lhs, rhs = _truth_table_fast(trace, f.left), _truth_table_fast(trace, f.right)
        if isinstance(f, And):
            return [a and b for a, b in zip(lhs, rhs)]
        if isinstance(f, Or):
            return [a or b for a, b in zip(lhs, rhs)]
        out = rhs
        for i in range(n - 2, -1, -1):
            out[i] = out[i] or (lhs[i] and out[i + 1])
        return out
    raise TypeError(f"not a formula node: {f!r}")


def _truth_mask(trace: Trace, f: Formula, atom_masks: dict) -> int:
    """``_truth_table_fast`` with the table of a sub-formula held in one Python integer (bit i = holds at position
    i): the expansion laws become shifts towards bit 0, run to their fixpoint by doubling the stride.  This is what
    ``separates_by_sat`` evaluates: a 16-node witness on 14 traces is ~200 integer operations instead of ~2000 list
    element operations (0.3 ms of a 6.4 ms ``synthesize`` call)."""
    n = trace.length
    full = (1 << n) - 1
    if isinstance(f, Atom):
        mask = atom_masks.get(f.index)
        if mask is None:
            mask = sum(1 << i for i, step in enumerate(trace.steps) if f.index in step)
            atom_masks[f.index] = mask
        return mask
    if isinstance(f, Not):
        return full ^ _truth_mask(trace, f.child, atom_masks)
    if isinstance(f, Next):
        return _truth_mask(trace, f.child, atom_masks) >> 1  # (false at the last position)
    if isinstance(f, (Future, Globally)):
        x = _truth_mask(trace, f.child, atom_masks)
        if isinstance(f, Globally):  # extension: G p = !F !p
            x ^= full
        s = 1
        while s < n:  # bit i |= bits i+1 .. : suffix OR
            x |= x >> s
            s <<= 1
        return x ^ full if isinstance(f, Globally) else x
    if isinstance(f, (And, Or, Until)):
        lhs, rhs = _truth_mask(trace, f.left, atom_masks), _truth_mask(trace, f.right, atom_masks)
        if isinstance(f, And):
            return lhs & rhs
        if isinstance(f, Or):
            return lhs | rhs
        out, run, s = rhs, lhs, 1  # out[i] = rhs[i] | (lhs[i] & out[i+1]);  run = "lhs holds on i .. i+s-1"
        while s < n:
            out |= run & (out >> s)
            run &= run >> s
            s <<= 1
        return out
    raise TypeError(f"not a formula node: {f!r}")


def sat(trace: Trace, i: int, f: Formula) -> bool:
    """Does ``f`` hold at position ``i`` of ``trace``?"""
    if i < 0 or i >= trace.length:
        raise ValueError(f"position {i} out of range for trace of length {trace.length}")
    return _truth_table(trace, f)[i]


def separates_by_sat(spec: Specification, f: Formula) -> bool:
    """Every positive trace satisfies ``f`` at position 0 and no negative one does (reference oracle.py:55-63)."""
    for trace in spec.positives:
        if not (trace.length and _truth_mask(trace, f, {}) & 1):
            return False
    for trace in spec.negatives:
        if trace.length and _truth_mask(trace, f, {}) & 1:
            return False
    return True
