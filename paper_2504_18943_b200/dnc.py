"""Divide-and-conquer over GPU leaves (reference ``pkg/src/ltlsynth/dnc.py``).

Behaviour of the reference, reproduced exactly: positives and negatives are halved in canonical
order (first ceil(n/2) against the rest, ``dnc.py:37-50``), every non-empty (P_i, N_j) pair is
solved recursively until a problem has at most ``max(dnc_threshold, 2)`` traces
(``dnc.py:88-98``), and the answers recombine as ``(f11 & f12) | (f21 & f22)`` in that order
(``dnc.py:100-120``).  The result separates but is not minimal once a split happened; a failing
leaf fails the run and is named in ``failure`` (``dnc.py:97``); counters are summed over the
leaves the reference would have solved (``dnc.py:93-95``).

What is different is the execution.  The split tree is a pure function of the specification,
so it is unfolded FIRST into the ordered list of leaves, and the leaves -- independent searches
(reference SPEC.md:371 notes they "may run concurrently"; ``dnc.py:110-118`` runs them one
after the other) -- are solved concurrently, one engine handle and CUDA stream per worker
thread, round-robin over the given devices.  Recombination then walks the tree in the
reference's order, so formula, cost, counters and failure label are what the sequential walk
produces; leaves past the first failing one are discarded exactly as if they had never run.
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, replace
from functools import reduce

from . import semantics
from .engine import OUTCOME_EXHAUSTED, OUTCOME_FOUND, EngineConfig, RunStats, SynthesisResult, synthesize
from .formulas import And, Or, cost as formula_cost
from .traces import Specification, Trace, validate_feasible


@dataclass(frozen=True)
class SplitPlan:
    """Reference ``dnc.py:30-35``."""

    p_split: tuple[tuple[Trace, ...], tuple[Trace, ...]]
    n_split: tuple[tuple[Trace, ...], tuple[Trace, ...]]
    threshold: int
    budget_per_leaf: EngineConfig


def _halves(traces):
    middle = -(-len(traces) // 2)  # ceil(n / 2): the first half is never the smaller one
    return tuple(traces[:middle]), tuple(traces[middle:])


def split(spec: Specification, threshold: int = 8, budget_per_leaf: EngineConfig | None = None) -> SplitPlan:
    """Halves of the positives and of the negatives in canonical order (reference ``dnc.py:43-50``)."""
    return SplitPlan(_halves(spec.positives), _halves(spec.negatives), threshold, budget_per_leaf or EngineConfig())


@dataclass
class _Node:
    """One problem of the split tree: a leaf (solved directly) or a 2x2 grid of children."""

    label: str
    spec: Specification
    rows: list | None = None  # per non-empty P_i: the children over the non-empty N_j
    leaf_index: int = -1


def _unfold(spec: Specification, config: EngineConfig, label: str, leaves: list) -> _Node:
    node = _Node(label, spec)
    if spec.trace_count <= max(config.dnc_threshold, 2):  # (a 1+1 split would reproduce its own leaf)
        node.leaf_index = len(leaves)
        leaves.append(node)
        return node
    plan = split(spec, config.dnc_threshold, config)
    p_sides = [(i, p) for i, p in enumerate(plan.p_split, start=1) if p] or [(1, ())]
    n_sides = [(j, n) for j, n in enumerate(plan.n_split, start=1) if n] or [(0, ())]
    node.rows = [[_unfold(Specification(spec.alphabet, p, n), config, f"{label}.P{i}N{j}", leaves) for j, n in n_sides]
                 for i, p in p_sides]
    return node


def synthesize_dnc(spec: Specification, config: EngineConfig = EngineConfig(), devices=None,
                   workers: int | None = None) -> SynthesisResult:
    """Split, solve the leaves on the GPU(s), recombine; sound, not minimal above the threshold.

    ``devices``: CUDA ordinals the leaves are spread over (default: ``config.device`` only);
    ``workers``: concurrent leaf searches (default: 4 per device).  Neither changes the result.
    """
    validate_feasible(spec)
    t0 = time.perf_counter()
    deadline = t0 + config.time_budget_s
    devices = list(devices) if devices else [config.device]
    leaves: list[_Node] = []
    root = _unfold(spec, config, "root", leaves)

    def solve(k: int) -> SynthesisResult:
        remaining = max(0.0, deadline - time.perf_counter())
        return synthesize(leaves[k].spec, replace(config, time_budget_s=remaining, device=devices[k % len(devices)]))

    n_workers = max(1, min(len(leaves), workers or 4 * len(devices)))
    if n_workers == 1:
        results = [solve(k) for k in range(len(leaves))]
    else:
        with ThreadPoolExecutor(n_workers) as pool:
            results = list(pool.map(solve, range(len(leaves))))

    stats = RunStats()

    def combine(node: _Node):
        """(formula, minimal, failure) of one problem, visiting leaves in the reference's order."""
        if node.rows is None:
            sub = results[node.leaf_index]
            stats.constructed += sub.stats.constructed
            stats.unique += sub.stats.unique
            stats.max_cost_reached = max(stats.max_cost_reached, sub.stats.max_cost_reached)
            if sub.outcome != OUTCOME_FOUND:
                return None, False, f"leaf {node.label}: {sub.failure or 'budget exhausted'}"
            return sub.formula, sub.minimal, None
        disjuncts = []
        for row in node.rows:
            conjuncts = []
            for child in row:
                formula, _, failure = combine(child)
                if formula is None:
                    return None, False, failure
                conjuncts.append(formula)
            disjuncts.append(reduce(And, conjuncts))
        return reduce(Or, disjuncts), False, None

    formula, minimal, failure = combine(root)
    stats.elapsed_s = time.perf_counter() - t0
    if formula is None:
        return SynthesisResult(None, None, False, OUTCOME_EXHAUSTED, stats, failure)
    if not semantics.separates_by_sat(spec, formula):
        raise RuntimeError("internal error: recombined formula fails the reference semantics")
    return SynthesisResult(formula, formula_cost(formula), minimal, OUTCOME_FOUND, stats)
