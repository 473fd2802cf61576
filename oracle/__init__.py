"""CPU oracle for the enumeration hot path -- TEST INFRASTRUCTURE, not product code.

Python face of ``oracle/ltl_oracle.c`` (a scalar C restatement of the
reference's ``engine.py`` + ``kernels.py``; see that file's header for how it is
pinned to the unmodified reference through ``tests/golden``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2504_18943_b200`` never does.

The classes mirror the reference's ``CandidateStore`` / ``expand_level`` /
``synthesize`` (reference ``engine.py:114-167, 367-451, 454-506``) closely
enough that a parity test reads the same against either.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess
import time
from dataclasses import dataclass, field
from itertools import product

import numpy as np

from paper_2504_18943_b200 import formulas as F
from paper_2504_18943_b200 import semantics
from paper_2504_18943_b200.traces import (
    Layout,
    Specification,
    atom_bitvectors,
    smallest_lane_dtype,
    validate_feasible,
)

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libltl_oracle.so"

OP_ATOM, OP_NOT, OP_NEXT, OP_FUTURE, OP_AND, OP_UNTIL, OP_OR = range(7)
OP_GLOBALLY = 7  # extension (see ltl_oracle.c's header): not in the reference
_OP_BIT = {"not": OP_NOT, "next": OP_NEXT, "future": OP_FUTURE, "and": OP_AND, "until": OP_UNTIL, "or": OP_OR,
           "globally": OP_GLOBALLY, "atom": OP_ATOM}
_STATUS_FAILURE = {1: "time budget exhausted", 2: "memory budget exhausted"}


def build(force: bool = False) -> pathlib.Path:
    """Compile the C oracle with gcc (seconds)."""
    src = _HERE / "ltl_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(_HERE), "-s", "-B"], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        i64, p = ctypes.c_int64, ctypes.c_void_p
        L.orc_create.restype = p
        L.orc_create.argtypes = [ctypes.c_int, ctypes.c_int, p, p, p, ctypes.c_int]
        L.orc_destroy.argtypes = [p]
        L.orc_set_weights.restype = ctypes.c_int
        L.orc_set_weights.argtypes = [p, p]
        L.orc_expand_level.restype = ctypes.c_int
        L.orc_expand_level.argtypes = [p, ctypes.c_int, ctypes.c_uint, ctypes.c_int, i64, i64, ctypes.c_double,
                                       ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.orc_now.restype = ctypes.c_double
        L.orc_total.restype = i64
        L.orc_total.argtypes = [p]
        L.orc_approx_bytes.restype = i64
        L.orc_approx_bytes.argtypes = [p]
        L.orc_level_info.argtypes = [p, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.orc_level_copy.argtypes = [p, ctypes.c_int, p, p, p, p]
        _lib = L
    return _lib


def op_mask(operators) -> int:
    return sum(1 << _OP_BIT[name] for name in F.EXTENDED_OPERATOR_NAMES if name in set(operators))


@dataclass
class OracleLevel:
    cms: np.ndarray
    op: np.ndarray
    left: np.ndarray
    right: np.ndarray
    base: int

    @property
    def n(self) -> int:
        return len(self.cms)


class OracleStore:
    """Reference-shaped candidate store backed by the C oracle."""

    def __init__(self, spec: Specification, dtype=None, operator_weights: dict | None = None):
        self.spec = spec
        self.dtype = np.dtype(dtype) if dtype is not None else smallest_lane_dtype(spec.max_length)
        self.layout = Layout.from_specification(spec, self.dtype)
        self.atoms = atom_bitvectors(spec, self.dtype)
        self.trace_count = spec.trace_count
        self.key_words = -(-(self.trace_count * self.dtype.itemsize) // 8)
        masks = np.ascontiguousarray(self.layout.masks.astype(np.uint64))
        target = np.ascontiguousarray(self.layout.target.astype(np.uint64))
        atoms = np.ascontiguousarray(self.atoms.astype(np.uint64))
        self._h = lib().orc_create(self.trace_count, self.dtype.itemsize * 8, masks.ctypes.data,
                                   target.ctypes.data, atoms.ctypes.data, spec.alphabet.n)
        if not self._h:
            raise RuntimeError("orc_create failed")
        if operator_weights:  # extension
            vec = [1] * 8
            for name, value in operator_weights.items():
                vec[_OP_BIT[name]] = int(value)
            if lib().orc_set_weights(self._h, (ctypes.c_int * 8)(*vec)) != 0:
                raise ValueError("bad operator weights")
        self.n_levels = 0
        self._cache: dict[int, OracleLevel] = {}

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.orc_destroy(h)

    @property
    def total(self) -> int:
        return int(lib().orc_total(self._h))

    @property
    def approx_bytes(self) -> int:
        return int(lib().orc_approx_bytes(self._h))

    def expand_level(self, cost, ops=F.DEFAULT_OPERATORS, exhaustive=False, batch_size=1 << 16,
                     memory_budget_mb=8192, deadline=None):
        """Returns (n_new, sep_gid|None, constructed_delta, failure|None)."""
        n_new, sep, cons = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        dl = -1.0 if deadline is None else float(deadline)
        st = lib().orc_expand_level(self._h, cost, op_mask(ops), int(bool(exhaustive)), int(batch_size),
                                    int(memory_budget_mb) * (1 << 20), dl,
                                    ctypes.byref(n_new), ctypes.byref(sep), ctypes.byref(cons))
        if st < 0:
            raise RuntimeError(f"orc_expand_level({cost}) rejected its arguments")
        self.n_levels += 1
        return n_new.value, (None if sep.value < 0 else sep.value), cons.value, _STATUS_FAILURE.get(st)

    def level(self, cost: int) -> OracleLevel:
        if cost not in self._cache:
            n, base = ctypes.c_int64(), ctypes.c_int64()
            if lib().orc_level_info(self._h, cost, ctypes.byref(n), ctypes.byref(base)) != 0:
                raise IndexError(cost)
            cms = np.empty((n.value, self.trace_count), dtype=self.dtype)
            op = np.empty(n.value, dtype=np.uint8)
            left = np.empty(n.value, dtype=np.int64)
            right = np.empty(n.value, dtype=np.int64)
            lib().orc_level_copy(self._h, cost, cms.ctypes.data, op.ctypes.data, left.ctypes.data, right.ctypes.data)
            self._cache[cost] = OracleLevel(cms, op, left, right, base.value)
        return self._cache[cost]

    @property
    def levels(self):
        return [self.level(c) for c in range(1, self.n_levels + 1)]

    def all_cms(self) -> np.ndarray:
        return np.concatenate([lv.cms for lv in self.levels], axis=0)

    def entry(self, gid: int):
        for lv in self.levels:
            if lv.base <= gid < lv.base + lv.n:
                k = gid - lv.base
                return int(lv.op[k]), int(lv.left[k]), int(lv.right[k])
        raise IndexError(gid)


def reconstruct(store, gid: int) -> F.Formula:
    """Witness from provenance (reference engine.py:170-182)."""
    tag, left, right = store.entry(gid)
    if tag == OP_ATOM:
        return F.Atom(left)
    if tag in (OP_NOT, OP_NEXT, OP_FUTURE, OP_GLOBALLY):
        return {OP_NOT: F.Not, OP_NEXT: F.Next, OP_FUTURE: F.Future, OP_GLOBALLY: F.Globally}[tag](reconstruct(store, left))
    node = {OP_AND: F.And, OP_UNTIL: F.Until, OP_OR: F.Or}[tag]
    return node(reconstruct(store, left), reconstruct(store, right))


@dataclass
class OracleResult:
    formula: F.Formula | None
    cost: int | None
    outcome: str
    constructed: int
    unique: int
    max_cost_reached: int
    elapsed_s: float
    failure: str | None = None
    store: OracleStore | None = field(default=None, repr=False)
    per_level: list = field(default_factory=list)


def synthesize(spec: Specification, operators=F.DEFAULT_OPERATORS, max_cost=20, time_budget_s=300.0,
               memory_budget_mb=8192, batch_size=1 << 16, exhaustive=False, operator_weights: dict | None = None) -> OracleResult:
    """Level loop of the reference's ``synthesize`` (engine.py:454-506) over the C oracle."""
    validate_feasible(spec)
    unknown = set(operators) - set(F.EXTENDED_OPERATOR_NAMES)
    if unknown:
        raise ValueError(f"unknown operators: {sorted(unknown)}")
    store = OracleStore(spec, operator_weights=operator_weights)
    t0 = time.perf_counter()
    deadline = lib().orc_now() + time_budget_s
    constructed, reached, found_gid, found_cost, failure = 0, 0, None, None, None
    per_level = []
    for cost in range(1, max_cost + 1):
        reached = cost
        n_new, sep, delta, fail = store.expand_level(cost, operators, exhaustive, batch_size,
                                                     memory_budget_mb, deadline)
        constructed += delta
        per_level.append((n_new, delta, sep))
        if fail:
            failure = fail
            break
        if sep is not None and found_gid is None:
            found_gid, found_cost = sep, cost
            if not exhaustive:
                break
    elapsed = time.perf_counter() - t0
    formula = reconstruct(store, found_gid) if found_gid is not None else None
    if formula is not None and not semantics.separates_by_sat(spec, formula):
        raise RuntimeError("oracle produced a non-separating formula")
    return OracleResult(formula, found_cost, "found" if formula is not None else "exhausted", constructed,
                        store.total, reached, elapsed, None if formula is not None else failure, store, per_level)


# ---- dedup-free brute force (reference oracle.py:67-109), for minimality checks on tiny specs


def enumerate_formulas(n_atoms: int, operators=F.DEFAULT_OPERATORS, max_cost: int = 6, operator_weights: dict | None = None):
    """Every formula tree by ascending cost, no dedup (reference oracle.py:67-93).  ``operator_weights`` / the operator
    ``globally`` are the extension: a node of operator ``name`` costs ``operator_weights.get(name, 1)``."""
    enabled = set(operators)
    w = lambda name: int((operator_weights or {}).get(name, 1))
    by_cost: list[list] = [[]]
    for c in range(1, max_cost + 1):
        here = []
        if c == w("atom"):
            here = [F.Atom(i) for i in range(n_atoms)]
        for name, node in (("not", F.Not), ("next", F.Next), ("future", F.Future), ("globally", F.Globally)):
            if name in enabled and c - w(name) >= 1:
                here += [node(g) for g in by_cost[c - w(name)]]
        for name, node in (("and", F.And), ("until", F.Until), ("or", F.Or)):
            if name in enabled:
                for c1 in range(1, c - w(name)):
                    here += [node(a, b) for a, b in product(by_cost[c1], by_cost[c - w(name) - c1])]
        yield from ((c, g) for g in here)
        by_cost.append(here)


def min_cost_bruteforce(spec: Specification, operators=F.DEFAULT_OPERATORS, max_cost: int = 8, operator_weights: dict | None = None):
    for c, g in enumerate_formulas(spec.alphabet.n, operators, max_cost, operator_weights):
        if semantics.separates_by_sat(spec, g):
            return c, g
    return None
