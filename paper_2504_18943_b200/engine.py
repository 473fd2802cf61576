"""Drop-in replacement for the reference's enumeration engine, running on a B200.

Same entry points, argument meaning, results and error behaviour as the
reference's ``pkg/src/ltlsynth/engine.py``:

=====================  ======================================================
here                   reference
=====================  ======================================================
``EngineConfig``       ``engine.py:61-80``
``RunStats``           ``engine.py:83-88``
``SynthesisResult``    ``engine.py:91-98``
``CandidateStore``     ``engine.py:114-167`` (the language cache; here in HBM)
``expand_level``       ``engine.py:367-451``
``synthesize``         ``engine.py:454-506``
``reconstruct``        ``engine.py:170-182``
``normalize_operators````engine.py:52-58``
=====================  ======================================================

The level loop, witness reconstruction and the final semantic re-check stay in
Python as in the reference; everything inside a level (candidate construction,
separation check, observational-equivalence dedup, ordering, append) is one call
into the CUDA library through the C ABI of ``include/ltlsynth_b200.h``.  There is
no CPU path: constructing a ``CandidateStore`` without the built library or
without a B200 raises ``NativeEngineError``.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _native, semantics
from .formulas import (
    DEFAULT_OPERATORS,
    EXTENDED_OPERATOR_NAMES,
    OPERATOR_NAMES,
    WEIGHT_NAMES,
    And,
    Atom,
    Formula,
    Future,
    Globally,
    Next,
    Not,
    Or,
    Until,
)
from .traces import Layout, Specification, atom_bitvectors, smallest_lane_dtype, validate_feasible

OP_ATOM, OP_NOT, OP_NEXT, OP_FUTURE, OP_AND, OP_UNTIL, OP_OR = range(7)
OP_GLOBALLY = 7  # EXTENSION: not a reference tag (engine.py:42 ends at OP_OR); only with EngineConfig.extended_grammar
_TAG_OF = {"not": OP_NOT, "next": OP_NEXT, "future": OP_FUTURE, "and": OP_AND, "until": OP_UNTIL, "or": OP_OR,
           "globally": OP_GLOBALLY, "atom": OP_ATOM}
_UNARY_NODE = {OP_NOT: Not, OP_NEXT: Next, OP_FUTURE: Future, OP_GLOBALLY: Globally}
_BINARY_NODE = {OP_AND: And, OP_UNTIL: Until, OP_OR: Or}

OUTCOME_FOUND = "found"
OUTCOME_EXHAUSTED = "exhausted"
_FAILURE_TEXT = {_native.TIME_BUDGET: "time budget exhausted", _native.MEMORY_BUDGET: "memory budget exhausted"}


def normalize_operators(operators, extended: bool = False) -> tuple[str, ...]:
    """Canonical operator order (reference engine.py:52-58).  ``extended`` also admits ``globally`` (an extension the
    reference rejects like any unknown name)."""
    names = EXTENDED_OPERATOR_NAMES if extended else OPERATOR_NAMES
    wanted = set(operators)
    bad = wanted.difference(names)
    if bad:
        raise ValueError(f"unknown operators: {sorted(bad)}")
    return tuple(name for name in names if name in wanted)


def operator_mask(operators) -> int:
    """Bit k set <=> operator tag k enabled (``op_mask`` of the C ABI)."""
    return sum(1 << _TAG_OF[name] for name in normalize_operators(operators, extended=True))


def weight_vector(weights: dict | None) -> list[int]:
    """Cost of one node per operator tag (index 0 = an atom) for ``ltlb200_set_weights``; all 1 = the reference."""
    vec = [1] * 16
    for name, value in (weights or {}).items():
        if name not in WEIGHT_NAMES:
            raise ValueError(f"unknown operator in operator_weights: {name!r}")
        if int(value) != value or int(value) < 1:
            raise ValueError("operator weights must be integers >= 1")
        vec[_TAG_OF[name]] = int(value)
    return vec


@dataclass(frozen=True)
class EngineConfig:
    operators: tuple[str, ...] = DEFAULT_OPERATORS
    max_cost: int = 20
    time_budget_s: float = 300.0
    memory_budget_mb: int = 8192  # the reference's host-side estimate, see CandidateStore.approx_bytes
    batch_size: int = 1 << 16  # only shapes the `constructed` counter on the level that ends the run
    threads: int | None = None  # accepted for compatibility; the device schedules its own parallelism
    exhaustive: bool = False
    dnc_threshold: int = 8
    device: int = 0  # extension: CUDA device ordinal
    hbm_budget_mb: int = 0  # extension: cap on device memory (0 = 90% of free HBM)
    # EXTENSIONS beyond the reference grammar and cost, off by default so that every reference
    # call behaves as the reference does: `extended_grammar` admits the operator "globally" (G; SPEC.md:211 lists it as a
    # non-goal), `operator_weights` gives one node of an operator a cost other than 1 ("config-extensible",
    # unimplemented in the reference): {"atom" | "not" | "next" | "future" | "globally" | "and" | "until" | "or": int >= 1}
    extended_grammar: bool = False
    operator_weights: tuple | None = None  # ((name, weight), ...): hashable form of the dict

    def __post_init__(self):
        if self.max_cost < 1:
            raise ValueError("max_cost must be >= 1")
        if self.time_budget_s < 0 or self.memory_budget_mb <= 0:
            raise ValueError("budgets must be positive")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.threads is not None and self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.operator_weights is not None:
            if isinstance(self.operator_weights, dict):
                object.__setattr__(self, "operator_weights", tuple(sorted(self.operator_weights.items())))
            if not self.extended_grammar:
                raise ValueError("operator_weights is an extension: set extended_grammar=True")
            weight_vector(dict(self.operator_weights))
        if "globally" in self.operators and not self.extended_grammar:
            raise ValueError("unknown operators: ['globally']")

    @property
    def weights(self) -> dict:
        return dict(self.operator_weights or ())


@dataclass
class RunStats:
    constructed: int = 0
    unique: int = 0
    elapsed_s: float = 0.0
    max_cost_reached: int = 0


@dataclass
class SynthesisResult:
    formula: Formula | None
    cost: int | None
    minimal: bool
    outcome: str
    stats: RunStats
    failure: str | None = None
    # beyond the reference's fields: counters of the device handle that ran the search (ltlb200_stats: bytes copied
    # host<->device, kernel launches, device time of the construction kernels, ...)
    device_stats: dict | None = None


class _Level:
    """One cost level of the cache; arrays are fetched from HBM on first use."""

    def __init__(self, store: "CandidateStore", cost: int, n: int, base: int):
        self._store, self._cost, self.n, self.base = store, cost, n, base
        self._arrays = None

    def _fetch(self):
        if self._arrays is None:
            self._arrays = self._store._copy_level(self._cost, self.n)
        return self._arrays

    cms = property(lambda self: self._fetch()[0])
    op = property(lambda self: self._fetch()[1])
    left = property(lambda self: self._fetch()[2])
    right = property(lambda self: self._fetch()[3])


class _DeviceMemory:
    """``__cuda_array_interface__`` face of a device buffer the engine owns (for ``torch.as_tensor``)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (int(ptr), False), "version": 2}


class CandidateStore:
    """Cost-indexed cache of unique CMs with provenance, resident on the GPU."""

    def __init__(self, spec: Specification, dtype=None, device: int = 0, hbm_budget_mb: int = 0, stream=None,
                 operator_weights: dict | None = None):
        self.spec = spec
        self.dtype = np.dtype(dtype) if dtype is not None else smallest_lane_dtype(spec.max_length)
        self.layout = Layout.from_specification(spec, self.dtype)
        self.atoms = atom_bitvectors(spec, self.dtype)
        self.trace_count = spec.trace_count
        self.key_words = -(-(self.trace_count * self.dtype.itemsize) // 8)
        self.levels: list[_Level] = []
        self._device = int(device)
        self._stream = int(stream or 0)
        lib = _native.load()
        if lib.ltlb200_device_count() < 1:
            raise _native.NativeEngineError("no usable B200: " + _native.last_error())
        as_u64 = lambda a: np.ascontiguousarray(a, dtype=np.uint64)
        masks, target, atoms = as_u64(self.layout.masks), as_u64(self.layout.target), as_u64(self.atoms)
        self._handle = lib.ltlb200_create(
            self.trace_count, self.dtype.itemsize * 8, masks.ctypes.data, target.ctypes.data, atoms.ctypes.data,
            spec.alphabet.n, int(device), int(hbm_budget_mb) << 20, ctypes.c_void_p(stream or 0),
        )
        if not self._handle:
            raise _native.NativeEngineError("ltlb200_create failed: " + _native.last_error())
        if operator_weights:  # extension: per-operator node costs
            vec = (ctypes.c_int32 * 16)(*weight_vector(operator_weights))
            _native.check(lib.ltlb200_set_weights(self._handle, vec), "set_weights")

    def close(self):
        handle, self._handle = getattr(self, "_handle", None), None
        if handle:
            _native.load().ltlb200_destroy(handle)

    __del__ = close

    def reset(self):
        """Empty the store but keep its device buffers (a fresh store on the same specification)."""
        _native.check(_native.load().ltlb200_reset(self._handle), "reset")
        self.levels = []

    # -- reference-shaped accessors -------------------------------------------------
    @property
    def total(self) -> int:
        return sum(level.n for level in self.levels)

    @property
    def approx_bytes(self) -> int:
        return int(_native.load().ltlb200_approx_bytes(self._handle))

    def level(self, cost: int) -> _Level:
        return self.levels[cost - 1]

    def entry(self, gid: int) -> tuple[int, int, int]:
        op, left, right = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        _native.check(
            _native.load().ltlb200_entry(self._handle, int(gid), ctypes.byref(op), ctypes.byref(left), ctypes.byref(right)),
            f"entry({gid})",
        )
        return op.value, left.value, right.value

    def all_cms(self) -> np.ndarray:
        parts = [level.cms for level in self.levels]
        if not parts:
            return np.empty((0, self.trace_count), dtype=self.dtype)
        return np.concatenate(parts, axis=0)

    # -- the reference's key helpers (engine.py:130, 151-167).  The dedup set itself lives on the device; these are
    # host-side views for callers that inspect a store the way the reference's tests could.
    def pack_rows(self, rows: np.ndarray) -> np.ndarray:
        """CM rows as (n, key_words) uint64 keys: the row's bytes, zero-padded to a multiple of eight."""
        rows = np.ascontiguousarray(rows, dtype=self.dtype)
        n, row_bytes = len(rows), self.trace_count * self.dtype.itemsize
        padded = np.zeros((n, self.key_words * 8), dtype=np.uint8)
        padded[:, :row_bytes] = rows.reshape(n, -1).view(np.uint8)
        return padded.view(np.uint64)

    def keys_of(self, packed: np.ndarray) -> list:
        """Hashable keys of packed rows: ints for one-word keys, bytes otherwise (as the reference's)."""
        packed = np.ascontiguousarray(packed, dtype=np.uint64)
        if self.key_words == 1:
            return [int(k) for k in packed[:, 0]]
        stride, raw = self.key_words * 8, packed.tobytes()
        return [raw[k:k + stride] for k in range(0, len(raw), stride)]

    @property
    def seen(self) -> set:
        """Keys of every stored CM, rebuilt from the levels on each access (the live set is the device hash set)."""
        return set(self.keys_of(self.pack_rows(self.all_cms()))) if self.levels else set()

    def device_stats(self) -> dict:
        st = _native.Stats()
        _native.check(_native.load().ltlb200_get_stats(self._handle, ctypes.byref(st)), "get_stats")
        return st.as_dict()

    # -- plumbing ---------------------------------------------------------------------
    def _expand(self, cost, op_mask, exhaustive, batch_size, memory_budget_bytes, deadline):
        n_new, sep, delta = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        status = _native.check(
            _native.load().ltlb200_expand_level(
                self._handle, cost, op_mask, int(exhaustive), int(batch_size), int(memory_budget_bytes),
                -1.0 if deadline is None else float(deadline),
                ctypes.byref(n_new), ctypes.byref(sep), ctypes.byref(delta)),
            f"expand_level({cost})",
        )
        base = self.total
        self.levels.append(_Level(self, cost, n_new.value, base))
        return status, n_new.value, (None if sep.value < 0 else sep.value), delta.value

    # -- shard-engine interface used by dist.sharded_expand_level (one search over several GPUs) ----
    def level_candidates(self, cost: int, op_mask: int) -> int:
        """Candidates level ``cost`` constructs when built in full (same number on every rank)."""
        n = ctypes.c_int64()
        _native.check(_native.load().ltlb200_level_candidates(self._handle, cost, op_mask, ctypes.byref(n)),
                      f"level_candidates({cost})")
        return int(n.value)

    def holds_separator(self) -> bool:
        """Some stored CM separates the examples (then a non-exhaustive level follows the reference's chunk
        truncation, which only the single-handle ``expand_level`` reproduces)."""
        return bool(_native.load().ltlb200_holds_separator(self._handle))

    def expand_local(self, cost, op_mask, exhaustive, batch_size, memory_budget_bytes, deadline):
        """The whole level on this device (``_expand``): what a sharded search does for its small levels."""
        native_deadline = None if deadline is None else _monotonic() + (deadline - time.perf_counter())
        return self._expand(cost, op_mask, exhaustive, batch_size, memory_budget_bytes, native_deadline)

    @property
    def key_bytes(self) -> int:
        return int(_native.load().ltlb200_key_bytes(self._handle))

    @property
    def torch_device(self):
        import torch

        return torch.device("cuda", self._device)

    # routed level of a sharded search (dist.sharded_expand_level; protocol in include/ltlsynth_b200.h)
    def _tensor(self, ptr: int, shape, dtype):
        """torch view of device memory the engine owns (zero copy; valid until the engine reuses the buffer)."""
        import torch

        count = 1
        for d in shape:
            count *= d
        if count == 0 or not ptr:
            return torch.empty(shape, dtype=dtype, device=self.torch_device)
        typestr = {torch.uint8: "|u1", torch.int64: "<i8", torch.int32: "<i4"}[dtype]
        return torch.as_tensor(_DeviceMemory(ptr, tuple(shape), typestr), device=self.torch_device)

    def _wait_for_torch(self):
        """The collectives ran on torch's current stream; unless that is the engine's stream, wait for them."""
        import torch

        stream = torch.cuda.current_stream(self.torch_device)
        if stream.cuda_stream != (self._stream or -1):
            stream.synchronize()

    def route_begin(self, cost, op_mask, exhaustive, deadline, rank, world):
        """Build this rank's share of level ``cost`` and route its candidates to their hash owners;
        ``deadline`` is on ``time.perf_counter()``.  -> (status, parts, sep_ord, n_seps)."""
        import torch

        counts, offsets = (ctypes.c_uint64 * world)(), (ctypes.c_uint64 * world)()
        rows_ptr, ords_ptr = ctypes.c_void_p(), ctypes.c_void_p()
        sep_ord, n_seps = ctypes.c_uint64(), ctypes.c_uint64()
        native_deadline = -1.0 if deadline is None else _monotonic() + (deadline - time.perf_counter())
        status = _native.check(
            _native.load().ltlb200_route_begin(self._handle, cost, op_mask, int(exhaustive), native_deadline, rank, world,
                                               counts, offsets, ctypes.byref(rows_ptr), ctypes.byref(ords_ptr),
                                               ctypes.byref(sep_ord), ctypes.byref(n_seps)),
            f"route_begin({cost})",
        )
        self._pending_seps = n_seps.value
        kb = self.key_bytes
        parts = []
        for o in range(world):
            n, off = int(counts[o]), int(offsets[o])
            parts.append((self._tensor((rows_ptr.value or 0) + off * kb, (n, kb), torch.uint8),
                          self._tensor((ords_ptr.value or 0) + off * 8, (n,), torch.int64)))
        if status != _native.OK:  # the level was closed (empty) by the engine
            self.levels.append(_Level(self, cost, 0, self.total))
        return status, parts, sep_ord.value, n_seps.value

    def exchange_recv(self, n_records: int):
        import torch

        rows_ptr, ords_ptr = ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(_native.load().ltlb200_exchange_recv(self._handle, int(n_records), ctypes.byref(rows_ptr),
                                                           ctypes.byref(ords_ptr)), "exchange_recv")
        return (self._tensor(rows_ptr.value, (n_records, self.key_bytes), torch.uint8),
                self._tensor(ords_ptr.value, (n_records,), torch.int64))

    def owner_reduce(self, n_records: int):
        import torch

        self._wait_for_torch()
        n_claimed, words, bitmap_ptr = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_void_p()
        status = _native.check(
            _native.load().ltlb200_owner_reduce(self._handle, int(n_records), ctypes.byref(n_claimed),
                                                ctypes.byref(bitmap_ptr), ctypes.byref(words)), "owner_reduce")
        if status != _native.OK:
            self.levels.append(_Level(self, len(self.levels) + 1, 0, self.total))
            return status, None
        return status, self._tensor(bitmap_ptr.value, (int(words.value),), torch.int32)

    def winners_export(self, sep_ord: int):
        import torch

        n, rows_ptr, ords_ptr = ctypes.c_uint64(), ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(_native.load().ltlb200_winners_export(self._handle, int(sep_ord), ctypes.byref(n),
                                                            ctypes.byref(rows_ptr), ctypes.byref(ords_ptr)), "winners_export")
        return (self._tensor(rows_ptr.value, (int(n.value), self.key_bytes), torch.uint8),
                self._tensor(ords_ptr.value, (int(n.value),), torch.int64))

    def level_abort(self) -> None:
        had = _native.load().ltlb200_num_levels(self._handle)
        _native.check(_native.load().ltlb200_level_abort(self._handle), "level_abort")
        if _native.load().ltlb200_num_levels(self._handle) > had:
            self.levels.append(_Level(self, len(self.levels) + 1, 0, self.total))

    def separating_ordinals(self):
        import torch

        n = int(getattr(self, "_pending_seps", 0))
        host = np.empty(max(n, 1), dtype=np.uint64)
        got = _native.load().ltlb200_seps_copy(self._handle, host.ctypes.data, n)
        _native.check(int(got), "seps_copy")
        return torch.from_numpy(host[: int(got)].astype(np.int64)).to(self.torch_device)

    def level_commit(self, sep_ord, seps, recv_counts, batch_size, memory_budget_bytes):
        """``recv_counts``: how many winners each other owner sent, in the order they sit in the receive buffers."""
        self._wait_for_torch()
        counts = (ctypes.c_uint64 * max(1, len(recv_counts)))(*recv_counts)
        n_new, sep, delta = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        seps_ptr, n_seps = None, 0
        if seps is not None:
            host = np.ascontiguousarray(seps.detach().cpu().numpy().astype(np.uint64))
            seps_ptr, n_seps = host.ctypes.data, len(host)
        status = _native.check(
            _native.load().ltlb200_level_commit(self._handle, int(sep_ord), seps_ptr, n_seps, counts, len(recv_counts),
                                                int(batch_size), int(memory_budget_bytes), ctypes.byref(n_new),
                                                ctypes.byref(sep), ctypes.byref(delta)),
            "level_commit",
        )
        self.levels.append(_Level(self, len(self.levels) + 1, n_new.value, self.total))
        return status, n_new.value, (None if sep.value < 0 else sep.value), delta.value

    def level_device(self, cost: int):
        """Zero-copy torch views of level ``cost`` on the device: rows uint8 [n, key_bytes] (the numpy row image, zero
        padded to 16-byte vectors) and the winning ordinals int64 [n].  Valid until the next level is built."""
        import torch

        rows_ptr, ords_ptr = ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(_native.load().ltlb200_level_device(self._handle, cost, ctypes.byref(rows_ptr), ctypes.byref(ords_ptr)),
                      f"level_device({cost})")
        n = self.level(cost).n
        return (self._tensor(rows_ptr.value, (n, self.key_bytes), torch.uint8), self._tensor(ords_ptr.value, (n,), torch.int64))

    def _copy_provenance(self, cost: int, n: int):
        """(op, left, right) of a level without its CMs (full-size tests read the rows on the device)."""
        op, left, right = np.empty(n, dtype=np.uint8), np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int64)
        if n:
            _native.check(_native.load().ltlb200_level_copy(self._handle, cost, 0, n, None, op.ctypes.data, left.ctypes.data,
                                                            right.ctypes.data), f"level_copy({cost})")
        return op, left, right

    def _copy_level(self, cost: int, n: int):
        cms = np.empty((n, self.trace_count), dtype=self.dtype)
        op = np.empty(n, dtype=np.uint8)
        left = np.empty(n, dtype=np.int64)
        right = np.empty(n, dtype=np.int64)
        if n:
            _native.check(
                _native.load().ltlb200_level_copy(self._handle, cost, 0, n, cms.ctypes.data, op.ctypes.data,
                                                  left.ctypes.data, right.ctypes.data),
                f"level_copy({cost})",
            )
        return cms, op, left, right


def reconstruct(store, gid: int) -> Formula:
    """Witness formula from (operator, child ids) provenance."""
    tag, left, right = store.entry(gid)
    if tag == OP_ATOM:
        return Atom(left)
    if tag in _UNARY_NODE:
        return _UNARY_NODE[tag](reconstruct(store, left))
    return _BINARY_NODE[tag](reconstruct(store, left), reconstruct(store, right))


class _BudgetExceeded(Exception):
    pass


def _monotonic() -> float:
    return float(_native.load().ltlb200_now())


def expand_level(store: CandidateStore, cost: int, ops=DEFAULT_OPERATORS, config: EngineConfig | None = None,
                 stats: RunStats | None = None, deadline: float | None = None, executor=None):
    """Build level ``cost``; returns ``(new entries, separator id or None)``.

    ``deadline`` is on the clock of ``time.perf_counter()`` as in the reference;
    ``executor`` is accepted and ignored (the device needs no worker threads).
    """
    config = config or EngineConfig()
    stats = stats if stats is not None else RunStats()
    mask = operator_mask(ops)
    native_deadline = None
    if deadline is not None:
        native_deadline = _monotonic() + (deadline - time.perf_counter())
    status, n_new, sep_gid, delta = store._expand(
        cost, mask, config.exhaustive, config.batch_size, config.memory_budget_mb << 20, native_deadline
    )
    stats.constructed += delta
    stats.unique = store.total
    if status in _FAILURE_TEXT:
        raise _BudgetExceeded(_FAILURE_TEXT[status])
    return n_new, sep_gid


def synthesize(spec: Specification, config: EngineConfig = EngineConfig()) -> SynthesisResult:
    """Minimum-cost separating formula by level-wise enumeration on the GPU."""
    validate_feasible(spec)
    ops = normalize_operators(config.operators, config.extended_grammar)
    t0 = time.perf_counter()
    store = CandidateStore(spec, device=config.device, hbm_budget_mb=config.hbm_budget_mb, operator_weights=config.weights)
    try:
        stats = RunStats()
        deadline = t0 + config.time_budget_s
        found, failure = None, None
        for cost in range(1, config.max_cost + 1):
            stats.max_cost_reached = cost
            try:
                _, sep_gid = expand_level(store, cost, ops, config=config, stats=stats, deadline=deadline)
            except _BudgetExceeded as stop:
                failure = str(stop)
                break
            if sep_gid is not None and found is None:
                found = (sep_gid, cost)
                if not config.exhaustive:
                    break
        stats.elapsed_s = time.perf_counter() - t0
        if found is None:
            return SynthesisResult(None, None, False, OUTCOME_EXHAUSTED, stats, failure, store.device_stats())
        formula = reconstruct(store, found[0])
        device_stats = store.device_stats()
    finally:
        store.close()
    if not semantics.separates_by_sat(spec, formula):
        raise RuntimeError("internal error: synthesized formula fails the reference semantics")
    return SynthesisResult(formula, found[1], True, OUTCOME_FOUND, stats, None, device_stats)
