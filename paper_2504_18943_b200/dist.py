"""One search sharded over several GPUs: the per-level exchange protocol.

The language cache (rows and winning ordinals of every finished level) is replicated on every rank, because any
rank reads any operand.  The dedup set is **owner-sharded**: rank ``r`` holds exactly the CMs whose hash owner is
``r``, of every level, so the set of an N-GPU search has N times the capacity of one GPU's and every rank probes
1/N of a level's candidates.  One level:

1. **route**    every rank builds its tile-strided share of the level's pair space; every candidate that is not a
                duplicate by construction goes, as a record ``{CM row, ordinal}``, to the send region of its
                hash owner (on the device, inside the construction kernel); one grouped send/recv of exact sizes
                moves the regions (``all_to_all``);
2. **reduce**   the owner folds what it received into its part of the set (insert-or-min on the device): it now
                knows, for the CMs it owns, whether they are new and the smallest ordinal that built them; it marks
                its winners in a bitmap with one bit per candidate ordinal of the level;
3. **rank**     ``all_reduce(SUM)`` of the bitmaps -- the owners' bits are disjoint, so the sum is the union --
                gives every rank the level's winners bitmap: the id of a winner is the number of set bits before
                its ordinal; the separator is the ``min`` of the ranks' smallest separating ordinals;
4. **publish**  every owner sends its winners up to the separator to every other rank (``all_gather`` of exact
                sizes); every rank appends its own and the received rows to its cache at their ids.

Per rank and level: C/N candidates built, (K+8)·C/N bytes out and in over NVLink, C/N random probes into a set of
1/N of the keys, and the u·C new rows that every replica of the cache stores anyway (sequential appends, no set
insert).  Metadata travels in two small ``all_gather``s; the host reads three counts per level.

The protocol is written against a small shard-engine interface so that the same code runs over NCCL with the CUDA
engine (``CandidateStore``) and, in the CPU test suite, over gloo with a numpy stand-in.  Collectives move torch
tensors that alias the engine's own buffers.
"""

from __future__ import annotations

import os
import time
from typing import Protocol

import torch
import torch.distributed as dist

from . import semantics
from .engine import (
    OUTCOME_EXHAUSTED,
    OUTCOME_FOUND,
    EngineConfig,
    RunStats,
    SynthesisResult,
    _BudgetExceeded,
    _FAILURE_TEXT,
    normalize_operators,
    operator_mask,
    reconstruct,
)
from .traces import validate_feasible

NO_SEPARATOR = (1 << 64) - 1
_I64_MAX = (1 << 63) - 1

# Levels with fewer candidates than this are built REDUNDANTLY on every rank instead of being sharded: the
# cache is replicated and the engine is deterministic, so every rank gets the same level without a single
# data-path collective, and a level of a few thousand candidates costs less than one exchange.  The count is
# a closed form of the stored level sizes (`level_candidates`), hence identical on every rank.
REPLICATE_BELOW = int(os.environ.get("LTLB200_REPLICATE_BELOW", str(1 << 22)))


class ShardEngine(Protocol):
    """What the exchange needs from a store (CandidateStore implements it on the GPU)."""

    key_bytes: int

    def route_begin(self, cost: int, op_mask: int, exhaustive: bool, deadline, rank: int, world: int):
        """-> (status, parts, sep_ord or NO_SEPARATOR, n_seps); parts[o] = (rows uint8 [n_o, key_bytes],
        ords int64 [n_o]): the records this rank built whose hash owner is o"""

    def exchange_recv(self, n_records: int) -> tuple[torch.Tensor, torch.Tensor]:
        """-> (rows uint8 [n, key_bytes], ords int64 [n]) to receive into"""

    def owner_reduce(self, n_records: int) -> tuple[int, torch.Tensor]:
        """folds the first n_records received records into the owned part of the set
        -> (status, bitmap int32 [words]: this owner's winners, one bit per ordinal of the level)"""

    def level_abort(self) -> None:
        """ends the pending level empty (some rank ran out of budget)"""

    def winners_export(self, sep_ord: int) -> tuple[torch.Tensor, torch.Tensor]:
        """-> (rows, ords) of this owner's winners with ordinal <= sep_ord"""

    def separating_ordinals(self) -> torch.Tensor:
        """int64 tensor of every separating ordinal this rank recorded in the pending level"""

    def level_commit(self, sep_ord: int, seps, recv_counts: list[int], batch_size: int, memory_budget_bytes: int):
        """-> (status, n_new, sep_gid or None, constructed_delta); the global bitmap is in owner_reduce's tensor,
        the receive buffers hold the winners of the other owners, recv_counts[k] records from the k-th source"""

    # optional: without these two every level goes through the exchange
    def level_candidates(self, cost: int, op_mask: int) -> int: ...

    def expand_local(self, cost: int, op_mask: int, exhaustive: bool, batch_size: int, memory_budget_bytes: int, deadline):
        """-> (status, n_new, sep_gid or None, constructed_delta): the whole level on this rank"""


def _gather_ints(values: list[int], device, group) -> list[list[int]]:
    """all_gather of a short int64 vector: result[r] = the vector of rank r."""
    world = dist.get_world_size(group)
    mine = torch.tensor(values, dtype=torch.int64, device=device)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return [[int(v) for v in p.tolist()] for p in parts]


def _exchange(send_parts, recv_bufs, recv_counts, group, include_self: bool):
    """One grouped exchange of exact sizes.  send_parts[peer] = tuple of tensors (same leading size) that goes to
    `peer`; what `src` sends lands in the tensors of recv_bufs at the offset of src (source-major, dense).  With
    include_self the rank's own part is copied in place; otherwise recv_counts[rank] must be 0."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    offsets = [0]
    for c in recv_counts:
        offsets.append(offsets[-1] + c)
    if include_self and recv_counts[rank]:
        for buf, part in zip(recv_bufs, send_parts[rank]):
            buf[offsets[rank]:offsets[rank + 1]].copy_(part)
    ops = []
    peer_of = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    for shift in range(1, world):  # every rank posts its sends and receives in the same relative order
        dst, src = (rank + shift) % world, (rank - shift) % world
        if send_parts[dst][0].shape[0]:
            ops += [dist.P2POp(dist.isend, part, peer_of(dst), group) for part in send_parts[dst]]
        if recv_counts[src]:
            ops += [dist.P2POp(dist.irecv, buf[offsets[src]:offsets[src + 1]], peer_of(src), group) for buf in recv_bufs]
    if ops:
        for work in dist.batch_isend_irecv(ops):  # NCCL: one ncclGroup of sends and receives
            work.wait()


def sharded_expand_level(store: ShardEngine, cost: int, ops, config: EngineConfig, stats: RunStats | None = None,
                         deadline: float | None = None, group=None):
    """``expand_level`` for a search whose pair space is sharded over the ranks of ``group``.

    Returns ``(new entries, separator id or None)`` -- identical on every rank and identical to
    the single-GPU ``expand_level``."""
    stats = stats if stats is not None else RunStats()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mask = ops if isinstance(ops, int) else operator_mask(ops)  # (an operator mask as it is: the regex front-end's tags)
    device = _device_of(store)
    # A NON-exhaustive level over a store that already holds a separating CM is built by every rank on its own,
    # whatever its size: the reference then truncates every chunk at its first separating candidate
    # (engine.py:334-335), which the single-handle expand_level reproduces and "minimum ordinal per CM" cannot.
    truncating = (not config.exhaustive) and getattr(store, "holds_separator", lambda: False)()
    if hasattr(store, "level_candidates") and hasattr(store, "expand_local") \
            and (truncating or store.level_candidates(cost, mask) < REPLICATE_BELOW):
        # small level: every rank builds all of it (see REPLICATE_BELOW); only the budget status is agreed on,
        # because the time budget is read from each rank's own clock
        status, n_new, sep_gid, delta = store.expand_local(cost, mask, config.exhaustive, config.batch_size,
                                                           config.memory_budget_mb << 20, deadline)
        flag = torch.tensor([status], dtype=torch.int64, device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        stats.constructed += delta
        stats.unique = store.total
        if int(flag.item()) in _FAILURE_TEXT:
            raise _BudgetExceeded(_FAILURE_TEXT[int(flag.item())])
        return n_new, sep_gid

    # 1. route: candidates to their hash owners
    status, parts, sep_local, n_seps = store.route_begin(cost, mask, config.exhaustive, deadline, rank, world)
    meta = _gather_ints([status, min(sep_local, _I64_MAX), n_seps] + [p[1].shape[0] for p in parts], device, group)
    worst = max(m[0] for m in meta)
    if worst != 0:  # a budget stop must be collective: every rank stops or none does
        store.level_abort()
        raise _BudgetExceeded(_FAILURE_TEXT.get(worst, "budget exhausted"))
    recv_counts = [m[3 + rank] for m in meta]
    n_records = sum(recv_counts)
    recv_rows, recv_ords = store.exchange_recv(n_records)
    _exchange(parts, (recv_rows, recv_ords), recv_counts, group, include_self=True)
    # 2. reduce on the owner; its winners up to the separator (the min of the ranks' smallest separating ordinals)
    sep_ord = min(m[1] for m in meta)
    sep_ord = NO_SEPARATOR if sep_ord == _I64_MAX else sep_ord
    status, bitmap = store.owner_reduce(n_records)
    win_rows = win_ords = None
    if status == 0:
        win_rows, win_ords = store.winners_export(sep_ord)
    counts = _gather_ints([status, 0 if win_ords is None else win_ords.shape[0]], device, group)
    worst = max(c[0] for c in counts)
    if worst != 0:  # an owner ran out of device memory
        store.level_abort()
        raise _BudgetExceeded(_FAILURE_TEXT.get(worst, "budget exhausted"))
    # 3. rank: the union of the owners' winners bitmaps (disjoint bits: a sum)
    dist.all_reduce(bitmap, op=dist.ReduceOp.SUM, group=group)
    # 4. publish: every owner's winners to every other rank
    seps_mine = store.separating_ordinals() if config.exhaustive else None
    win_counts = [0 if r == rank else counts[r][1] for r in range(world)]
    n_received = sum(win_counts)
    recv_rows, recv_ords = store.exchange_recv(n_received)
    _exchange([(win_rows, win_ords)] * world, (recv_rows, recv_ords), win_counts, group, include_self=False)
    seps = None
    if config.exhaustive:  # every separating ordinal of the level, for the reference's chunk-exact separator id
        sep_counts = [m[2] for m in meta]
        seps = torch.empty((sum(sep_counts),), dtype=torch.int64, device=device)
        _exchange([(seps_mine,)] * world, (seps,), sep_counts, group, include_self=True)
    status, n_new, sep_gid, delta = store.level_commit(sep_ord, seps, [c for c in win_counts if c], config.batch_size,
                                                       config.memory_budget_mb << 20)
    flag = torch.tensor([status], dtype=torch.int64, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)  # (a rank whose device filled up while appending)
    stats.constructed += delta
    stats.unique = store.total
    if int(flag.item()) in _FAILURE_TEXT:
        raise _BudgetExceeded(_FAILURE_TEXT[int(flag.item())])
    return n_new, sep_gid


def _device_of(store) -> torch.device:
    return getattr(store, "torch_device", torch.device("cpu"))


def synthesize_sharded(spec, config: EngineConfig = EngineConfig(), group=None, store_factory=None) -> SynthesisResult:
    """``synthesize`` with every level's pair space sharded over the ranks of ``group``.
    Every rank returns the same result as the single-GPU ``synthesize``."""
    from .engine import CandidateStore

    validate_feasible(spec)
    ops = normalize_operators(config.operators, config.extended_grammar)
    t0 = time.perf_counter()
    if store_factory:
        store = store_factory(spec)
    else:  # on torch's current stream: the collectives and the engine's kernels are then ordered without host waits
        store = CandidateStore(spec, device=config.device, hbm_budget_mb=config.hbm_budget_mb, operator_weights=config.weights,
                               stream=torch.cuda.current_stream(torch.device("cuda", config.device)).cuda_stream)
    try:
        stats = RunStats()
        deadline = t0 + config.time_budget_s
        found, failure = None, None
        for cost in range(1, config.max_cost + 1):
            stats.max_cost_reached = cost
            try:
                _, sep_gid = sharded_expand_level(store, cost, ops, config, stats, deadline, group)
            except _BudgetExceeded as stop:
                failure = str(stop)
                break
            if sep_gid is not None and found is None:
                found = (sep_gid, cost)
                if not config.exhaustive:
                    break
        stats.elapsed_s = time.perf_counter() - t0
        device_stats = store.device_stats() if hasattr(store, "device_stats") else None
        if found is None:
            return SynthesisResult(None, None, False, OUTCOME_EXHAUSTED, stats, failure, device_stats)
        formula = reconstruct(store, found[0])
        device_stats = store.device_stats() if hasattr(store, "device_stats") else None
    finally:
        close = getattr(store, "close", None)
        if close:
            close()
    if not semantics.separates_by_sat(spec, formula):
        raise RuntimeError("internal error: synthesized formula fails the reference semantics")
    return SynthesisResult(formula, found[1], True, OUTCOME_FOUND, stats, None, device_stats)
