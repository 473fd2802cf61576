"""One search sharded over several GPUs: the per-level exchange protocol.

Every rank holds the complete language cache of the finished levels (replicated).  For a
new level each rank enumerates a tile-strided shard of the level's pair space into its
local hash set, then the ranks agree on the level's contents with one exchange:

1. **route**   every rank sends its local claims ``{CM row, min ordinal}`` to the row's hash
               owner (``all_to_all``: counts, then rows and ordinals);
2. **reduce**  the owner folds what it received into its own set (insert-or-min on the device),
               so that for the CMs it owns it now knows the smallest ordinal over all ranks;
3. **publish** every owner ``all_gather``\\ s its winners; every rank folds all of them into its
               set.  Now every set holds exactly the level's new CMs with their global minimum
               ordinals, so the finalisation (rank by ordinal, append, assign ids) produces the
               same level -- bytes, provenance, ids -- on every rank and on one GPU;
4. **separator** ``all_reduce(min)`` of the smallest fresh separating ordinal (plus an
               ``all_gather`` of all separating ordinals in exhaustive runs, for the
               reference's chunk-exact separator id).

The protocol is written against a small shard-engine interface so that the same code runs
over NCCL with the CUDA engine (``CandidateStore``) and, in the CPU test suite, over gloo with
a numpy stand-in.  Collectives move torch tensors that live wherever the engine lives.
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

# Levels with fewer candidates than this are built REDUNDANTLY on every rank instead of being sharded: the
# cache is replicated and the engine is deterministic, so every rank gets the same level without a single
# data-path collective, and a level of a few thousand candidates costs less than one exchange.  The count is
# a closed form of the stored level sizes (`level_candidates`), hence identical on every rank.
REPLICATE_BELOW = int(os.environ.get("LTLB200_REPLICATE_BELOW", str(1 << 22)))


class ShardEngine(Protocol):
    """What the exchange needs from a store (CandidateStore implements it on the GPU)."""

    key_bytes: int

    def level_begin(self, cost: int, op_mask: int, exhaustive: bool, deadline, shard_index: int, shard_count: int):
        """-> (status, n_claimed, sep_ord or NO_SEPARATOR, n_seps)"""

    def claims_count(self, owners: int) -> list[int]: ...

    def claims_pack(self, owners: int, total: int) -> tuple[torch.Tensor, torch.Tensor]:
        """-> rows uint8 [total, key_bytes], ords int64 [total], grouped by owner (owner 0 first)"""

    def claims_import(self, rows: torch.Tensor, ords: torch.Tensor) -> None: ...

    def separating_ordinals(self) -> torch.Tensor:
        """int64 tensor of every separating ordinal recorded in the pending level"""

    def level_end(self, sep_ord: int, seps, batch_size: int, memory_budget_bytes: int):
        """-> (status, n_new, sep_gid or None, constructed_delta)"""

    # optional: without these two every level is sharded
    def level_candidates(self, cost: int, op_mask: int) -> int: ...

    def expand_local(self, cost: int, op_mask: int, exhaustive: bool, batch_size: int, memory_budget_bytes: int, deadline):
        """-> (status, n_new, sep_gid or None, constructed_delta): the whole level on this rank"""


def _all_to_all_v(send: torch.Tensor, send_counts: list[int], recv_counts: list[int], group) -> torch.Tensor:
    """Variable-size all-to-all along dim 0."""
    out = send.new_empty((sum(recv_counts),) + tuple(send.shape[1:]))
    if dist.get_backend(group) == "gloo":
        # gloo has no all_to_all_single for uneven splits everywhere: use pairwise isend/irecv
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        s_off = [0]
        r_off = [0]
        for c in send_counts:
            s_off.append(s_off[-1] + c)
        for c in recv_counts:
            r_off.append(r_off[-1] + c)
        out[r_off[rank]:r_off[rank + 1]] = send[s_off[rank]:s_off[rank + 1]]
        reqs = []
        for peer in range(world):
            if peer == rank:
                continue
            if send_counts[peer]:
                reqs.append(dist.isend(send[s_off[peer]:s_off[peer + 1]].contiguous(), dist.get_global_rank(group, peer) if group else peer, group=group))
            if recv_counts[peer]:
                buf = out[r_off[peer]:r_off[peer + 1]]
                reqs.append(dist.irecv(buf, dist.get_global_rank(group, peer) if group else peer, group=group))
        for r in reqs:
            r.wait()
        return out
    dist.all_to_all_single(out, send.contiguous(), recv_counts, send_counts, group=group)
    return out


def _all_gather_v(local: torch.Tensor, group) -> torch.Tensor:
    """Concatenation over ranks (rank order) of tensors whose dim 0 differs per rank."""
    world = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    sizes = [int(c.item()) for c in counts]
    biggest = max(sizes) if sizes else 0
    if biggest == 0:
        return local.new_empty((0,) + tuple(local.shape[1:]))
    padded = local.new_zeros((biggest,) + tuple(local.shape[1:]))
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:k] for p, k in zip(parts, sizes)], dim=0)


def sharded_expand_level(store: ShardEngine, cost: int, ops, config: EngineConfig, stats: RunStats | None = None,
                         deadline: float | None = None, group=None):
    """``expand_level`` for a search whose pair space is sharded over the ranks of ``group``.

    Returns ``(new entries, separator id or None)`` -- identical on every rank and identical to
    the single-GPU ``expand_level``."""
    stats = stats if stats is not None else RunStats()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mask = operator_mask(ops)
    # ... and so is a NON-exhaustive level over a store that already holds a separating CM, whatever its size: the
    # reference then truncates every chunk at its first separating candidate (engine.py:334-335), which the
    # single-handle expand_level reproduces and the claim exchange (minimum ordinal per CM) cannot
    truncating = (not config.exhaustive) and getattr(store, "holds_separator", lambda: False)()
    if hasattr(store, "level_candidates") and hasattr(store, "expand_local") \
            and (truncating or store.level_candidates(cost, mask) < REPLICATE_BELOW):
        # small level: every rank builds all of it (see REPLICATE_BELOW); only the budget status is agreed on,
        # because the time budget is read from each rank's own clock
        status, n_new, sep_gid, delta = store.expand_local(cost, mask, config.exhaustive, config.batch_size,
                                                           config.memory_budget_mb << 20, deadline)
        flag = torch.tensor([status], dtype=torch.int64, device=_device_of(store))
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        stats.constructed += delta
        stats.unique = store.total
        if int(flag.item()) in _FAILURE_TEXT:
            raise _BudgetExceeded(_FAILURE_TEXT[int(flag.item())])
        return n_new, sep_gid
    status, _, sep_local, _ = store.level_begin(cost, mask, config.exhaustive, deadline, rank, world)

    # a budget stop must be collective: every rank stops or none does
    flag = torch.tensor([status], dtype=torch.int64, device=_device_of(store))
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if int(flag.item()) != 0:
        code = int(flag.item())
        if status == 0:  # this rank began the level: close it empty
            store.level_end(NO_SEPARATOR, None, config.batch_size, 0)
        raise _BudgetExceeded(_FAILURE_TEXT.get(code, "budget exhausted"))

    # 1. route local claims to their hash owners
    send_counts = store.claims_count(world)
    rows, ords = store.claims_pack(world, sum(send_counts))
    counts_t = torch.tensor(send_counts, dtype=torch.int64, device=rows.device)
    recv_t = torch.empty_like(counts_t)
    dist.all_to_all_single(recv_t, counts_t, group=group) if dist.get_backend(group) != "gloo" else _gloo_counts(recv_t, counts_t, group)
    recv_counts = [int(c) for c in recv_t.tolist()]
    got_rows = _all_to_all_v(rows, send_counts, recv_counts, group)
    got_ords = _all_to_all_v(ords, send_counts, recv_counts, group)
    # 2. the owner reduces: min ordinal over all ranks for the CMs it owns
    store.claims_import(got_rows, got_ords)
    # 3. owners publish their winners, everybody folds them in
    own_counts = store.claims_count(world)
    all_rows, all_ords = store.claims_pack(world, sum(own_counts))
    lo = sum(own_counts[:rank])
    mine_rows, mine_ords = all_rows[lo:lo + own_counts[rank]], all_ords[lo:lo + own_counts[rank]]
    store.claims_import(_all_gather_v(mine_rows, group), _all_gather_v(mine_ords, group))
    # 4. separator
    sep_t = torch.tensor([min(sep_local, (1 << 63) - 1)], dtype=torch.int64, device=rows.device)
    dist.all_reduce(sep_t, op=dist.ReduceOp.MIN, group=group)
    sep_ord = int(sep_t.item())
    sep_ord = NO_SEPARATOR if sep_ord == (1 << 63) - 1 else sep_ord
    seps = None
    if config.exhaustive:
        seps = _all_gather_v(store.separating_ordinals(), group)
    status, n_new, sep_gid, delta = store.level_end(sep_ord, seps, config.batch_size, config.memory_budget_mb << 20)
    stats.constructed += delta
    stats.unique = store.total
    if status in _FAILURE_TEXT:
        raise _BudgetExceeded(_FAILURE_TEXT[status])
    return n_new, sep_gid


def _gloo_counts(recv_t, counts_t, group):
    world = dist.get_world_size(group)
    parts = [torch.empty_like(counts_t) for _ in range(world)]
    dist.all_gather(parts, counts_t, group=group)
    rank = dist.get_rank(group)
    for peer in range(world):
        recv_t[peer] = parts[peer][rank]


def _device_of(store) -> torch.device:
    return getattr(store, "torch_device", torch.device("cpu"))


def synthesize_sharded(spec, config: EngineConfig = EngineConfig(), group=None, store_factory=None) -> SynthesisResult:
    """``synthesize`` with every level's pair space sharded over the ranks of ``group``.
    Every rank returns the same result as the single-GPU ``synthesize``."""
    from .engine import CandidateStore

    validate_feasible(spec)
    ops = normalize_operators(config.operators)
    t0 = time.perf_counter()
    store = store_factory(spec) if store_factory else CandidateStore(spec, device=config.device, hbm_budget_mb=config.hbm_budget_mb)
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
        if found is None:
            return SynthesisResult(None, None, False, OUTCOME_EXHAUSTED, stats, failure)
        formula = reconstruct(store, found[0])
    finally:
        close = getattr(store, "close", None)
        if close:
            close()
    if not semantics.separates_by_sat(spec, formula):
        raise RuntimeError("internal error: synthesized formula fails the reference semantics")
    return SynthesisResult(formula, found[1], True, OUTCOME_FOUND, stats)
