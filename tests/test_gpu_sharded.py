"""GPU tests of the sharded-search primitives of the C ABI (route_begin / owner_reduce / winners_export / level_commit).

Only one GPU is available to the test run, so two stores on the same device play two ranks
and the test moves the exchange records between them by hand, step for step as
dist.sharded_expand_level does over NCCL; a second test drives the real protocol code through
a one-rank NCCL group.  Bar: both "ranks" end every level byte-identical to the CPU oracle."""

import os
import socket

import pytest
import torch

import oracle
from helpers import assert_levels_equal
from paper_2504_18943_b200 import dist as pdist
from paper_2504_18943_b200 import engine, to_text, workloads

pytestmark = pytest.mark.gpu
NO_SEP = (1 << 64) - 1


def _exchange_level(stores, cost, cfg, mask=None):
    """dist.sharded_expand_level with the collectives done by hand between stores on one device."""
    world = len(stores)
    mask = engine.operator_mask(cfg.operators) if mask is None else mask
    # 1. route
    begun = [s.route_begin(cost, mask, cfg.exhaustive, None, r, world) for r, s in enumerate(stores)]
    assert all(b[0] == 0 for b in begun)
    for owner, s in enumerate(stores):  # "all-to-all": what every rank built for this owner, source-major
        counts = [begun[src][1][owner][1].shape[0] for src in range(world)]
        rows, ords = s.exchange_recv(sum(counts))
        at = 0
        for src in range(world):
            part_rows, part_ords = begun[src][1][owner]
            rows[at:at + counts[src]].copy_(part_rows)
            ords[at:at + counts[src]].copy_(part_ords)
            at += counts[src]
    torch.cuda.synchronize()
    sep = min(b[2] for b in begun)
    # 2. reduce, 3. rank ("all-reduce": sum of the owners' bitmaps)
    reduced = [s.owner_reduce(sum(begun[src][1][owner][1].shape[0] for src in range(world))) for owner, s in enumerate(stores)]
    assert all(r[0] == 0 for r in reduced)
    winners = [s.winners_export(sep) for s in stores]
    total = sum(r[1] for r in reduced)
    for _, bitmap in reduced:
        bitmap.copy_(total)
    # 4. publish ("all-gather": the winners of the other owners)
    received = []
    for r, s in enumerate(stores):
        others = [winners[o] for o in range(world) if o != r]
        n = sum(w[1].shape[0] for w in others)
        rows, ords = s.exchange_recv(n)
        at = 0
        for w_rows, w_ords in others:
            k = w_ords.shape[0]
            rows[at:at + k].copy_(w_rows)
            ords[at:at + k].copy_(w_ords)
            at += k
        received.append([w[1].shape[0] for w in others if w[1].shape[0]])
    torch.cuda.synchronize()
    seps = torch.cat([s.separating_ordinals() for s in stores]) if cfg.exhaustive else None
    return [s.level_commit(sep, seps, received[r], cfg.batch_size, 0) for r, s in enumerate(stores)]


@pytest.mark.parametrize("workload,seed,max_cost,exhaustive,world", [
    ("spec1", 0, 6, False, 2),
    ("spec2", 0, 10, True, 2),
    ("c3", 0, 9, True, 3),
    ("c5", 0, 7, True, 2),       # 128-byte rows
    ("c3wide", 0, 7, True, 2),   # 80-byte rows (5 vectors in groups of 8 lanes)
    ("c1", 1, 14, False, 2),
    ("c3", 1, 11, True, 8),      # the most ranks a route kernel stages for
    ("w64n", 0, 9, True, 4),     # 64-bit lanes
    ("c3", 0, 13, True, 2),      # 12 M candidates in the last level: big route regions, probe kernel at scale
    ("spec2", 0, 14, False, 3),  # non-exhaustive, no separator up to here
])
def test_shards_on_one_gpu_agree_with_oracle(workload, seed, max_cost, exhaustive, world):
    spec = workloads.named_workload(workload, seed)
    cfg = engine.EngineConfig(max_cost=max_cost, exhaustive=exhaustive, memory_budget_mb=1 << 20)
    stores = [engine.CandidateStore(spec) for _ in range(world)]
    ref = oracle.OracleStore(spec)
    try:
        found = None
        for cost in range(1, max_cost + 1):
            results = _exchange_level(stores, cost, cfg)
            o_new, o_sep, o_delta, _ = ref.expand_level(cost, cfg.operators, exhaustive, cfg.batch_size, memory_budget_mb=1 << 20)
            for r, (status, n_new, sep, delta) in enumerate(results):
                where = f"{workload} cost {cost} rank {r}"
                assert (status, n_new, sep, delta) == (0, o_new, o_sep, o_delta), where
                assert_levels_equal(stores[r].level(cost), ref.level(cost), where)
            if o_sep is not None and found is None:
                found = (o_sep, cost)
                if not exhaustive:
                    break
        if found:
            want = to_text(oracle.reconstruct(ref, found[0]), spec.alphabet)
            assert all(to_text(engine.reconstruct(s, found[0]), spec.alphabet) == want for s in stores)
    finally:
        for s in stores:
            s.close()


def test_protocol_over_nccl_with_one_rank():
    import torch.distributed as dist

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    default_threshold = pdist.REPLICATE_BELOW
    try:
        spec = workloads.spec2()
        cfg = engine.EngineConfig(max_cost=11, exhaustive=True, memory_budget_mb=1 << 20)
        want = oracle.synthesize(spec, max_cost=11, exhaustive=True)
        # every level through the exchange / levels under 10,000 candidates built locally / (default) all local
        for replicate_below in (0, 10_000, default_threshold):
            pdist.REPLICATE_BELOW = replicate_below
            res = pdist.synthesize_sharded(spec, cfg)
            assert (res.outcome, res.stats.unique, res.stats.constructed) == (want.outcome, want.unique, want.constructed)
            res = pdist.synthesize_sharded(workloads.spec1(), engine.EngineConfig())
            assert to_text(res.formula, workloads.spec1().alphabet) == "!(b U a)"
    finally:
        pdist.REPLICATE_BELOW = default_threshold
        dist.destroy_process_group()


def test_sharded_protocol_follows_the_reference_on_truncating_levels():
    """Non-exhaustive levels over a store that already holds a separating CM through dist.sharded_expand_level with
    every level forced through the exchange: the protocol must hand exactly those levels to the single-handle path
    (reference chunk truncation, engine.py:334-335) and so reproduce the reference's fixtures."""
    import json
    import pathlib

    import torch.distributed as dist

    from helpers import assert_level_matches_golden

    cases = [c for c in json.loads((pathlib.Path(__file__).resolve().parent / "golden_schedules" / "schedules.json").read_text())
             if c["name"] in ("c1_s0_cut_then_nonexhaustive", "c1_s4_cut_then_nonexhaustive", "w32_s0_cut_then_nonexhaustive")]
    assert len(cases) == 3
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    default_threshold = pdist.REPLICATE_BELOW
    try:
        pdist.REPLICATE_BELOW = 0
        for case in cases:
            spec = workloads.named_workload(case["workload"], case["seed"])
            store = engine.CandidateStore(spec)
            try:
                for (ops, exhaustive), gl in zip(case["schedule"], case["levels"]):
                    cfg = engine.EngineConfig(exhaustive=exhaustive, operators=tuple(ops), memory_budget_mb=1 << 20)
                    stats = engine.RunStats()
                    n_new, sep = pdist.sharded_expand_level(store, gl["cost"], tuple(ops), cfg, stats)
                    where = f"{case['name']} cost {gl['cost']}"
                    assert (n_new, sep, stats.constructed) == (gl["n"], gl["sep_gid"], gl["constructed"]), where
                    assert_level_matches_golden(store.level(gl["cost"]), dict(gl, base=store.level(gl["cost"]).base), where)
            finally:
                store.close()
    finally:
        pdist.REPLICATE_BELOW = default_threshold
        dist.destroy_process_group()
