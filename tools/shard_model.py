#!/usr/bin/env python3
"""Per-rank work of a sharded search, measured on ONE GPU (measurement tool, not product code).

    python tools/shard_model.py [--workload c3] [--max-cost 14] [--world 1 2 4 8]

No box with several GPUs is available to this repository's runs, so the ranks of an N-GPU search are played one
after the other by N stores on the same device: every store runs the real phases of dist.sharded_expand_level --
route (its 1/N share of the pair space), owner-side reduce (the records of its 1/N of the key space), publish,
commit -- and the "collectives" are device-to-device copies.  What this yields is the PER-RANK device time of every
phase as a function of N (the terms of DESIGN.md's work model) and the bytes each rank would put on NVLink; what it
cannot yield is the collectives' own time and the overlap between ranks.  One JSON line per N.
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2504_18943_b200 import dist as pdist  # noqa: E402
from paper_2504_18943_b200 import engine, workloads  # noqa: E402


def exchange_level(stores, cost, cfg, acc):
    world = len(stores)
    mask = engine.operator_mask(cfg.operators)
    key_bytes = stores[0].key_bytes
    begun = [s.route_begin(cost, mask, cfg.exhaustive, None, r, world) for r, s in enumerate(stores)]
    per_owner = []
    for owner, s in enumerate(stores):
        counts = [begun[src][1][owner][1].shape[0] for src in range(world)]
        rows, ords = s.exchange_recv(sum(counts))
        at = 0
        for src in range(world):
            rows[at:at + counts[src]].copy_(begun[src][1][owner][0])
            ords[at:at + counts[src]].copy_(begun[src][1][owner][1])
            at += counts[src]
        per_owner.append(sum(counts))
        acc["a2a_bytes_per_rank"] += (sum(counts) - counts[owner]) * (key_bytes + 8) / world
    torch.cuda.synchronize()
    sep = min(b[2] for b in begun)
    reduced = [s.owner_reduce(per_owner[o]) for o, s in enumerate(stores)]
    winners = [s.winners_export(sep) for s in stores]
    total = sum(r[1] for r in reduced)
    acc["bitmap_bytes_per_rank"] += total.numel() * 4
    for _, bitmap in reduced:
        bitmap.copy_(total)
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
        acc["gather_bytes_per_rank"] += n * (key_bytes + 8) / world
    torch.cuda.synchronize()
    seps = torch.cat([s.separating_ordinals() for s in stores]) if cfg.exhaustive else None
    return [s.level_commit(sep, seps, received[r], cfg.batch_size, 0) for r, s in enumerate(stores)]


def main() -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--max-cost", type=int, default=14)
    ap.add_argument("--world", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--hbm-mb", type=int, default=0, help="device-memory budget per store (0: an equal share of the device)")
    args = ap.parse_args()
    spec = workloads.named_workload(args.workload, 0)
    cfg = engine.EngineConfig(max_cost=args.max_cost, exhaustive=True, memory_budget_mb=1 << 22)

    # the single-GPU engine on the same workload, for the N = 1 reference line (second run: buffers allocated, clocks up)
    store = engine.CandidateStore(spec)
    for attempt in range(2):
        store.reset()
        before = store.device_stats()
        stats = engine.RunStats()
        t0 = time.perf_counter()
        for cost in range(1, args.max_cost + 1):
            engine.expand_level(store, cost, cfg.operators, config=cfg, stats=stats)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    single = store.device_stats()
    print(json.dumps({"mode": "single-GPU engine (fused construct + probe)", "workload": args.workload, "max_cost": args.max_cost,
                      "unique": stats.unique, "constructed": stats.constructed,
                      "enumerate_ms": single["enumerate_ms"] - before["enumerate_ms"],
                      "finalize_ms": single["finalize_ms"] - before["finalize_ms"], "wall_ms": 1e3 * wall}), flush=True)
    store.close()

    free_mb = torch.cuda.mem_get_info()[0] >> 20
    for world in args.world:
        budget = args.hbm_mb or int(free_mb * 0.9 / world)
        stores = [engine.CandidateStore(spec, hbm_budget_mb=budget) for _ in range(world)]
        acc = {"a2a_bytes_per_rank": 0.0, "bitmap_bytes_per_rank": 0.0, "gather_bytes_per_rank": 0.0}
        try:
            for attempt in range(2):  # the second run is the measured one (buffers allocated)
                for s in stores:
                    s.reset()
                for k in acc:
                    acc[k] = 0.0
                base = [s.device_stats() for s in stores]
                for cost in range(1, args.max_cost + 1):
                    # small levels are built by every rank on its own, as dist.sharded_expand_level does
                    if stores[0].level_candidates(cost, engine.operator_mask(cfg.operators)) < pdist.REPLICATE_BELOW:
                        for s in stores:
                            s.expand_local(cost, engine.operator_mask(cfg.operators), True, cfg.batch_size, 0, None)
                        continue
                    exchange_level(stores, cost, cfg, acc)
            per_rank = [{k: (v - base[r][k] if k.endswith("_ms") or k.endswith("_records") else v) for k, v in s.device_stats().items()}
                        for r, s in enumerate(stores)]
            mean = lambda key: sum(p[key] for p in per_rank) / world
            worst = lambda key: max(p[key] for p in per_rank)
            print(json.dumps({
                "mode": "sharded search, ranks played in turn on one GPU", "world": world, "workload": args.workload,
                "max_cost": args.max_cost, "unique": stores[0].total,
                "route_ms_per_rank": mean("route_ms"), "route_ms_max": worst("route_ms"),
                "probe_ms_per_rank": mean("probe_ms"), "probe_ms_max": worst("probe_ms"),
                "finalize_ms_per_rank": mean("finalize_ms"),
                "local_small_levels_ms_per_rank": mean("enumerate_ms") - mean("route_ms") - mean("probe_ms"),
                "routed_records_per_rank": mean("routed_records"), "received_records_per_rank": mean("received_records"),
                "table_slots_per_rank": mean("table_slots"), "device_bytes_per_rank": mean("device_bytes"),
                "nvlink_bytes_per_rank": {k: v for k, v in acc.items()},
            }), flush=True)
        finally:
            for s in stores:
                s.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
