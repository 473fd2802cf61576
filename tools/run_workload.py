#!/usr/bin/env python3
"""Run one named workload through the public API on cuda:0 and print per-level device timings."""
import argparse
import json
import sys
import time
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2504_18943_b200 import engine, to_text, workloads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-cost", type=int, default=16)
    ap.add_argument("--exhaustive", action="store_true")
    ap.add_argument("--repeat", type=int, default=1)
    args = ap.parse_args()
    spec = workloads.named_workload(args.workload, args.seed)
    cfg = engine.EngineConfig(max_cost=args.max_cost, exhaustive=args.exhaustive, memory_budget_mb=1 << 20,
                              time_budget_s=3600)
    for rep in range(args.repeat):
        store = engine.CandidateStore(spec)
        stats = engine.RunStats()
        t0 = time.perf_counter()
        prev = store.device_stats()
        for cost in range(1, cfg.max_cost + 1):
            t1 = time.perf_counter()
            try:
                n_new, sep = engine.expand_level(store, cost, cfg.operators, config=cfg, stats=stats)
            except engine._BudgetExceeded as e:
                print("budget:", e)
                break
            st = store.device_stats()
            print(json.dumps(dict(cost=cost, n_new=n_new, sep=sep, constructed=stats.constructed,
                                  wall_ms=round(1e3 * (time.perf_counter() - t1), 3),
                                  enum_ms=round(st["enumerate_ms"] - prev["enumerate_ms"], 3),
                                  fin_ms=round(st["finalize_ms"] - prev["finalize_ms"], 3),
                                  slots=st["table_slots"], rebuilds=st["table_rebuilds"],
                                  dev_mb=st["device_bytes"] >> 20)), flush=True)
            prev = st
            if sep is not None and not cfg.exhaustive:
                print("formula:", to_text(engine.reconstruct(store, sep), spec.alphabet))
                break
        wall = time.perf_counter() - t0
        st = store.device_stats()
        print(json.dumps(dict(rep=rep, wall_s=round(wall, 4), constructed=stats.constructed, unique=store.total,
                              enum_ms=round(st["enumerate_ms"], 3), fin_ms=round(st["finalize_ms"], 3),
                              cand_per_s=round(stats.constructed / wall), launches=st["kernel_launches"],
                              alloc_ms=round(st["alloc_ms"], 3), rebuild_host_ms=round(st["rebuild_host_ms"], 3), create_ms=round(st["create_ms"], 3), rebuilds=st["table_rebuilds"])), flush=True)
        store.close()


if __name__ == "__main__":
    main()
