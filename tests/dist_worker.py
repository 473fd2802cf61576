"""Worker of the world-size-2 gloo tests: runs the multi-GPU exchange protocol on CPU with the
numpy shard engine and checks every level, on every rank, against the C oracle."""

import json
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np
import torch.distributed as dist

import oracle
from cpu_shard_engine import CpuShardEngine
from paper_2504_18943_b200 import dist as pdist
from paper_2504_18943_b200 import to_text, workloads
from paper_2504_18943_b200.engine import EngineConfig, RunStats


def main():
    workload, seed, max_cost, exhaustive, ops = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == "1", sys.argv[5].split(",")
    dist.init_process_group("gloo", rank=int(os.environ["RANK"]), world_size=int(os.environ["WORLD_SIZE"]))
    rank = dist.get_rank()
    spec = workloads.named_workload(workload, seed)
    cfg = EngineConfig(operators=tuple(ops), max_cost=max_cost, exhaustive=exhaustive, memory_budget_mb=1 << 20)
    report = dict(rank=rank, levels=[])

    # level by level against the oracle
    store, ref, stats = CpuShardEngine(spec), oracle.OracleStore(spec), RunStats()
    found = None
    for cost in range(1, max_cost + 1):
        n_new, sep = pdist.sharded_expand_level(store, cost, cfg.operators, cfg, stats)
        o_new, o_sep, _, _ = ref.expand_level(cost, cfg.operators, exhaustive, cfg.batch_size, memory_budget_mb=1 << 20)
        a, b = store.level(cost), ref.level(cost)
        assert n_new == o_new == a.n, (cost, n_new, o_new)
        assert a.base == b.base
        for name in ("cms", "op", "left", "right"):
            assert np.array_equal(getattr(a, name), getattr(b, name)), (cost, name)
        if found is None:
            assert sep == o_sep, (cost, sep, o_sep)
        report["levels"].append(n_new)
        if sep is not None and found is None:
            found = (sep, cost)
            if not exhaustive:
                break

    # whole search through synthesize_sharded
    res = pdist.synthesize_sharded(spec, cfg, store_factory=CpuShardEngine)
    want = oracle.synthesize(spec, operators=cfg.operators, max_cost=max_cost, exhaustive=exhaustive)
    assert res.outcome == want.outcome and res.cost == want.cost
    if want.formula is not None:
        assert to_text(res.formula, spec.alphabet) == to_text(want.formula, spec.alphabet)
    assert res.stats.unique == want.unique
    report["formula"] = None if res.formula is None else to_text(res.formula, spec.alphabet)
    report["unique"] = res.stats.unique
    dist.barrier()
    dist.destroy_process_group()
    pathlib.Path(sys.argv[6] + f".{rank}").write_text(json.dumps(report))


if __name__ == "__main__":
    main()
