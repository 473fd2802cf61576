"""Full-size properties of the GPU engine (sizes the CPU oracle cannot replay in a test).

`c3` (2 atoms, 8+8 traces of length 8: CM = exactly one uint4) is enumerated exhaustively through
cost 14 -- 82.5 M candidates, 19.1 M stored CMs -- and checked through properties that do not
depend on size (SURVEY 8c / tier rule 3):

  * levels <= 12 still match the golden digests of the unmodified reference;
  * `constructed` of every level equals the closed form of the canonical block list
    (#unary ops * n(c-1) + rectangles n(c1)*n(c2) + same-cost triangles n(n+1)/2);
  * all stored CMs are pairwise distinct (observational-equivalence dedup; reference
    tests/test_engine.py:81-87), checked on the device with a row-wise unique;
  * children sit strictly below their parent's level (reference tests/test_engine.py:90-99);
  * every stored CM is reproduced by applying its recorded operator to its recorded children
    (reconstruct round trip, reference tests/test_engine.py:102-117), on the device for all rows;
  * a second run gives the same digests (determinism of the concurrent hash set + min-ordinal rule).
"""

import numpy as np
import pytest

from helpers import level_digests, load_golden
from paper_2504_18943_b200 import engine, workloads
from paper_2504_18943_b200.engine import OP_AND, OP_FUTURE, OP_NEXT, OP_NOT, OP_UNTIL

pytestmark = pytest.mark.gpu

MAX_COST = 14


def _closed_form(sizes, cost, n_unary=3):
    if cost == 1:
        return None
    total = n_unary * sizes[cost - 1]
    for commutative in (True, False):  # AND, then UNTIL (default operator set)
        for c1 in range(1, cost - 1):
            c2 = cost - 1 - c1
            if commutative and c1 > c2:
                break
            na, nb = sizes[c1], sizes[c2]
            total += na * (na + 1) // 2 if (commutative and c1 == c2) else na * nb
    return total


def _run():
    spec = workloads.named_workload("c3", 0)
    cfg = engine.EngineConfig(exhaustive=True, max_cost=MAX_COST, memory_budget_mb=1 << 20, time_budget_s=3600)
    store = engine.CandidateStore(spec)
    stats = engine.RunStats()
    per_level = []
    for cost in range(1, MAX_COST + 1):
        before = stats.constructed
        n_new, _ = engine.expand_level(store, cost, cfg.operators, config=cfg, stats=stats)
        per_level.append((n_new, stats.constructed - before))
    return spec, store, stats, per_level


def test_c3_full_size_properties():
    import torch

    spec, store, stats, per_level = _run()
    try:
        gold = load_golden("c3_s0_exh12")
        for gl in gold["levels"]:
            got = level_digests(store.level(gl["cost"]))
            assert all(got[k] == gl[k] for k in got), f"cost {gl['cost']} differs from the reference"
        sizes = {c: store.level(c).n for c in range(1, MAX_COST + 1)}
        assert stats.unique == store.total == sum(sizes.values())
        for cost in range(2, MAX_COST + 1):
            assert per_level[cost - 1][1] == _closed_form(sizes, cost), f"constructed of cost {cost}"

        dev = torch.device("cuda", 0)
        rows = torch.from_numpy(store.all_cms().view(np.int64).reshape(-1, 2)).to(dev)  # 16 bytes = 2 x int64
        assert rows.shape[0] == store.total
        assert torch.unique(rows, dim=0).shape[0] == store.total, "stored CMs are not pairwise distinct"

        # provenance: children strictly below the level, and op(children) == the stored CM, for every row
        lanes = torch.from_numpy(store.all_cms()).to(dev)  # (N, 16) uint8, one lane per trace
        masks = torch.from_numpy(np.array(store.layout.masks, copy=True)).to(dev)
        for cost in range(2, MAX_COST + 1):
            lv = store.level(cost)
            op = torch.from_numpy(lv.op.astype(np.int64)).to(dev)
            left = torch.from_numpy(lv.left).to(dev)
            right = torch.from_numpy(lv.right).to(dev)
            assert int(left.max()) < lv.base and int(right.max()) < lv.base
            a = lanes[left]
            b = lanes[torch.clamp(right, min=0)]
            want = lanes[lv.base:lv.base + lv.n]
            got = torch.zeros_like(want)
            m = op == OP_NOT
            got[m] = (~a[m]) & masks
            m = op == OP_NEXT
            got[m] = a[m] >> 1
            m = op == OP_FUTURE
            f = a[m]
            for s in (1, 2, 4):
                f = f | (f >> s)
            got[m] = f
            m = op == OP_AND
            got[m] = a[m] & b[m]
            m = op == OP_UNTIL
            r, q = b[m], a[m]
            for s in (1, 2, 4):
                r = r | (q & (r >> s))
                q = q & (q >> s)
            got[m] = r & masks
            assert torch.equal(got, want), f"cost {cost}: a stored CM is not op(children)"
        first = [level_digests(store.level(c)) for c in range(1, MAX_COST + 1)]
    finally:
        store.close()

    _, again, _, _ = _run()
    try:
        assert [level_digests(again.level(c)) for c in range(1, MAX_COST + 1)] == first
    finally:
        again.close()
