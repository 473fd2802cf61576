"""Full-size properties of the WIDE path (multi-vector CMs; sizes the CPU oracle cannot replay in a test).

`c5` (BASELINE configs[4]: 4 atoms, 32+32 traces of length 16, 128-byte CMs) exhaustively through cost 12 --
170.6 M candidates, 100.8 M stored CMs, 12.9 GB of rows -- and `c4-1024` (BASELINE configs[3]: 3 atoms, 32+32 traces
of length <= 16, 1024-bit CMs) through cost 11, checked through properties that do not depend on size, on the
device (the rows never leave it: CandidateStore.level_device):

  * the levels the unmodified reference reaches still match its golden digests (c5: cost <= 11, 19.0 M CMs;
    c4-1024: cost <= 10);
  * `constructed` of every level equals the closed form of the canonical block list;
  * all stored CMs are pairwise distinct (reference tests/test_engine.py:81-87): two independent 64-bit hashes of
    every row, no hash pair twice;
  * children sit strictly below their parent's level and op(children) == the stored CM for EVERY row
    (reference tests/test_engine.py:90-117);
  * a second run -- with the new-CM estimate scaled down (LTLB200_EST_SCALE) so that the staging pool overflows and
    every big level goes through regrow + redo -- gives the same order-sensitive digests: determinism of the
    concurrent set and exactness of the overflow path.

A third test drives `c3` into the device-memory limit with a small `hbm_budget_mb` and expects the reference's
outcome for a spent memory budget (reference engine.py:443-444, tests/test_engine.py:192-198).
"""

import os
import pathlib
import subprocess
import sys

import numpy as np
import pytest

from helpers import level_digests, load_golden
from paper_2504_18943_b200 import engine, workloads
from paper_2504_18943_b200.engine import OP_AND, OP_FUTURE, OP_NEXT, OP_NOT, OP_UNTIL

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parent.parent
CHUNK = 1 << 21  # rows per provenance-check step


def _closed_form(sizes, cost, n_unary=3):
    total = n_unary * sizes[cost - 1]
    for commutative in (True, False):  # AND, then UNTIL (default operator set)
        for c1 in range(1, cost - 1):
            c2 = cost - 1 - c1
            if commutative and c1 > c2:
                break
            na, nb = sizes[c1], sizes[c2]
            total += na * (na + 1) // 2 if (commutative and c1 == c2) else na * nb
    return total


def _build(workload, max_cost):
    spec = workloads.named_workload(workload, 0)
    cfg = engine.EngineConfig(exhaustive=True, max_cost=max_cost, memory_budget_mb=1 << 22, time_budget_s=3600)
    store = engine.CandidateStore(spec)
    stats, per_level = engine.RunStats(), []
    for cost in range(1, max_cost + 1):
        before = stats.constructed
        n_new, _ = engine.expand_level(store, cost, cfg.operators, config=cfg, stats=stats)
        per_level.append((n_new, stats.constructed - before))
    return store, stats, per_level


def _lanes(rows_u8, lane_bytes, trace_count):
    """[n, key_bytes] uint8 rows -> [n, T] int32 lanes (values of the unsigned lane type)."""
    import torch

    assert lane_bytes == 2
    pairs = rows_u8[:, : trace_count * 2].reshape(rows_u8.shape[0], trace_count, 2).to(torch.int32)
    return pairs[:, :, 0] | (pairs[:, :, 1] << 8)


def _row_hashes(rows_u8):
    """two independent 64-bit hashes per row (int64 wrap-around arithmetic on the row's 8-byte words)"""
    import torch

    words = rows_u8.view(torch.int64)
    g = torch.Generator(device="cpu").manual_seed(12345)
    k1 = (torch.randint(-(1 << 62), 1 << 62, (words.shape[1],), generator=g, dtype=torch.int64) | 1).to(words.device)
    k2 = (torch.randint(-(1 << 62), 1 << 62, (words.shape[1],), generator=g, dtype=torch.int64) | 1).to(words.device)
    h1 = (words * k1).sum(dim=1)
    h2 = ((words ^ (words >> 29)) * k2).sum(dim=1)
    return h1, h2


def _device_digest(store, max_cost):
    """order-sensitive digest of every level's rows and ordinals, computed on the device"""
    import torch

    out = []
    for cost in range(1, max_cost + 1):
        rows, ords = store.level_device(cost)
        if rows.shape[0] == 0:
            out.append((0, 0, 0))
            continue
        h1, h2 = _row_hashes(rows)
        pos = torch.arange(1, rows.shape[0] + 1, dtype=torch.int64, device=rows.device)
        out.append((int((h1 * (2 * pos + 1)).sum().item()), int((h2 ^ pos).sum().item()), int((ords * (2 * pos + 1)).sum().item())))
    return out


def _check_properties(workload, max_cost, golden, golden_cost):
    import torch

    store, stats, per_level = _build(workload, max_cost)
    try:
        gold = load_golden(golden)
        for gl in gold["levels"][:golden_cost]:
            got = level_digests(store.level(gl["cost"]))
            assert all(got[k] == gl[k] for k in got), f"{workload} cost {gl['cost']} differs from the reference"
        sizes = {c: store.level(c).n for c in range(1, max_cost + 1)}
        assert stats.unique == store.total == sum(sizes.values())
        for cost in range(2, max_cost + 1):
            assert per_level[cost - 1][1] == _closed_form(sizes, cost), f"{workload}: constructed of cost {cost}"

        dev = torch.device("cuda", 0)
        T, lane_bytes = store.trace_count, store.dtype.itemsize
        lane_bits = 8 * lane_bytes
        views = [store.level_device(c)[0] for c in range(1, max_cost + 1)]
        # ---- pairwise distinct
        h1 = torch.cat([_row_hashes(v)[0] for v in views if v.shape[0]])
        h2 = torch.cat([_row_hashes(v)[1] for v in views if v.shape[0]])
        assert h1.shape[0] == store.total
        order = torch.argsort(h1)
        same = (h1[order][1:] == h1[order][:-1]) & (h2[order][1:] == h2[order][:-1])
        assert not bool(same.any()), f"{workload}: two stored CMs are equal"
        del h1, h2, order, same
        # ---- provenance, level by level in chunks: op(children) == stored CM
        bases = [store.level(c).base for c in range(1, max_cost + 1)]
        all_rows = torch.cat([v for v in views if v.shape[0]])  # ids are positions in this concatenation
        masks = torch.from_numpy(np.array(store.layout.masks, copy=True).astype(np.int32)).to(dev)
        shifts = [s for s in (1, 2, 4, 8, 16, 32) if s < lane_bits]
        for cost in range(2, max_cost + 1):
            lv = store.level(cost)
            op_h, left_h, right_h = store._copy_provenance(cost, lv.n)
            assert int(left_h.max()) < lv.base and int(right_h.max()) < lv.base, f"{workload} cost {cost}: child not below the level"
            for lo in range(0, lv.n, CHUNK):
                hi = min(lv.n, lo + CHUNK)
                op = torch.from_numpy(op_h[lo:hi].astype(np.int64)).to(dev)
                left = torch.from_numpy(left_h[lo:hi]).to(dev)
                right = torch.from_numpy(right_h[lo:hi]).to(dev).clamp(min=0)
                a = _lanes(all_rows[left], lane_bytes, T)
                b = _lanes(all_rows[right], lane_bytes, T)
                want = _lanes(all_rows[bases[cost - 1] + lo: bases[cost - 1] + hi], lane_bytes, T)
                fut = a.clone()
                for s in shifts:
                    fut |= fut >> s
                r, q = b.clone(), a.clone()
                for s in shifts:
                    r |= q & (r >> s)
                    q &= q >> s
                got = torch.where((op == OP_NOT)[:, None], (~a) & masks,
                      torch.where((op == OP_NEXT)[:, None], a >> 1,
                      torch.where((op == OP_FUTURE)[:, None], fut,
                      torch.where((op == OP_AND)[:, None], a & b, r & masks))))
                assert bool(((op == OP_NOT) | (op == OP_NEXT) | (op == OP_FUTURE) | (op == OP_AND) | (op == OP_UNTIL)).all())
                assert torch.equal(got, want), f"{workload} cost {cost} rows {lo}..{hi}: a stored CM is not op(children)"
        del all_rows
        return _device_digest(store, max_cost), sizes
    finally:
        store.close()


CHILD = """
import sys, json
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import test_gpu_scale_wide as t
store, stats, per_level = t._build({workload!r}, {max_cost})
print("DIGEST " + json.dumps([t._device_digest(store, {max_cost}), store.device_stats()["table_rebuilds"]]))
store.close()
"""


def _digest_with_forced_overflow(workload, max_cost):
    import json

    env = dict(os.environ, LTLB200_EST_SCALE="0.05")
    code = CHILD.format(root=str(ROOT), tests=str(ROOT / "tests"), workload=workload, max_cost=max_cost)
    proc = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=1200)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-4000:]
    digest, rebuilds = json.loads([ln for ln in proc.stdout.splitlines() if ln.startswith("DIGEST ")][-1][7:])
    return [tuple(d) for d in digest], rebuilds


def test_c5_full_size_properties_and_overflow_redo():
    digest, sizes = _check_properties("c5", 12, "c5_s0_exh11", 11)
    assert sum(sizes.values()) == 100_803_440
    again, rebuilds = _digest_with_forced_overflow("c5", 12)
    assert again == digest, "the overflow -> regrow -> redo path changed the result"
    assert rebuilds >= 6, "the scaled-down estimate did not force any redo"


def test_c4_1024_full_size_properties_and_overflow_redo():
    digest, _ = _check_properties("c4-1024", 11, "c4-1024_s0_exh10", 10)
    again, _ = _digest_with_forced_overflow("c4-1024", 11)
    assert again == digest


def test_device_memory_exhaustion_ends_with_the_reference_outcome():
    """A search that fills its device-memory budget stops with outcome "exhausted" / "memory budget exhausted", like
    the reference when its accounting passes memory_budget_mb (engine.py:443-444), and everything stored before is intact."""
    # the paper's 7+7 example has no separator below cost 16, and its cost-15 level needs a 1 GB set
    res = engine.synthesize(workloads.spec2(), engine.EngineConfig(max_cost=16, memory_budget_mb=1 << 22, hbm_budget_mb=1024))
    assert res.outcome == "exhausted" and res.failure == "memory budget exhausted" and res.formula is None
    assert res.stats.unique > 1_000_000 and 14 <= res.stats.max_cost_reached <= 16
    spec = workloads.named_workload("c3", 0)
    cfg = engine.EngineConfig(exhaustive=True, max_cost=20, memory_budget_mb=1 << 22, time_budget_s=3600, hbm_budget_mb=1536)
    # level by level: the levels completed before the budget ran out are the reference's
    store = engine.CandidateStore(spec, hbm_budget_mb=1536)
    try:
        gold = load_golden("c3_s0_exh12")
        stats = engine.RunStats()
        for gl in gold["levels"]:
            engine.expand_level(store, gl["cost"], cfg.operators, config=cfg, stats=stats)
            got = level_digests(store.level(gl["cost"]))
            assert all(got[k] == gl[k] for k in got)
        with pytest.raises(engine._BudgetExceeded, match="memory budget exhausted"):
            for cost in range(13, 21):
                engine.expand_level(store, cost, cfg.operators, config=cfg, stats=stats)
        assert store.total == stats.unique >= sum(g["n"] for g in gold["levels"])
    finally:
        store.close()


def test_deadline_is_polled_inside_a_level():
    """The reference checks its deadline before every chunk (engine.py:416-417); the device checks it with every tile a
    warp starts: a level that would run for tens of milliseconds stops a few milliseconds after its deadline, keeps
    the partial level and reports the reference's failure text."""
    import time

    spec = workloads.named_workload("c5", 0)
    cfg = engine.EngineConfig(exhaustive=True, max_cost=12, memory_budget_mb=1 << 22)
    full = None
    for budget_s in (None, 0.004):
        store = engine.CandidateStore(spec)
        try:
            stats = engine.RunStats()
            for cost in range(1, 12):
                engine.expand_level(store, cost, cfg.operators, config=cfg, stats=stats)
            t0 = time.perf_counter()
            if budget_s is None:
                engine.expand_level(store, 12, cfg.operators, config=cfg, stats=stats)  # also allocates the buffers of level 12
                full = (store.level(12).n, time.perf_counter() - t0)
            else:
                with pytest.raises(engine._BudgetExceeded, match="time budget exhausted"):
                    engine.expand_level(store, 12, cfg.operators, config=cfg, stats=stats, deadline=t0 + budget_s)
                elapsed = time.perf_counter() - t0
                assert 0 < store.level(12).n < full[0], "the partial level was not kept"
                assert elapsed < 0.020, f"the level ran {1e3 * elapsed:.1f} ms past a {1e3 * budget_s:.0f} ms deadline"
                rows, _ = store.level_device(12)  # what was stored is still a set of distinct rows
                h1, h2 = _row_hashes(rows)
                order = __import__("torch").argsort(h1)
                assert not bool(((h1[order][1:] == h1[order][:-1]) & (h2[order][1:] == h2[order][:-1])).any())
        finally:
            store.close()
