#!/usr/bin/env python3
"""Where do a level's duplicates come from?  (CPU oracle, analysis only.)

For each cost level prints the share of candidates that are new, that duplicate a CM built
earlier in the same level, and that duplicate a CM stored d levels below.  This decides how
much of the dedup probing can be served by an L2-resident table of the low levels.
"""
import argparse
import ctypes
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import oracle
from paper_2504_18943_b200 import formulas as F
from paper_2504_18943_b200 import workloads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--max-cost", type=int, default=14)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    oracle.build()
    L = oracle.lib()
    L.orc_dup_hist.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
    L.orc_dup_hist.restype = None
    spec = workloads.named_workload(args.workload, args.seed)
    store = oracle.OracleStore(spec)
    hist = (ctypes.c_int64 * 64)()
    for cost in range(1, args.max_cost + 1):
        store.expand_level(cost, F.DEFAULT_OPERATORS, True)
        L.orc_dup_hist(store._h, hist)
        h = list(hist)
        total = sum(h) or 1
        new, same = h[0], h[cost]
        below = [h[c] for c in range(cost - 1, 0, -1)]  # d = 1, 2, ...
        cum = 0
        parts = []
        for d, v in enumerate(below, 1):
            cum += v
            if d <= 6:
                parts.append(f"d{d} {100 * v / total:4.1f}%")
        print(f"cost {cost:2d}: cand {total:10d}  new {100 * new / total:5.1f}%  same-level {100 * same / total:5.1f}%  "
              f"older {100 * sum(below) / total:5.1f}%  [{'  '.join(parts)}]  stored {store.total}", flush=True)


if __name__ == "__main__":
    main()
