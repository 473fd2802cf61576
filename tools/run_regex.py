"""Runs a regex workload (paper_2504_18943_b200.workloads.regex_workload: re-c0, re-email, re-c2, re-c3) on the GPU:
exhaustive levels up to --max-cost; per level the candidates constructed, the new CSs and the wall time of the call.

    python tools/run_regex.py --workload re-email --max-cost 12
"""
import argparse
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2504_18943_b200 import regex as rx  # noqa: E402
from paper_2504_18943_b200.workloads import regex_workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="re-email")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-cost", type=int, default=9)
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    spec = regex_workload(args.workload, args.seed)
    for rep in range(args.repeat):
        store = rx.RegexStore(spec)
        rows = []
        t_all = time.perf_counter()
        for c in range(1, args.max_cost + 1):
            t0 = time.perf_counter()
            status, n_new, sep, constructed = store.expand(c, exhaustive=True)
            rows.append({"cost": c, "status": status, "constructed": constructed, "new": n_new, "ms": round(1e3 * (time.perf_counter() - t0), 3)})
            if status != 0:
                break
        total_ms = 1e3 * (time.perf_counter() - t_all)
        st = store.device_stats()
        store.close()
        print(json.dumps({"workload": args.workload, "run": rep, "n_bits": store.ix.n_bits, "guide_entries": len(store.ix.splits),
                          "total_ms": round(total_ms, 2), "enumerate_ms": round(st["enumerate_ms"], 3),
                          "finalize_ms": round(st["finalize_ms"], 3), "device_bytes": st["device_bytes"], "levels": rows}))


if __name__ == "__main__":
    main()
