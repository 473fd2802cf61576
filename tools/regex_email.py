"""Times the regex front-end on the paper's e-mail example (528 infixes, 4103 guide entries): exhaustive
levels up to --max-cost, per level the candidates constructed, the new CSs and the wall time of the expand call.

    python tools/regex_email.py --max-cost 10
"""
import argparse
import json
import sys
import time
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2504_18943_b200 import regex as rx  # noqa: E402

EMAIL_P = ("geon@ex.io", "test@gmail.com", "mail@test.org", "mail@testing.com")
EMAIL_N = ("hello@", "@test", "email@gmail", "t@test@gmail.com", "mail with@space.com")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-cost", type=int, default=9)
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    spec = rx.RegexSpecification(EMAIL_P, EMAIL_N)
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
        print(json.dumps({"run": rep, "n_bits": store.ix.n_bits, "guide_entries": len(store.ix.splits), "total_ms": round(total_ms, 2),
                          "enumerate_ms": round(st["enumerate_ms"], 3), "finalize_ms": round(st["finalize_ms"], 3), "levels": rows}))


if __name__ == "__main__":
    main()
