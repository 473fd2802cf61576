"""Command line of the B200 engine: the reference's ``ltlsynth synth | check`` (reference
``pkg/src/ltlsynth/cli.py``) with the same flags, report keys, text layout and exit codes, so
that scripts written against the reference run unchanged:

    python -m paper_2504_18943_b200 synth --input spec.trc [--mode enumerate|dnc] [--format json] ...
    python -m paper_2504_18943_b200 check --input spec.trc --formula '!(b U a)'

synth exit codes: 0 separator found, 2 budget exhausted, 1 input error (``cli.py:1-5``).
check exit codes: 0 formula separates, 2 it does not, 1 input error.
Extensions (absent from the reference, default to its behaviour): ``--device``, ``--gpus``.
``--threads`` is accepted and ignored: the device schedules its own parallelism, and the
reference guarantees that the thread count changes nothing (its tests/test_cli.py:130-140).
"""

from __future__ import annotations

import argparse
import json
import sys

from . import semantics
from .dnc import synthesize_dnc
from .engine import OUTCOME_FOUND, EngineConfig, normalize_operators, synthesize
from .formulas import DEFAULT_OPERATORS, FormulaSyntaxError, parse_formula, to_text
from .traces import SpecError, parse_specification

SYNTH_FLAGS = (  # (flag, keyword arguments): the reference's synth options, cli.py:24-38
    ("--input", dict(required=True, help="trace specification file")),
    ("--mode", dict(choices=("enumerate", "dnc"), default="enumerate")),
    ("--ops", dict(default=",".join(DEFAULT_OPERATORS), help="comma list from not,and,or,next,future,until")),
    ("--max-cost", dict(type=int, default=20)),
    ("--time-budget-s", dict(type=float, default=300.0)),
    ("--memory-budget-mb", dict(type=int, default=8192)),
    ("--batch-size", dict(type=int, default=1 << 16)),
    ("--threads", dict(type=int, default=None, help="accepted for compatibility, ignored")),
    ("--dnc-threshold", dict(type=int, default=8, help="direct-solve size bound in dnc mode")),
    ("--format", dict(choices=("text", "json"), default="text")),
    ("--device", dict(type=int, default=0, help="CUDA device ordinal (extension)")),
    ("--gpus", dict(type=int, default=1, help="dnc mode: spread the leaves over this many devices (extension)")),
)


def make_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="ltlsynth-b200", description=__doc__,
                                     formatter_class=argparse.RawDescriptionHelpFormatter)
    commands = parser.add_subparsers(dest="command", required=True)
    synth = commands.add_parser("synth", help="synthesize a minimum-cost separating formula")
    for flag, kwargs in SYNTH_FLAGS:
        synth.add_argument(flag, **kwargs)
    check = commands.add_parser("check", help="check a formula against a specification")
    check.add_argument("--input", required=True, help="trace specification file")
    check.add_argument("--formula", required=True, help="formula text, e.g. '!(b U a)'")
    return parser


def _read_spec(path: str):
    with open(path, "r", encoding="utf-8") as handle:
        return parse_specification(handle.read())


def run_synth(args) -> int:
    try:
        spec = _read_spec(args.input)
        config = EngineConfig(
            operators=normalize_operators(name.strip() for name in args.ops.split(",")),
            max_cost=args.max_cost, time_budget_s=args.time_budget_s, memory_budget_mb=args.memory_budget_mb,
            batch_size=args.batch_size, threads=args.threads, dnc_threshold=args.dnc_threshold, device=args.device,
        )
    except (OSError, SpecError, ValueError) as problem:
        print(f"error: {problem}", file=sys.stderr)
        return 1
    if args.mode == "dnc":
        result = synthesize_dnc(spec, config, devices=range(args.device, args.device + max(1, args.gpus)))
    else:
        result = synthesize(spec, config)
    found = result.formula is not None
    report = {  # key set and order of the reference's report, cli.py:51-68
        "formula": to_text(result.formula, spec.alphabet) if found else None,
        "cost": result.cost,
        "minimal": result.minimal,
        "constructed": result.stats.constructed,
        "unique": result.stats.unique,
        "elapsed_ms": round(1000.0 * result.stats.elapsed_s, 3),
        "mode": args.mode,
        "operator_set": list(config.operators),
        "budgets": {"max_cost": args.max_cost, "time_budget_s": args.time_budget_s,
                    "memory_budget_mb": args.memory_budget_mb},
        "outcome": result.outcome,
    }
    if args.format == "json":
        print(json.dumps(report))
    else:
        if found:
            print(f"formula: {report['formula']}\ncost: {result.cost}\nminimal: {'yes' if result.minimal else 'no'}")
        else:
            print(f"no formula found ({result.failure or 'budget exhausted'})")
        print(f"constructed: {report['constructed']}  unique: {report['unique']}  elapsed_ms: {report['elapsed_ms']}")
    return 0 if result.outcome == OUTCOME_FOUND else 2


def run_check(args) -> int:
    try:
        spec = _read_spec(args.input)
        formula = parse_formula(args.formula, spec.alphabet)
    except (OSError, SpecError, FormulaSyntaxError) as problem:
        print(f"error: {problem}", file=sys.stderr)
        return 1
    positives = len(spec.positives)
    all_good = True
    for index, trace in enumerate(spec.traces):
        holds, wanted = semantics.sat(trace, 0, formula), index < positives
        all_good = all_good and holds == wanted
        print(f"trace {index} ({'positive' if wanted else 'negative'}): {'sat' if holds else 'unsat'}  "
              f"{'ok' if holds == wanted else 'VIOLATION'}")
    print(f"separates: {'yes' if all_good else 'no'}")
    return 0 if all_good else 2


def main(argv=None) -> int:
    args = make_parser().parse_args(argv)
    return run_synth(args) if args.command == "synth" else run_check(args)


def entry_point() -> None:
    sys.exit(main())


if __name__ == "__main__":
    entry_point()
