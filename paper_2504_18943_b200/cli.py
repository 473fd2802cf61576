"""Command line of the B200 engine: the reference's ``ltlsynth synth | check`` (reference
``pkg/src/ltlsynth/cli.py``) with the same flags, report keys, text layout and exit codes, so
that scripts written against the reference run unchanged:

    python -m paper_2504_18943_b200 synth --input spec.trc [--mode enumerate|dnc] [--format json] ...
    python -m paper_2504_18943_b200 check --input spec.trc --formula '!(b U a)'

synth exit codes: 0 separator found, 2 budget exhausted, 1 input error (``cli.py:1-5``).
check exit codes: 0 formula separates, 2 it does not, 1 input error.
Extensions (absent from the reference, default to its behaviour): ``--device``, ``--gpus``, and the ``regex``
command of the regex front-end (no reference counterpart):

    python -m paper_2504_18943_b200 regex --input examples.txt [--cost 1,1,1,1,1] [--max-cost 12] [--format json]

where the file holds one example string per line, the positives, a line ``---``, the negatives (a line ``<eps>`` is
the empty string).  Exit codes as for synth.
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
    regex = commands.add_parser("regex", help="synthesize a minimum-cost regular expression (extension)")
    regex.add_argument("--input", required=True, help="example strings: positives, a line '---', negatives")
    regex.add_argument("--cost", default="1,1,1,1,1", help="cost of a literal, ?, *, concatenation, union")
    regex.add_argument("--max-cost", type=int, default=12)
    regex.add_argument("--time-budget-s", type=float, default=300.0)
    regex.add_argument("--format", choices=("text", "json"), default="text")
    regex.add_argument("--device", type=int, default=0)
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


def parse_examples(text: str):
    """Example strings of the regex command: one per line, positives / ``---`` / negatives; ``<eps>`` = the empty string."""
    sides, current = [[], []], 0
    for number, line in enumerate(text.splitlines(), 1):
        line = line.rstrip("\r\n")
        if line.strip() == "---":
            if current == 1:
                raise ValueError(f"line {number}: a second '---'")
            current = 1
        elif line.strip() == "<eps>":
            sides[current].append("")
        elif line:
            sides[current].append(line)
    if current == 0:
        raise ValueError("no '---' line between the positive and the negative examples")
    return tuple(sides[0]), tuple(sides[1])


def run_regex(args) -> int:
    from .regex import CostFunction, RegexConfig, RegexSpecification, synthesize_regex  # (needs the CUDA engine)
    from .traces import InfeasibleSpecificationError

    try:
        with open(args.input, "r", encoding="utf-8") as handle:
            positives, negatives = parse_examples(handle.read())
        parts = [int(x) for x in args.cost.split(",")]
        if len(parts) != 5:
            raise ValueError("--cost takes five integers: literal, ?, *, concatenation, union")
        spec = RegexSpecification(positives, negatives)
        config = RegexConfig(cost=CostFunction(*parts), max_cost=args.max_cost, time_budget_s=args.time_budget_s, device=args.device)
    except (OSError, ValueError, InfeasibleSpecificationError) as problem:
        print(f"error: {problem}", file=sys.stderr)
        return 1
    result = synthesize_regex(spec, config)
    report = {"regex": result.pattern, "cost": result.cost, "constructed": result.stats.constructed, "unique": result.stats.unique,
              "elapsed_ms": round(1000.0 * result.stats.elapsed_s, 3), "cost_function": parts,
              "budgets": {"max_cost": args.max_cost, "time_budget_s": args.time_budget_s}, "outcome": result.outcome}
    if args.format == "json":
        print(json.dumps(report))
    else:
        print(f"regex: {result.pattern}\ncost: {result.cost}" if result.pattern is not None
              else f"no expression found ({result.failure or 'budget exhausted'})")
        print(f"constructed: {report['constructed']}  unique: {report['unique']}  elapsed_ms: {report['elapsed_ms']}")
    return 0 if result.outcome == OUTCOME_FOUND else 2


def main(argv=None) -> int:
    args = make_parser().parse_args(argv)
    return {"synth": run_synth, "check": run_check, "regex": run_regex}[args.command](args)


def entry_point() -> None:
    sys.exit(main())


if __name__ == "__main__":
    entry_point()
