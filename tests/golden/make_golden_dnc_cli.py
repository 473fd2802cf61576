#!/usr/bin/env python3
"""Golden outputs of the UNMODIFIED reference's divide-and-conquer driver and CLI.

Run in the build container (the reference does not travel to the GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_dnc_cli.py

Writes tests/golden_callers/dnc_cases.json and tests/golden_callers/cli_cases.json.  Every case
carries its input (.trc text) so the GPU tests need neither the reference nor a shared generator.
"""
import contextlib
import io
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))

import ltlsynth  # the reference
from ltlsynth.cli import main as ref_cli_main
from ltlsynth.dnc import synthesize_dnc as ref_dnc
from ltlsynth.engine import EngineConfig as RefConfig
from ltlsynth.formulas import to_text as ref_to_text
from ltlsynth.traces import parse_specification as ref_parse

from paper_2504_18943_b200 import workloads
from paper_2504_18943_b200.traces import serialize_specification

OUT = ROOT / "tests" / "golden_callers"
OUT.mkdir(exist_ok=True)
DATA = pathlib.Path("/root/reference/pkg/tests/data")


def dnc_case(name, trc, **cfg):
    spec = ref_parse(trc)
    res = ref_dnc(spec, RefConfig(threads=1, **cfg))
    return dict(name=name, trc=trc, config=cfg,
                formula=ref_to_text(res.formula, spec.alphabet) if res.formula is not None else None,
                cost=res.cost, minimal=res.minimal, outcome=res.outcome, failure=res.failure,
                constructed=res.stats.constructed, unique=res.stats.unique, max_cost_reached=res.stats.max_cost_reached)


def cli_case(name, files, argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = ref_cli_main(argv)
    return dict(name=name, files=files, argv=argv, code=code, stdout=out.getvalue(), stderr=err.getvalue())


def main():
    spec1 = (DATA / "spec1.trc").read_text()
    spec2 = (DATA / "spec2.trc").read_text()
    cases = [
        dnc_case("spec1_below_threshold", spec1),
        dnc_case("spec1_forced_split", spec1, dnc_threshold=2),
        dnc_case("spec1_threshold3", spec1, dnc_threshold=3),
        dnc_case("spec2_threshold8", spec2),
        dnc_case("spec2_threshold4", spec2, dnc_threshold=4),
        dnc_case("spec2_leaf_failure", spec2, dnc_threshold=8, max_cost=5),
    ]
    for seed, (atoms, pos, neg, length, thr) in enumerate([(2, 6, 6, 5, 8), (2, 8, 8, 6, 8), (3, 10, 10, 5, 8), (2, 9, 7, 6, 4),
                                                            (3, 7, 12, 4, 6), (2, 16, 16, 5, 8), (4, 10, 10, 6, 8), (2, 5, 9, 7, 3)]):
        spec = workloads.synthetic_spec(seed + 100, atoms, pos, neg, length, False)
        cases.append(dnc_case(f"random_s{seed + 100}_a{atoms}_p{pos}_n{neg}_t{thr}", serialize_specification(spec), dnc_threshold=thr, max_cost=12))
    (OUT / "dnc_cases.json").write_text(json.dumps(cases, indent=1))
    print("dnc:", [(c["name"], c["outcome"], c["cost"]) for c in cases])

    tmp = pathlib.Path("/tmp/golden_cli")
    tmp.mkdir(exist_ok=True)
    files = {"spec1.trc": spec1, "spec2.trc": spec2, "bad.trc": "1;0\n---\n1;0\n"}
    for fname, text in files.items():
        (tmp / fname).write_text(text)
    p = lambda f: str(tmp / f)
    cli = [
        cli_case("synth_text", ["spec1.trc"], ["synth", "--input", p("spec1.trc"), "--threads", "1"]),
        cli_case("synth_json", ["spec1.trc"], ["synth", "--input", p("spec1.trc"), "--format", "json", "--threads", "1"]),
        cli_case("synth_exhausted", ["spec1.trc"], ["synth", "--input", p("spec1.trc"), "--max-cost", "3", "--format", "json"]),
        cli_case("synth_exhausted_text", ["spec1.trc"], ["synth", "--input", p("spec1.trc"), "--max-cost", "3"]),
        cli_case("synth_or_ops", ["spec1.trc"], ["synth", "--input", p("spec1.trc"), "--ops", "not,and,or,until", "--format", "json"]),
        cli_case("synth_spec2_cost9", ["spec2.trc"], ["synth", "--input", p("spec2.trc"), "--max-cost", "9", "--format", "json"]),
        cli_case("synth_infeasible", ["bad.trc"], ["synth", "--input", p("bad.trc")]),
        cli_case("synth_missing", [], ["synth", "--input", p("nope.trc")]),
        cli_case("synth_unknown_ops", ["spec1.trc"], ["synth", "--input", p("spec1.trc"), "--ops", "not,xor"]),
        cli_case("synth_dnc", ["spec1.trc"], ["synth", "--input", p("spec1.trc"), "--mode", "dnc", "--dnc-threshold", "2", "--format", "json"]),
        cli_case("synth_dnc_spec2", ["spec2.trc"], ["synth", "--input", p("spec2.trc"), "--mode", "dnc", "--format", "json"]),
        cli_case("check_ok", ["spec1.trc"], ["check", "--input", p("spec1.trc"), "--formula", "!(b U a)"]),
        cli_case("check_violation", ["spec1.trc"], ["check", "--input", p("spec1.trc"), "--formula", "a"]),
        cli_case("check_parse_error", ["spec1.trc"], ["check", "--input", p("spec1.trc"), "--formula", "(b U"]),
    ]
    for c in cli:  # paths are re-rooted by the tests
        c["argv"] = [a.replace(str(tmp) + "/", "{dir}/") for a in c["argv"]]
        c["stderr"] = c["stderr"].replace(str(tmp) + "/", "{dir}/")
    (OUT / "cli_cases.json").write_text(json.dumps(dict(files=files, cases=cli), indent=1))
    print("cli:", [(c["name"], c["code"]) for c in cli])


if __name__ == "__main__":
    main()
