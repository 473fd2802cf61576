"""Host-side logic of the callers (no GPU): the split tree of the divide-and-conquer driver and
the CLI paths that end before any device work (reference tests/test_dnc.py:19-37,
tests/test_cli.py:68-83,117-121)."""

import json
import pathlib

from paper_2504_18943_b200 import cli, dnc, parse_specification, spec_from_steps, workloads
from paper_2504_18943_b200.engine import EngineConfig

GOLD = pathlib.Path(__file__).resolve().parent / "golden_callers"


def _sizes(plan):
    return tuple(len(s) for s in plan.p_split), tuple(len(s) for s in plan.n_split)


def test_split_halves_in_canonical_order():
    spec = workloads.spec2()
    plan = dnc.split(spec)
    assert _sizes(plan) == ((4, 3), (4, 3))
    assert plan.p_split[0] + plan.p_split[1] == tuple(spec.positives)
    assert plan.n_split[0] + plan.n_split[1] == tuple(spec.negatives)
    single = spec_from_steps([["a"]], [["b"], ["ab"], [""]], "ab")
    assert _sizes(dnc.split(single)) == ((1, 0), (2, 1))


def test_unfold_lists_leaves_in_the_reference_order():
    leaves = []
    dnc._unfold(workloads.spec2(), EngineConfig(dnc_threshold=8), "root", leaves)
    assert [leaf.label for leaf in leaves] == ["root.P1N1", "root.P1N2", "root.P2N1", "root.P2N2"]
    assert [leaf.spec.trace_count for leaf in leaves] == [8, 7, 7, 6]
    leaves = []
    dnc._unfold(workloads.spec1(), EngineConfig(dnc_threshold=0), "root", leaves)  # clamped to 2
    assert all(leaf.spec.trace_count <= 2 for leaf in leaves) and len(leaves) == 9
    # an empty positive half contributes no disjunct (reference tests/test_dnc.py:63-70)
    lopsided = spec_from_steps([["a", "a"]], [["b"], ["ab"], ["a"], [""]], "ab")
    leaves = []
    dnc._unfold(lopsided, EngineConfig(dnc_threshold=2), "root", leaves)
    assert all(".P2" not in leaf.label.split(".")[1] for leaf in leaves)


def test_cli_input_errors_need_no_device(tmp_path, capsys):
    cases = json.loads((GOLD / "cli_cases.json").read_text())
    for case in cases["cases"]:
        if case["name"] not in ("synth_infeasible", "synth_missing", "synth_unknown_ops", "check_parse_error"):
            continue
        for name in case["files"]:
            (tmp_path / name).write_text(cases["files"][name])
        code = cli.main([a.replace("{dir}", str(tmp_path)) for a in case["argv"]])
        out, err = capsys.readouterr()
        assert code == case["code"] == 1
        assert err == case["stderr"].replace("{dir}", str(tmp_path))
        assert out == ""


def test_cli_check_uses_the_naive_semantics(tmp_path, capsys):
    cases = json.loads((GOLD / "cli_cases.json").read_text())
    (tmp_path / "spec1.trc").write_text(cases["files"]["spec1.trc"])
    for name in ("check_ok", "check_violation"):
        case = next(c for c in cases["cases"] if c["name"] == name)
        code = cli.main([a.replace("{dir}", str(tmp_path)) for a in case["argv"]])
        out, _ = capsys.readouterr()
        assert (code, out) == (case["code"], case["stdout"])
