"""Host-side data model: .trc format, layout, formula printer/parser, naive semantics.
Mirrors what the reference pins in tests/test_traces.py, tests/test_formulas.py and
tests/test_oracle.py (same observable behaviour, independent implementation)."""

import random

import numpy as np
import pytest

from paper_2504_18943_b200 import (
    Alphabet,
    And,
    Atom,
    Future,
    InfeasibleSpecificationError,
    Layout,
    Next,
    Not,
    Or,
    SpecError,
    SpecFormatError,
    Until,
    atom_bitvectors,
    cost,
    parse_formula,
    parse_specification,
    sat,
    semantics,
    serialize_specification,
    smallest_lane_dtype,
    spec_from_steps,
    to_text,
    word_trace,
    workloads,
)
from paper_2504_18943_b200.formulas import FormulaSyntaxError


def test_trc_round_trip_and_canonical_order():
    spec = parse_specification(workloads.SPEC1_TRC)
    assert spec.alphabet.names == ("a", "b", "c")
    assert (len(spec.positives), len(spec.negatives), spec.trace_count, spec.max_length) == (3, 3, 6, 3)
    assert parse_specification(serialize_specification(spec)) == spec
    assert spec.traces == spec.positives + spec.negatives


def test_trc_without_header_gets_default_names():
    spec = parse_specification("1,0\n---\n0,1;1,1\n")
    assert spec.alphabet.names == ("p0", "p1") and spec.negatives[0].length == 2


@pytest.mark.parametrize("text,line,column,fragment", [
    ("#atoms: a b\n1,0\n1\n", 3, 1, "expected 2"),
    ("#atoms: a b\n1,x\n", 2, 3, "expected 0 or 1"),
    ("1,0;;0,1\n", 1, 5, "empty timestep"),
    ("1,0\n---\n---\n", 3, None, "more than one"),
    ("1,0\n#atoms: a b\n", 2, None, "must precede"),
    ("#atoms: a a\n", 1, None, "duplicate"),
    ("# nothing\n", None, None, "no traces"),
])
def test_trc_errors_carry_position(text, line, column, fragment):
    with pytest.raises(SpecFormatError) as err:
        parse_specification(text)
    assert fragment in str(err.value)
    assert (err.value.line, err.value.column) == (line, column)


def test_infeasible_file_is_rejected():
    with pytest.raises(InfeasibleSpecificationError):
        parse_specification("1,0\n---\n1,0\n")


def test_model_validation():
    with pytest.raises(SpecError):
        Alphabet(())
    with pytest.raises(SpecError):
        word_trace("", Alphabet.of("ab"))
    with pytest.raises(SpecError):
        word_trace("a" * 65, Alphabet.of("ab"))
    with pytest.raises(SpecError):
        spec_from_steps([], [], "ab")


def test_lane_dtype_table_and_layout():
    assert [smallest_lane_dtype(n).itemsize for n in (1, 8, 9, 16, 17, 32, 33, 64)] == [1, 1, 2, 2, 4, 4, 8, 8]
    with pytest.raises(SpecError):
        smallest_lane_dtype(65)
    spec = workloads.spec1()
    layout = Layout.from_specification(spec, np.uint8)
    assert layout.lengths == (1, 2, 1, 2, 3, 3) and layout.width == 8
    assert layout.masks.tolist() == [1, 3, 1, 3, 7, 7] and layout.target.tolist() == [1, 1, 1, 0, 0, 0]
    atoms = atom_bitvectors(spec, np.uint8)
    assert atoms.shape == (3, 6)
    assert atoms[0].tolist() == [0, 2, 0, 2, 3, 2]  # 'a' per trace, bit j = position j
    assert not (atoms & ~layout.masks).any()


def test_printer_uses_minimal_parentheses():
    a, b, c = Atom(0), Atom(1), Atom(2)
    abc = Alphabet.of("abc")
    cases = {
        Not(Until(b, a)): "!(b U a)",
        Until(a, Until(b, c)): "a U b U c",
        Until(Until(a, b), c): "(a U b) U c",
        And(And(a, b), c): "a & b & c",
        And(a, And(b, c)): "a & (b & c)",
        Or(And(a, b), c): "a & b | c",
        And(Or(a, b), c): "(a | b) & c",
        Next(Future(Not(a))): "X F !a",
        Until(Not(And(b, Next(b))), a): "!(b & X b) U a",
        Future(Until(a, b)): "F (a U b)",
    }
    for tree, text in cases.items():
        assert to_text(tree, abc) == text
        assert parse_formula(text, abc) == tree


def test_print_parse_round_trip_on_random_trees():
    rng = random.Random(11)
    abc = Alphabet.of("abc")

    def tree(size):
        if size == 1:
            return Atom(rng.randrange(3))
        if size == 2 or rng.random() < 0.4:
            return rng.choice((Not, Next, Future))(tree(size - 1))
        left = rng.randint(1, size - 2)
        return rng.choice((And, Or, Until))(tree(left), tree(size - 1 - left))

    for _ in range(300):
        f = tree(rng.randint(1, 9))
        assert parse_formula(to_text(f, abc), abc) == f
        assert cost(f) == to_text(f, abc).count("!") + sum(to_text(f, abc).count(s) for s in ("X ", "F ", " U ", " & ", " | ")) + \
            sum(1 for tok in to_text(f, abc).replace("(", " ").replace(")", " ").replace("!", " ").split() if tok in "abc")


@pytest.mark.parametrize("text,position", [("a &", 3), ("(a", 2), ("a b", 2), ("d", 0), ("a $ b", 2), ("", 0)])
def test_parse_errors_report_offsets(text, position):
    with pytest.raises(FormulaSyntaxError) as err:
        parse_formula(text, Alphabet.of("abc"))
    assert err.value.position == position


def test_naive_semantics_fixtures():
    """reference tests/test_oracle.py:14-44 and test_acceptance.py:49-62 (the squeegee judgements)."""
    alphabet = Alphabet.of("egqsu")
    tr = word_trace("squeegee", alphabet)
    judge = lambda text, pos: sat(tr, pos, parse_formula(text, alphabet))
    assert judge("F g", 0) and not judge("e", 2) and judge("F e", 2) and judge("(F g) U !F g", 0)
    assert not judge("X e", 7)  # nothing holds beyond the last position
    with pytest.raises(ValueError):
        sat(tr, 8, Atom(0))
    spec = workloads.spec1()
    assert semantics.separates_by_sat(spec, parse_formula("!(b U a)", spec.alphabet))
    assert not semantics.separates_by_sat(spec, parse_formula("c", spec.alphabet))


def test_fast_witness_check_agrees_with_the_quantifier_semantics():
    """semantics._truth_table_fast (expansion laws, one backward pass per node) and semantics._truth_mask (the same on
    integer bit masks, doubling shifts) == semantics._truth_table (quantifiers of F and U written out) on random formulas
    over random traces."""
    import random

    from paper_2504_18943_b200.formulas import And, Future, Globally, Next, Not, Or, Until
    from paper_2504_18943_b200.traces import Trace

    rng = random.Random(0xF457)

    def formula(depth):
        if depth == 0 or rng.random() < 0.2:
            return Atom(rng.randrange(3))
        kind = rng.choice(("not", "next", "future", "globally", "and", "or", "until"))
        if kind == "not":
            return Not(formula(depth - 1))
        if kind == "next":
            return Next(formula(depth - 1))
        if kind == "future":
            return Future(formula(depth - 1))
        if kind == "globally":
            return Globally(formula(depth - 1))
        node = {"and": And, "or": Or, "until": Until}[kind]
        return node(formula(depth - 1), formula(depth - 1))

    for _ in range(400):
        length = rng.randint(1, 19)
        tr = Trace(tuple(frozenset(p for p in range(3) if rng.random() < 0.5) for _ in range(length)))
        f = formula(rng.randint(1, 5))
        want = semantics._truth_table(tr, f)
        assert semantics._truth_table_fast(tr, f) == want, (tr, f)
        mask = semantics._truth_mask(tr, f, {})  # the integer tables separates_by_sat evaluates
        assert [bool(mask >> i & 1) for i in range(length)] == want and mask >> length == 0, (tr, f)


def test_bench_gpus_flag_starts_that_many_ranks():
    """`bench.py --gpus 2` outside torchrun must START two processes (it silently measured one).  No GPU
    here, so the launch path is exercised with --selftest-cpu: gloo + the numpy shard engine run the sharded protocol."""
    import json
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parent.parent
    proc = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--selftest-cpu"], capture_output=True,
                          text=True, timeout=300)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-2000:]
    line = json.loads([ln for ln in proc.stdout.splitlines() if ln.startswith("{")][-1])
    assert (line["n_gpus"], line["processes"], line["witness"], line["unique_per_step"]) == (2, 2, "!(b U a)", 33)


def test_bench_reference_arm_runs_the_cpu_enumerator_on_the_gpu_arms_config():
    import json
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parent.parent
    proc = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--workload", "spec1", "--steps", "1",
                           "--warmup", "0"], capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stderr[-2000:]
    line = json.loads(proc.stdout.splitlines()[-1])
    assert line["impl"] == "reference" and line["config"]["max_cost"] == 10 and line["config"]["workload"] == "spec1"
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert "233 unique" in line["cpu_baseline"]["sample"]
