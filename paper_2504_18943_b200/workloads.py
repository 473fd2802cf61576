"""Named example sets: the paper's two worked LTL examples and the seeded
synthetic specifications the benchmark and the parity tests run on.

SURVEY.md section 8(d) maps BASELINE.json's five configurations onto concrete
inputs; ``named_workload`` is that mapping.  The synthetic generator draws
traces the way the reference's test generators do
(``pkg/tests/strategies.py:53-60`` and ``:81-100``: every atom holds at every
step with probability 1/2, and the whole draw is repeated when a negative
trace equals a positive one), from ``random.Random(seed)``, so the same seed
gives the same specification on every machine.
"""

from __future__ import annotations

import random

from .traces import Alphabet, Specification, Trace, spec_from_steps

# The 3+3-trace example over {a,b,c}; minimal separator has 4 nodes
# (reference pkg/tests/data/spec1.trc, PAPER.md worked example 1).
SPEC1_TRC = """#atoms: a b c
0,0,1
0,0,1;1,0,0
0,1,0
---
0,1,0;1,0,0
1,0,0;1,0,0;0,0,1
0,1,0;1,0,0;0,0,1
"""

# The 7+7-trace example over {a,b}, all traces of length 6; minimal separator
# has 16 nodes (reference pkg/tests/data/spec2.trc).
_SPEC2_POS = ["ab ab a b a ab", "- ab a b b -", "ab a - b a ab", "b b ab b a ab",
              "ab a ab a - a", "a ab ab b a ab", "b - a - a a"]
_SPEC2_NEG = ["b ab ab b a ab", "ab ab ab a - a", "- ab ab b a a", "b b a - a ab",
              "ab ab a b a a", "ab a b b a a", "b a ab b a a"]


def spec1() -> Specification:
    from .traces import parse_specification

    return parse_specification(SPEC1_TRC)


def spec2() -> Specification:
    unpack = lambda rows: [[("" if s == "-" else s) for s in row.split()] for row in rows]
    return spec_from_steps(unpack(_SPEC2_POS), unpack(_SPEC2_NEG), "ab")


def _draw_trace(rng: random.Random, n_atoms: int, length: int, fixed: bool) -> Trace:
    steps_n = length if fixed else rng.randint(1, length)
    return Trace(
        tuple(frozenset(p for p in range(n_atoms) if rng.random() < 0.5) for _ in range(steps_n))
    )


def synthetic_spec(seed: int, n_atoms: int, n_pos: int, n_neg: int, length: int,
                   fixed_length: bool) -> Specification:
    """Seeded random specification with exactly n_pos / n_neg traces."""
    rng = random.Random(seed)
    alphabet = Alphabet.default(n_atoms)
    while True:
        pos = [_draw_trace(rng, n_atoms, length, fixed_length) for _ in range(n_pos)]
        neg = [_draw_trace(rng, n_atoms, length, fixed_length) for _ in range(n_neg)]
        taken = {t.steps for t in pos}
        if not any(t.steps in taken for t in neg):
            return Specification(alphabet, tuple(pos), tuple(neg))


# name -> (n_atoms, n_pos, n_neg, length, fixed_length); CM bytes in the comment
_SYNTHETIC = {
    "c1": (2, 4, 4, 5, False),  # 8 lanes x 8 bit = 8 B
    "c3": (2, 8, 8, 8, True),  # 16 x 8 bit = 16 B (one uint4)
    "c3wide": (2, 20, 20, 10, False),  # 40 x 16 bit = 80 B
    "c4-512": (3, 16, 16, 16, False),  # 32 x 16 bit = 64 B
    "c4-1024": (3, 32, 32, 16, False),  # 64 x 16 bit = 128 B
    "c4xl": (3, 64, 64, 16, False),  # 128 x 16 bit = 256 B
    "c5": (4, 32, 32, 16, True),  # 64 x 16 bit = 128 B
    "w32": (2, 3, 3, 20, False),  # 32-bit lanes
    "w64": (2, 2, 3, 40, False),  # 64-bit lanes
    "w32n": (2, 2, 2, 20, False),  # 4 x 32 bit = 16 B (one uint4)
    "w64n": (3, 1, 1, 40, False),  # 2 x 64 bit = 16 B (one uint4)
}


def named_workload(name: str, seed: int = 0) -> Specification:
    """Specification for a BASELINE.json configuration name."""
    key = name.lower()
    if key in ("spec1", "c2-spec1"):
        return spec1()
    if key in ("spec2", "c2", "c2-spec2"):
        return spec2()
    if key in _SYNTHETIC:
        return synthetic_spec(seed, *_SYNTHETIC[key])
    raise KeyError(f"unknown workload {name!r}; known: spec1, spec2, {', '.join(_SYNTHETIC)}")


def workload_names() -> tuple[str, ...]:
    return ("spec1", "spec2") + tuple(_SYNTHETIC)


# ---- regular-expression example sets (regex front-end; BASELINE.json configs[0]-[3] as literally worded) ----------

EMAIL_POSITIVES = ("geon@ex.io", "test@gmail.com", "mail@test.org", "mail@testing.com")  # reference PAPER.md:83-94
EMAIL_NEGATIVES = ("hello@", "@test", "email@gmail", "t@test@gmail.com", "mail with@space.com")

# name -> (letters, strings per side, maximum length)
_REGEX_SYNTHETIC = {
    "re-c0": ("01", 4, 5),      # configs[0]: a few dozen infixes, one uint4 per characteristic sequence
    "re-c2": ("01", 20, 10),    # configs[2]: ~200 infixes
    "re-c3": ("abc", 64, 16),   # configs[3]: ~2700 infixes (22 uint4 per sequence)
}


def regex_workload(name: str, seed: int = 0):
    """Example strings of a regex workload as a ``RegexSpecification``: distinct random strings of length
    1..maximum over the letters, drawn from ``random.Random(seed)``, the first half positive."""
    from .regex import RegexSpecification

    key = name.lower()
    if key in ("re-email", "re-c1"):
        return RegexSpecification(EMAIL_POSITIVES, EMAIL_NEGATIVES)
    if key not in _REGEX_SYNTHETIC:
        raise KeyError(f"unknown regex workload {name!r}; known: re-email, {', '.join(_REGEX_SYNTHETIC)}")
    letters, per_side, longest = _REGEX_SYNTHETIC[key]
    rng = random.Random(seed)
    words: set[str] = set()
    while len(words) < 2 * per_side:
        words.add("".join(rng.choice(letters) for _ in range(rng.randint(1, longest))))
    drawn = sorted(words)
    rng.shuffle(drawn)
    return RegexSpecification(tuple(drawn[:per_side]), tuple(drawn[per_side:]))
