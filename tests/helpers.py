"""Shared helpers for the parity tests: golden loading and level digests."""

from __future__ import annotations

import hashlib
import json
import pathlib

import numpy as np

GOLDEN_DIR = pathlib.Path(__file__).resolve().parent / "golden"


def golden_names(include_slow: bool = True):
    return sorted(p.stem for p in GOLDEN_DIR.glob("*.json"))


def load_golden(name: str) -> dict:
    return json.loads((GOLDEN_DIR / (name + ".json")).read_text())


def sha(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def level_digests(level) -> dict:
    return dict(
        n=int(level.n),
        base=int(level.base),
        cms_sha256=sha(level.cms),
        op_sha256=sha(level.op),
        left_sha256=sha(level.left),
        right_sha256=sha(level.right),
    )


def assert_level_matches_golden(level, gold_level: dict, where: str):
    got = level_digests(level)
    for key, value in got.items():
        assert value == gold_level[key], f"{where}: {key} differs (got {value}, golden {gold_level[key]})"


def assert_levels_equal(a, b, where: str):
    """Full-array comparison of two level objects (cms/op/left/right/base)."""
    assert a.n == b.n, f"{where}: n {a.n} != {b.n}"
    assert a.base == b.base, f"{where}: base {a.base} != {b.base}"
    assert a.cms.dtype == b.cms.dtype and a.cms.shape == b.cms.shape, where
    for field in ("cms", "op", "left", "right"):
        x, y = getattr(a, field), getattr(b, field)
        if not np.array_equal(x, y):
            bad = np.flatnonzero((x != y).reshape(len(x), -1).any(axis=1))
            raise AssertionError(f"{where}: {field} differs at {len(bad)} rows, first {bad[:5]}")
