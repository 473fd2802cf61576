"""The C-ABI library loads and exports every symbol include/ltlsynth_b200.h declares.
No compute calls: this runs without a GPU."""

import ctypes
import pathlib
import re

import pytest

from paper_2504_18943_b200 import _native

ROOT = pathlib.Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as entry

    entry.build()
    return _native.load()


def test_header_symbols_are_exported(lib):
    header = (ROOT / "include" / "ltlsynth_b200.h").read_text()
    declared = set(re.findall(r"\b(ltlb200_[a-z_0-9]+)\s*\(", header))
    assert declared == set(_native.EXPORTED_SYMBOLS)
    for name in declared:
        assert getattr(lib, name) is not None, name


def test_abi_version_matches_header(lib):
    header = (ROOT / "include" / "ltlsynth_b200.h").read_text()
    version = int(re.search(r"#define LTLB200_ABI_VERSION (\d+)", header).group(1))
    assert lib.ltlb200_abi_version() == version == _native.ABI_VERSION


def test_stats_struct_matches_header(lib):
    header = (ROOT / "include" / "ltlsynth_b200.h").read_text()
    body = re.search(r"typedef struct ltlb200_stats \{(.*?)\} ltlb200_stats;", header, re.S).group(1)
    fields = re.findall(r"\b(?:uint64_t|uint32_t|double)\s+([a-z_0-9]+);", body)
    assert fields == [name for name, _ in _native.Stats._fields_]


def test_no_device_means_loud_failure(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible; the no-device behaviour is checked on CPU boxes")
    assert lib.ltlb200_device_count() == 0
    from paper_2504_18943_b200 import engine, workloads

    with pytest.raises(_native.NativeEngineError):
        engine.CandidateStore(workloads.spec1())
