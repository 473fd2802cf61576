"""World-size-2 gloo runs of the multi-GPU level exchange (paper_2504_18943_b200/dist.py) on CPU.

The protocol code is the one the CUDA engine uses over NCCL; only the shard engine underneath
is swapped for the numpy stand-in of tests/cpu_shard_engine.py.  Each rank checks every level
(cms, op, left, right, base, separator id) against the C oracle, i.e. "N ranks == 1 rank ==
reference", the multi-GPU analogue of the reference's thread-count determinism tests
(reference tests/test_engine.py:162-175)."""

import json
import os
import pathlib
import socket
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
DEFAULT_OPS = "not,next,future,and,until"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(tmp_path, workload, seed, max_cost, exhaustive, ops=DEFAULT_OPS, world=2, replicate_below=0):
    """replicate_below: levels with fewer candidates are built redundantly on every rank (dist.REPLICATE_BELOW);
    0 = every level goes through the exchange."""
    port = _free_port()
    out = tmp_path / "report"
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   LTLB200_REPLICATE_BELOW=str(replicate_below))
        procs.append(subprocess.Popen(
            [sys.executable, str(ROOT / "tests" / "dist_worker.py"), workload, str(seed), str(max_cost),
             "1" if exhaustive else "0", ops, str(out)], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = [p.communicate(timeout=300)[0] for p in procs]
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    reports = [json.loads(pathlib.Path(str(out) + f".{r}").read_text()) for r in range(world)]
    assert all(r["levels"] == reports[0]["levels"] and r["formula"] == reports[0]["formula"] for r in reports)
    return reports[0]


def test_two_ranks_find_the_reference_witness_on_spec1(tmp_path):
    rep = _run(tmp_path, "spec1", 0, 6, exhaustive=False)
    assert rep["formula"] == "!(b U a)" and rep["unique"] == 33


def test_two_ranks_exhaustive_levels_match_oracle(tmp_path):
    rep = _run(tmp_path, "spec1", 0, 6, exhaustive=True)
    assert rep["levels"] == [3, 8, 14, 21, 32, 34]


def test_two_ranks_wide_rows_and_or_operator(tmp_path):
    # 64 lanes x 16 bit = 128-byte rows travel through the exchange; `or` adds a second triangle family
    _run(tmp_path, "c5", 0, 5, exhaustive=True, ops=DEFAULT_OPS + ",or")


def test_three_ranks_c1(tmp_path):
    rep = _run(tmp_path, "c1", 4, 9, exhaustive=False, world=3)
    assert rep["formula"] == "!F !(!F p1 U p0)"


def test_small_levels_replicated_large_levels_sharded(tmp_path):
    # levels under 200 candidates are built on every rank without an exchange, the rest are sharded:
    # the mix must give the same levels as the all-sharded run and as the oracle
    mixed = _run(tmp_path, "c1", 4, 9, exhaustive=False, replicate_below=200)
    assert mixed["formula"] == "!F !(!F p1 U p0)"
    everything_local = _run(tmp_path, "spec1", 0, 6, exhaustive=True, replicate_below=1 << 30)
    assert everything_local["levels"] == [3, 8, 14, 21, 32, 34]
