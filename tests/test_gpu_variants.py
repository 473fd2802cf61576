"""GPU parity of the engine's run-time switches.

The switches are environment variables that the library reads once per process, so each variant runs the parity
cases in a child process:

  LTLB200_NO_DEFER=1    two synchronisations per level (finalisation launched after the counters
                        were read) instead of the deferred, device-bounded finalisation
  LTLB200_PRUNE=0       no associativity pruning: every AND candidate is probed
  LTLB200_TINY=0        every level through its own launches, instead of the tiny levels of a search built several
                        per launch by narrow_tiny_levels_kernel / wide2_tiny_levels_kernel (the default, which every
                        other test therefore runs)
  LTLB200_TINY_MAX=32768 / LTLB200_WIDE_TINY_MAX=32768  levels of up to 2^15 candidates (default 4096) in the one-CTA kernels
  LTLB200_EARLY_COUNTERS=0  the host waits for the whole finalisation of a level before it reads its counters (default:
                        it reads them behind the summary kernel, while the scatter still runs)
  LTLB200_OPSTREAMS=0   every operator launch of a level on the engine's own stream, one after the
                        other, instead of fanned out over side streams (the default)

Every variant must reproduce the golden fixtures of the unmodified reference bit for bit.
"""

import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parent.parent
CASES = ["spec1_found", "spec1_exh10", "spec2_exh11", "c1_s1", "c3_s0_exh12", "c3_s1_found", "spec2_fuo_exh8"]
WIDE_CASES = ["c3wide_s0_exh8", "c4-512_s0_exh8", "c4-1024_s0_exh8", "c4xl_s0_exh7", "c5_s0_exh8", "c5_s0_or_exh7",
              "w32_s1_found", "w64n_s0_exh9"]

CHILD = """
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import test_gpu_parity as t
for name in {cases!r}:
    t._run_case(name)
print("variant ok")
"""


@pytest.mark.parametrize("switch,value,cases", [("LTLB200_NO_DEFER", "1", CASES + WIDE_CASES),
                                                 ("LTLB200_OPSTREAMS", "0", CASES + WIDE_CASES),
                                                 ("LTLB200_PRUNE", "0", CASES),
                                                 ("LTLB200_TINY", "0", CASES + WIDE_CASES + ["spec1_found_b1", "spec1_or_found", "c1_s0", "c1_s3", "w32n_s2_found", "w64n_s3_found"]),
                                                 ("LTLB200_WIDE_TINY_MAX", "32768", WIDE_CASES),
                                                 ("LTLB200_TINY_MAX", "32768", CASES),
                                                 ("LTLB200_EARLY_COUNTERS", "0", CASES + WIDE_CASES)])
def test_variant_matches_reference(switch, value, cases):
    env = dict(os.environ)
    env[switch] = value
    code = CHILD.format(root=str(ROOT), tests=str(ROOT / "tests"), cases=cases)
    proc = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0 and "variant ok" in proc.stdout, proc.stdout[-2000:] + proc.stderr[-4000:]


REGEX_CHILD = """
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import test_gpu_regex as t
t.test_sequences_wider_than_128_bits_equal_the_oracle(0, t.rx.CostFunction(), 5)
t.test_baseline_shaped_example_sets_equal_the_oracle("re-c2", 10, 207)
t.test_cut_levels_on_top_of_a_store_that_holds_a_solution(207)
print("variant ok")
"""


@pytest.mark.parametrize("switch,value", [("LTLB200_GUIDE_SMEM", "1"), ("LTLB200_NO_DEFER", "1"), ("LTLB200_OPSTREAMS", "0"),
                                          ("LTLB200_TINY", "0"), ("LTLB200_WIDE_TINY_MAX", "32768")])
def test_regex_variant_matches_the_oracle(switch, value):
    """LTLB200_GUIDE_SMEM=1: the regex guide tables staged in the CTA's shared memory (off by default: it costs
    occupancy); and the regex tiles under the two scheduling switches above."""
    env = dict(os.environ)
    env[switch] = value
    code = REGEX_CHILD.format(root=str(ROOT), tests=str(ROOT / "tests"))
    proc = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0 and "variant ok" in proc.stdout, proc.stdout[-2000:] + proc.stderr[-4000:]
