"""The reference's behavioural known answers, checked on the CPU oracle (see tests/behaviour.py)."""

import pytest

import behaviour


@pytest.mark.parametrize("check", behaviour.ALL_CHECKS, ids=lambda f: f.__name__)
def test_oracle(check):
    check(behaviour.OracleBackend())
