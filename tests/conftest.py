import pathlib
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")
    config.addinivalue_line("markers", "slow: minute-long CPU case, not part of the default run")


@pytest.fixture(scope="session")
def spec1():
    from paper_2504_18943_b200 import workloads

    return workloads.spec1()


@pytest.fixture(scope="session")
def spec2():
    from paper_2504_18943_b200 import workloads

    return workloads.spec2()
