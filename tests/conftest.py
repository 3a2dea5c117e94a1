import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running statistical test")


def _ensure_built():
    lib = os.path.join(REPO, "paper_1605_02669_b200", "libacs_b200.so")
    orc = os.path.join(REPO, "oracle", "liboracle.so")
    if not (os.path.exists(lib) and os.path.exists(orc)):
        subprocess.run(["make", "-s", "-j8"], cwd=REPO, check=True)


_ensure_built()


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref (reference build) not present")
    return oracle.Reference()


@pytest.fixture(scope="session")
def acs():
    import paper_1605_02669_b200 as P
    return P


@pytest.fixture(scope="session")
def gpu(acs):
    if acs.device_count() < 1:
        pytest.fail("no CUDA device visible to libacs_b200.so (gpu-marked test on a CPU box?)")
    return 0
