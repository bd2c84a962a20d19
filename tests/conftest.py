import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (large shapes)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    if not oracle.have("oracle"):
        subprocess_build()
    return oracle


def subprocess_build():
    import subprocess
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all"], check=True, capture_output=True)


@pytest.fixture(scope="session")
def have_ref():
    import oracle
    if not oracle.have("ref"):
        if os.path.isdir("/root/reference/proj"):
            import subprocess
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True, capture_output=True)
    return oracle.have("ref")
