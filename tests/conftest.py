import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the built engine")
    config.addinivalue_line("markers", "slow: long-running CPU oracle comparison")


@pytest.fixture(scope="session")
def lto():
    from oracle.bindings import Lto
    return Lto()


@pytest.fixture(scope="session")
def ref():
    """The reference library compiled in place (oracle/_ref); skipped only
    where neither the built .so nor /root/reference exists."""
    from oracle.bindings import Ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return Ref()


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
