import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def ref_api():
    from oracle import bindings as ob
    if not ob.ref_available():
        pytest.skip("reference oracle (oracle/_ref) not built")
    return ob.ref_api()


@pytest.fixture(scope="session")
def has_ref():
    from oracle import bindings as ob
    return ob.ref_available()
