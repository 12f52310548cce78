import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libheinfer_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session", autouse=True)
def _built():
    # Build the checkers (and the product, if nvcc is present) once per session.
    from paper_2204_05496_b200 import build

    try:
        build.build_oracle()
    except Exception as e:  # pragma: no cover
        pytest.exit(f"oracle build failed: {e}")
    if not os.path.exists(build.LIB):
        build.build_product()
    yield
