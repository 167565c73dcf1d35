import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(autouse=True)
def _parity_context(request):
    """Tag parity records (tests/gpu_common.record) with the running test's id."""
    try:
        from tests import gpu_common
    except ImportError:
        import gpu_common
    gpu_common.CURRENT["test"] = request.node.nodeid
    yield


def pytest_sessionfinish(session, exitstatus):
    """PARITY_REPORT=path: write the measured parity maxima of this session (GPU parity tests)."""
    path = os.environ.get("PARITY_REPORT")
    if not path:
        return
    try:
        from tests import gpu_common
    except ImportError:
        import gpu_common
    if gpu_common.REPORT:
        with open(path, "w") as f:
            json.dump({"exitstatus": int(exitstatus), "records": gpu_common.REPORT}, f, indent=1)
