import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# In-process TMP groups (tests/test_gpu_group.py) run T ranks' streams in one CUDA context: more hardware
# queues keep the ranks from serialising behind each other (read when the context is created).  Correctness
# does not depend on it: the group issues its ranks' calls in a topological order (api.cu, InprocGroup).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running (full-size oracle)")


@pytest.fixture(scope="session")
def repo_root():
    return ROOT
