import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs on one box")


def _gpu_count():
    try:
        from paper_1906_05936_b200 import host

        return host.device_count()
    except Exception:
        return 0


@pytest.fixture(scope="session")
def n_gpus():
    return _gpu_count()
