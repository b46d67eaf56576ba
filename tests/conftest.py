import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU check")


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ctx():
    """One HostContext for the GPU tests: four logical devices on CUDA device 0
    (each with its own stream and buffer store), so partitioned launches over
    P = 1, 2, 4 queues run on a single B200 — the way the reference runs P
    daemons on localhost."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2005_08466_b200 import HostContext

    # on a multi-GPU box the other GPUs are appended as devices 4.. (one per
    # GPU) for tests/test_gpu_multi.py; the first four stay logical devices of GPU 0
    ordinals = [0, 0, 0, 0] + list(range(1, torch.cuda.device_count()))
    c = HostContext(ordinals)
    c.cuda_ordinals = ordinals
    yield c
    c.close()
