import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running CPU oracle test")


@pytest.fixture(scope="session")
def cfg1():
    import synth
    return synth.get_config(1)


@pytest.fixture(scope="session")
def prob1(cfg1):
    from oracle import entries
    return entries.problem_from_config(cfg1)


@pytest.fixture(scope="session")
def dense1(prob1):
    """Dense Z of config 1 (5184 x 1128) by the oracle quadrature (≈25 s, once per session)."""
    from oracle import entries
    return entries.dense(prob1)


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
