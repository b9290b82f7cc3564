"""Shared test setup: the `gpu` marker, repo on sys.path, golden fixture loaders."""

import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def blur_input(seed, side, dim):
    """Same generator as tests/golden/make_golden.py:blur_input."""
    return np.random.default_rng(seed).normal(0.0, 1.0, (side, side, dim)).astype(np.float32)


@pytest.fixture(scope="session")
def have_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
