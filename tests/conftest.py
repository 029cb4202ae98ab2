"""Test configuration.

Markers: ``gpu`` — needs a B200 (run with ``-m gpu`` on the GPU box); every
other test runs on the CPU container. The CPU oracle (``oracle/``) is test
infrastructure and is imported only from here, smoke() and bench.py.
"""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            with np.load(GOLDEN / f"{name}.npz") as d:
                cache[name] = {k: d[k] for k in d.files}
        return cache[name]

    return load


@pytest.fixture(scope="session")
def cuda():
    """GPU tests must run on the device: fail (not skip) without one."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    from paper_2510_26180_b200 import _lib

    _lib.load()
    return torch.device("cuda")


def c1_config():
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid

    model = LogNormalKL1D(nx=127, d=4, sigma=0.5, ell=0.3)
    grid = make_time_grid(1.0, 16, 32)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    return model, grid, cfg
