import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: full-size configurations (minutes)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_value(x):
    """JSON golden values use the string "INF" for 2^64-1."""
    if isinstance(x, list):
        return [golden_value(v) for v in x]
    return 0xFFFFFFFFFFFFFFFF if x == "INF" else x


@pytest.fixture(scope="session")
def cuda_device():
    """GPU tests fail loudly (never skip) when no CUDA device is present."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test run without a CUDA device"
    return torch.device("cuda:0")


def rng_graphs(count, seed0=1, nmax=300, directed=None):
    """Seeded small random graphs of varying size/density (directed and undirected)."""
    import gen

    rs = np.random.default_rng(seed0)
    out = []
    for i in range(count):
        n = int(rs.integers(1, nmax + 1))
        draws = int(rs.integers(0, 4 * n + 1))
        d = bool(rs.integers(0, 2)) if directed is None else directed
        wmax = int(rs.choice([1, 3, 100, (1 << 18) - 1]))
        g = gen.random_graph(n, draws, seed=seed0 * 1000 + i, directed=d, wmax=wmax)
        g.source = int(rs.integers(0, n))
        g.meta["directed"] = d
        out.append(g)
    return out
