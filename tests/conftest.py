import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libnnmg_cuda.so")
    config.addinivalue_line("markers", "slow: full-size configuration (minutes)")


def golden(name):
    path = os.path.join(GOLDEN, name + ".npz")
    return dict(np.load(path, allow_pickle=False))


def golden_names(prefix):
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.startswith(prefix) and f.endswith(".npz"))


def dirichlet_arg(s):
    s = str(s)
    if s == "None":
        return None
    if s == "all":
        return "all"
    return [int(t) for t in s.strip("[]").split(",") if t.strip()]


@pytest.fixture(scope="session")
def oracle():
    from oracle import nnmg_oracle

    return nnmg_oracle
