import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def records_from(g, prefix):
    """Unpack concatenated record arrays written by oracle/make_golden.py."""
    na, ne = g[prefix + "n_atoms"], g[prefix + "n_edges"]
    ao = np.concatenate([[0], np.cumsum(na)])
    eo = np.concatenate([[0], np.cumsum(ne)])
    out = []
    for i in range(len(na)):
        out.append(dict(
            z=g[prefix + "z"][ao[i]:ao[i + 1]],
            pos=g[prefix + "pos"][ao[i]:ao[i + 1]],
            edges=g[prefix + "edges"][eo[i]:eo[i + 1]],
            energy=float(g[prefix + "energy"][i]),
            forces=g[prefix + "forces"][ao[i]:ao[i + 1]],
        ))
    return out


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
