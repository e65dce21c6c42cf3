import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def golden(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


FLAT_KEYS = ("wake_pos", "wake_gamma", "wake_age", "n_wake", "ring_a", "ring_b", "prev_pos",
             "prev_gamma", "n_prev", "prev_lev", "ema")


def flat_of(g):
    """The reference's flattened 11-tuple (rollout.py:59-62) from a fixture dict."""
    out = []
    for k in FLAT_KEYS:
        v = g[k]
        if k in ("n_wake", "ring_a", "ring_b", "n_prev"):
            v = int(v)
        elif k == "prev_lev":
            v = float(v)
        out.append(v)
    return tuple(out)


@pytest.fixture(scope="session")
def oracle_core():
    from oracle import core
    core.build()
    return core
