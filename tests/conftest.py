import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle


class _Cache(dict):
    """Session cache of seeded config images and full-size oracle solves, so that the slow
    stated-K parity tests (which share images and, for some deltas, oracle runs) build each
    one once.  Keys are plain tuples; values are whatever the builder returned."""

    def get_or(self, key, build):
        if key not in self:
            self[key] = build()
        return self[key]


@pytest.fixture(scope="session")
def cache():
    return _Cache()
