import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libensi.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def c1(oracle_mod):
    """C1 toy parameter set (N'=2^12, L=3, alpha=1, dnum=3) with one key pair."""
    o = oracle_mod.Oracle(12, 3, 1, 3)
    skc, sk, pk = o.keygen(0x454E5349 + 1)
    return o, skc, sk, pk
