import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle_bindings import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_bindings import RefLib, REF_SO, build_oracle

    if not os.path.exists(REF_SO) and os.path.isdir("/root/reference/proj/src"):
        build_oracle(ref=True)
    if not os.path.exists(REF_SO):
        pytest.skip("compiled reference (oracle/_ref) unavailable")
    return RefLib()


@pytest.fixture(scope="session")
def agpm():
    import paper_2405_03488_b200 as A

    A.lib()  # raises ExtensionMissing if the .so is not built
    return A
