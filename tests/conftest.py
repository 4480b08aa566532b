import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_addoption(parser):
    parser.addoption("--odpo-lib", default=None,
                     help="run the GPU tests against another build of libodpo.so (e.g. "
                          "build_variants/libodpo_experimental.so with the experimental schedules)")


def pytest_configure(config):
    lib = config.getoption("--odpo-lib")
    if lib:
        import paper_2410_18252_b200 as odpo
        odpo.LIB_PATH = os.path.abspath(lib)
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libodpo.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle
