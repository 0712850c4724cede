import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle():
    from oracle import fbf_oracle
    return fbf_oracle.Oracle()


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import fbf_oracle
    if not fbf_oracle.RefLibrary.available():
        if os.path.isdir("/root/reference/proj/src"):
            fbf_oracle.build_oracle(with_ref=True)
        else:
            pytest.skip("oracle/_ref/libfbf_ref.so not built (no /root/reference here)")
    return fbf_oracle.RefLibrary()


@pytest.fixture(scope="session")
def fb():
    import paper_1811_02168_b200 as fb
    fb._lib.load()
    return fb


@pytest.fixture(scope="session")
def gpu(fb):
    if fb._lib.load().fbf_device_count() < 1:
        pytest.skip("no CUDA device")
    return fb
