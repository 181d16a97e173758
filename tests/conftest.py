import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# the upload wire's on/off default depends on the host's core count: pin it on so the
# wire tests (and every large upload) take the same path on any box (read once, at the
# library's first use: MHG_OPT_UPLOAD_WIRE's initial value)
os.environ.setdefault("MHG_UPLOAD_WIRE", "16")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.binding import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The reference library compiled in place (oracle/_ref/libmhref.so)."""
    from oracle.binding import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libmhref.so not built (reference tree absent)")
    return Reference()


@pytest.fixture(scope="session")
def mh():
    import paper_1705_04807_b200 as m
    return m


@pytest.fixture(scope="session")
def gpu(mh):
    """Fails (does not skip) when a gpu-marked test runs without a usable B200."""
    import torch
    assert torch.cuda.is_available(), "gpu test without a CUDA device"
    st = mh.lib().mhg_device_check()
    assert st == 0, mh.lib().mhg_last_error().decode()
    return torch.device("cuda:0")


@pytest.fixture
def opts(mh):
    """opts(key, value): set an mhg option (mh.OPT_*) for this test only."""
    saved = {}

    def set_(key, value):
        if key not in saved:
            saved[key] = mh.get_option(key)
        mh.set_option(key, value)
    yield set_
    for k, v in saved.items():
        mh.set_option(k, v)
