import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")


@pytest.fixture(scope="session")
def orc():
    """The CPU oracle (checker) bound through the same ctypes wrapper."""
    import oracle
    return oracle.api()


@pytest.fixture(scope="session")
def gpu():
    """The B200 library.  Fails loudly (no fallback) when it cannot run."""
    if os.environ.get("MPREC_TEST_GPU_AS") == "ref":
        # development aid: run the -m gpu tests' logic against the reference build
        import oracle
        return oracle.ref_api()
    from paper_1912_04385_b200.api import gpu as _gpu
    api = _gpu()
    import ctypes as C
    sm, ma, mi, mem = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    api.call("device_info", C.byref(sm), C.byref(ma), C.byref(mi), C.byref(mem))
    assert (ma.value, mi.value) == (10, 0), f"expected an sm_100 device, got {ma.value}.{mi.value}"
    return api


@pytest.fixture(scope="session")
def ref():
    """The reference's own sources (oracle/_ref, built against the Eigen-subset
    shim) through the same ctypes wrapper; skipped where it was not built."""
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref/libmprec_ref.so not built (needs /root/reference at build time)")
    return oracle.ref_api()
