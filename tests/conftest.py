import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); runs through the C ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(autouse=True)
def _guard_bands(request):
    """DC_GUARD=1 (tools/guardcheck.sh): after every GPU test, every live device buffer's
    guard bands must be intact -- no kernel wrote out of bounds (the memory checker of this
    repo; compute-sanitizer is not available on the GPU pool)."""
    yield
    if os.environ.get("DC_GUARD") != "1" or request.node.get_closest_marker("gpu") is None:
        return
    import ctypes as C
    from paper_1910_01031_b200 import _lib
    if _lib._lib is None:
        return
    msg = C.create_string_buffer(4096)
    n = C.c_int32()
    _lib._lib.dc_check_guards(msg, 4096, C.byref(n))
    assert n.value == 0, msg.value.decode()


@pytest.fixture(scope="session")
def oracle():
    from checkers import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from checkers import Ref, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built (reference headers absent on this host)")
    return Ref()
