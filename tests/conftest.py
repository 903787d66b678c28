import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libtpshift_b200.so")
    config.addinivalue_line("markers", "reference: imports the read-only reference (container only)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_ref = pytest.mark.skip(reason="/root/reference not present")
    has_ref = os.path.isdir(REFERENCE_SRC)
    for item in items:
        if "gpu" in item.keywords and not has_gpu:
            item.add_marker(skip_gpu)
        if "reference" in item.keywords and not has_ref:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def device():
    import torch
    return torch.device("cuda:0")


@pytest.fixture(autouse=True)
def _device_watchdog(request):
    """A GPU test fails if a device watchdog fired during it (soft abort word, no trap); the
    word is cleared so the next test starts clean."""
    yield
    if "gpu" not in request.node.keywords:
        return
    import torch
    if not torch.cuda.is_available():
        return
    from paper_2605_23945_b200 import _native as nat
    if nat._lib is None:
        return
    torch.cuda.synchronize()
    nat.check_abort(request.node.nodeid)
