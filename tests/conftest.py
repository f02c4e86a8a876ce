"""Test configuration: the `gpu` marker, import paths, shared fixtures.

CPU tests (-m "not gpu") check the oracle against the reference's golden
vectors, the C-ABI library, and the native block manager bit-for-bit against
the reference Engine.  GPU tests (-m gpu) are the attention parity tests and
call through the C-ABI.  When the reference package is present (the build
container), its path is added so the drop-in shares its exception classes.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFERENCE_SRC = os.environ.get("FK_REFERENCE", "/root/reference/pkg/src")
HAVE_REFERENCE = os.path.isdir(os.path.join(REFERENCE_SRC, "semflow"))
# the reference package installed unmodified into baseline/_ref (travels to
# the GPU box, where /root/reference does not exist): the runtime the
# manager-driven GPU tests put above the B200 engine
BASELINE_REF = os.path.join(ROOT, "baseline", "_ref")
if not HAVE_REFERENCE and os.path.isdir(os.path.join(BASELINE_REF, "semflow")):
    REFERENCE_SRC = BASELINE_REF

for p in (ROOT, os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)
if os.path.isdir(os.path.join(REFERENCE_SRC, "semflow")) and REFERENCE_SRC not in sys.path:
    sys.path.insert(1, REFERENCE_SRC)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


def pytest_collection_modifyitems(config, items):
    skip_ref = pytest.mark.skip(reason="reference package not present")
    for item in items:
        if "reference" in item.keywords and not HAVE_REFERENCE:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but no CUDA device is visible")
    return 0
