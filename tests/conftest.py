import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")

for p in (str(ROOT),):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_sessionstart(session):
    """Build the sm_100a library in-tree if it is missing (nvcc cross-compiles on
    the CPU box; the GPU box image has it too).  Building is not a fallback: the
    CUDA path is still the only one."""
    lib = ROOT / "paper_2411_02820_b200" / "libdroidspeak.so"
    if not lib.exists():
        try:
            from paper_2411_02820_b200 import _build
            _build.build()
        except Exception as exc:  # the ABI tests report the missing library
            print(f"library build failed: {exc}")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout (build container only)")


def have_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_ref = pytest.mark.skip(reason="reference checkout absent")
    cuda = have_cuda()
    ref = REFERENCE_SRC.is_dir()
    for item in items:
        if "gpu" in item.keywords and not cuda:
            item.add_marker(skip_gpu)
        if "reference" in item.keywords and not ref:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def crosskv_ref():
    """The real reference package, imported read-only (build container only)."""
    if not REFERENCE_SRC.is_dir():
        pytest.skip("reference checkout absent")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import crosskv.model as m
    return m
