"""Test configuration.

Markers: ``gpu`` tests run the CUDA path on a B200 (driver: ``pytest -m gpu``);
everything else runs on CPU (``pytest -m "not gpu"``).  The checkers under
oracle/ are test infrastructure; the product (paper_1903_00227_b200) never
imports them.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large sizes (minutes)")


def _ensure_built():
    # oracle/liboracle.so (gcc, seconds) and the product library (nvcc); both
    # are normally prebuilt by __graft_entry__.build() and travel with the repo.
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_1903_00227_b200", "libwrs_b200.so")):
        subprocess.run(["make", "-s", "-j4", "-C",
                        os.path.join(ROOT, "paper_1903_00227_b200", "csrc")], check=True)


_ensure_built()


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
