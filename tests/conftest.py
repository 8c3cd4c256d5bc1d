"""Shared test setup: the `gpu` marker, repo on sys.path, native libs built."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through libphx.so)")
    # build the checker and the product library if they are missing (nvcc
    # cross-compiles sm_100a without a GPU)
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2509_26475_b200", "lib", "libphx.so")):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2509_26475_b200", "csrc")],
                       check=True)


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
