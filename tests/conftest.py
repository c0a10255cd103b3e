"""Shared pytest setup: marker registration, in-tree native build, repo on sys.path."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run through gpurun)")
    config.addinivalue_line("markers", "slow: takes more than ~10 s on the CPU")
    # Host-side artefacts (generator, oracle) are cheap to (re)build; `make` is a
    # no-op when they are current.  The CUDA library is built by build() / make.
    targets = ["workloads/libgskgen.so", "oracle/liboracle.so"]
    subprocess.run(["make", "-s", "-C", ROOT] + targets, check=True)


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(pytest.mark.timeout(900))
