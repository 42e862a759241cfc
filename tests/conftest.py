import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a engine")


@pytest.fixture(scope="session", autouse=True)
def _library_built():
    from paper_1909_01786_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        import subprocess
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "paper_1909_01786_b200", "csrc"), "-j4"])
    yield


def pytest_collection_modifyitems(config, items):
    # a device-side deadlock would otherwise hold the GPU box until the outer
    # limit: give every GPU test a watchdog that dumps the stacks and exits
    if not config.pluginmanager.hasplugin("timeout"):
        return
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(300, method="thread"))
