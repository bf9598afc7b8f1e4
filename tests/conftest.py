import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(session, config, items):
    """When GPU tests run, put a first test in front that launches libatp's own
    kernels (one tiny layer on a virtual mesh, inputs generated on the host),
    so the first kernel launches of a -m gpu session are the library's rather
    than the device-side input generator's torch kernels."""
    gpu = [it for it in items if it.get_closest_marker("gpu")]
    first = [it for it in gpu if it.name == "test_libatp_kernels_first"]
    if gpu and first:
        items.remove(first[0])
        items.insert(0, first[0])
