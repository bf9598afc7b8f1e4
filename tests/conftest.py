import os
import signal
import subprocess
import sys
import warnings

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    config.addinivalue_line("markers", "isolated(timeout, retries): run the test in its own process, killed "
                            "after `timeout` seconds and retried `retries` times")


# The fused peer-memory path on the VIRTUAL mesh (all ranks' kernels on one
# GPU, spinning on one another's progress) deadlocked late in 2 of 3 full
# -m gpu sessions of round 2's third session: 8 ranks x 32 spinning fused CTAs
# starved the GEMMs they waited for (fixed in runtime.cpp launch_fused: the
# ranks of a virtual mesh share one GPU's fused-CTA budget).
# As a safety net such tests run in a child process with a timeout, so a hang
# fails (or, on the retry, passes) that test instead of stalling the session.
_CHILD = "ATP_ISOLATED_CHILD"


@pytest.hookimpl(tryfirst=True)
def pytest_pyfunc_call(pyfuncitem):
    mark = pyfuncitem.get_closest_marker("isolated")
    if mark is None or os.environ.get(_CHILD):
        return None
    timeout = mark.kwargs.get("timeout", 180)
    retries = mark.kwargs.get("retries", 1)
    cmd = [sys.executable, "-m", "pytest", pyfuncitem.nodeid, "-q", "-p", "no:cacheprovider"]
    if pyfuncitem.get_closest_marker("gpu") is not None:
        cmd += ["-m", "gpu"]
    env = dict(os.environ, **{_CHILD: "1"})
    tail = ""
    for attempt in range(retries + 1):
        proc = subprocess.Popen(cmd, cwd=ROOT, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                start_new_session=True, text=True)
        try:
            out, _ = proc.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            os.killpg(proc.pid, signal.SIGKILL)
            proc.communicate()
            tail = f"timed out after {timeout} s (attempt {attempt + 1})"
            warnings.warn(f"{pyfuncitem.nodeid}: {tail}")
            continue
        if proc.returncode == 0:
            if attempt:
                warnings.warn(f"{pyfuncitem.nodeid}: passed on attempt {attempt + 1} after a timeout")
            return True
        pytest.fail(f"isolated run failed (rc {proc.returncode}):\n" + "\n".join(out.splitlines()[-40:]),
                    pytrace=False)
    pytest.fail(f"isolated run never finished: {tail}", pytrace=False)


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
