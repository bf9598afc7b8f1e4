"""The `isolated` marker (tests/conftest.py) runs a test in a child process
with a timeout: a passing test passes through it, a failing one reports the
child's output, and a hang is killed (CPU-only checks of the mechanism the
fused / gated virtual-mesh GPU tests rely on)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.isolated(timeout=120, retries=0)
def test_isolated_child_runs():
    # runs inside the child process only
    assert os.environ.get("ATP_ISOLATED_CHILD") == "1"


def test_isolated_hang_is_killed(tmp_path):
    body = (
        "import pytest, time\n"
        "@pytest.mark.isolated(timeout=3, retries=1)\n"
        "def test_hangs():\n"
        "    time.sleep(60)\n"
    )
    f = tmp_path / "test_hang_probe.py"
    f.write_text(body)
    conftest = os.path.join(ROOT, "tests", "conftest.py")
    (tmp_path / "conftest.py").write_text(open(conftest).read().replace(
        'ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))', f'ROOT = {str(tmp_path)!r}'))
    out = subprocess.run([sys.executable, "-m", "pytest", str(f), "-q", "-p", "no:cacheprovider", "-rw"],
                         capture_output=True, text=True, timeout=120, cwd=str(tmp_path))
    assert out.returncode != 0
    assert "never finished" in out.stdout and "attempt 2" in out.stdout, out.stdout[-2000:]
