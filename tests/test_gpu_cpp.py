"""The reference's C++ API on the GPU: tests/cpp/dropin_test (built against
include/fastdeconv/{convolve,rl}.hpp + the reference's data-model headers)
runs its device checks and compares against the oracle."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_on_device():
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    assert os.path.exists(exe), "tests/cpp/dropin_test must be built (make cpptests) before the GPU run"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
