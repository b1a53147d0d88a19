"""GPU: the C++ drop-in API (include/curvalign/*.hpp) passes the reference's own
hot-path test cases, restated in tests/cpp/test_dropin.cpp (built by `make all`)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_suite(cuda):
    exe = os.path.join(ROOT, "tests", "cpp", "bin", "test_dropin")
    assert os.path.exists(exe), "build/test_dropin missing: run `make dropin_test`"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
