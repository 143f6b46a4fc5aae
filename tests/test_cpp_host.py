"""Runs the C++ operator-API test driver (tests/cpp/portten_tests): host-only checks on
CPU, and the device parity checks through the C++ API under -m gpu."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "portten_tests")


def _run(*args):
    assert os.path.exists(BIN), "tests/cpp/portten_tests not built (make tests)"
    r = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
    return r.stdout


def test_cpp_host_api():
    _run()


@pytest.mark.gpu
def test_cpp_api_on_device():
    out = _run("--gpu")
    assert "(gpu)" in out
