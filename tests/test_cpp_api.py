"""The reference's C++ API (include/projprod/*.hpp) as a drop-in: the library
links against the engine's C-ABI, and the reference's own test cases
(restated in tests/cpp/test_projprod.cpp) pass on a B200."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "cpp", "build", "test_projprod")


def test_cpp_api_builds_and_links():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "cpp")], check=True)
    assert os.path.exists(BIN)
    out = subprocess.run(["ldd", os.path.join(ROOT, "cpp", "build", "libprojprod.so")],
                         capture_output=True, text=True).stdout
    assert "libppc.so" in out and "not found" not in out.split("libppc.so")[1].splitlines()[0]


@pytest.mark.gpu
def test_cpp_api_reference_cases_on_gpu():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "cpp")], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout
