"""GPU: the C++ tucker:: drop-in (libtucker_b200.so) exercised from C++ in the
reference tests' idiom (tests/cpp/test_shim.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_shim():
    binp = os.path.join(ROOT, "tests", "cpp", "test_shim.bin")
    lib = os.path.join(ROOT, "paper_2510_16930_b200", "lib")
    src = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
    shim = os.path.join(ROOT, "paper_2510_16930_b200", "lib", "libtucker_b200.so")
    if not os.path.exists(binp) or os.path.getmtime(binp) < max(os.path.getmtime(src), os.path.getmtime(shim)):
        subprocess.check_call(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                               os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-L", lib, "-ltucker_b200",
                               "-lhoqri_b200", f"-Wl,-rpath,{lib}", "-o", binp])
    r = subprocess.run([binp], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
