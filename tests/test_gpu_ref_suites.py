"""The reference's OWN test programs, compiled unmodified against the drop-in.

tests/cpp/build_ref_suites.sh compiles proj/tests/acceptance.cpp and the
doctest unit suites (proj/tests/*_test.cpp) against include/tucker/*.hpp and
libtucker_b200.so, so every ``tucker::`` call they make runs on the B200
engine.  The binaries are built here (where /root/reference exists) and
travel to the GPU box in tests/_refbin/.

One assertion is excluded, by file:line: harness_test.cpp:192 asks that a
TTMcTC call on 10 000 nonzeros take at least 5x as long as one on 1 000
(CPU-serial time scaling).  On the device both calls are launch-latency bound
(~10 us), so the ratio is about 1; DESIGN.md records this deviation.
"""
import os
import re
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "_refbin")
REF_TESTS = "/root/reference/proj/tests"
# (file, line) of assertions that encode CPU timing behaviour, not results
EXPECTED_DEVIATIONS = {("harness_test.cpp", 192)}


def _binary(name):
    p = os.path.join(BIN, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (tests/cpp/build_ref_suites.sh needs /root/reference)")
    return p


def test_ref_suites_compile_against_dropin():
    """CPU: the reference's test sources compile and link against the drop-in headers + shim."""
    if not os.path.isdir(REF_TESTS):
        pytest.skip("reference tests not present")
    r = subprocess.run(["bash", os.path.join(ROOT, "tests", "cpp", "build_ref_suites.sh")], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    for name in ("acceptance_b200", "unit_b200"):
        assert os.path.exists(os.path.join(BIN, name))


@pytest.mark.gpu
def test_reference_acceptance_suite():
    r = subprocess.run([_binary("acceptance_b200")], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    passed = re.findall(r"^criterion (\d+) \(.*\): PASS", r.stdout, re.M)
    assert r.returncode == 0, r.stdout + r.stderr
    assert sorted(int(c) for c in passed) == list(range(1, 10)), r.stdout


@pytest.mark.gpu
def test_reference_unit_suites():
    r = subprocess.run([_binary("unit_b200")], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    failures = re.findall(r"([\w.]+):(\d+): FAILED", r.stderr)
    unexpected = [f for f in failures if (os.path.basename(f[0]), int(f[1])) not in EXPECTED_DEVIATIONS]
    assert not unexpected, r.stderr
    summary = re.search(r"test cases: (\d+) \| (\d+) passed", r.stdout)
    assert summary and int(summary.group(1)) >= 58, r.stdout
