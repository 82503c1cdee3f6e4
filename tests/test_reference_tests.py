"""The reference's own unit tests (proj/tests/test_*.cpp) and acceptance gate
(proj/tests/acceptance.cpp), compiled UNCHANGED against this repo's drop-in
headers (include/lpmc) and liblpmc_b200.so by tests/cpp/Makefile (the
doctest interface comes from tests/cpp/doctest_shim/doctest.h).

* CPU: the sources compile and link (where /root/reference exists).
* B200: every unit case passes; acceptance criteria 1-8 print PASS
  (criterion 9 drives the reference's CLI, which is out of scope).
The binaries are built in this container (build() / make -C tests/cpp) and
travel to the GPU box with the library; /root/reference is not read there.
"""
from __future__ import annotations

import os
import re
import subprocess

import pytest

from conftest import ROOT

CPP = os.path.join(ROOT, "tests", "cpp")
OUT = os.path.join(CPP, "_reftests")
REF_TESTS = "/root/reference/proj/tests"


def test_reference_tests_build():
    if not os.path.isdir(REF_TESTS):
        pytest.skip("reference sources absent (GPU box): the binaries were built in the container")
    r = subprocess.run(["make", "-C", CPP, "-j4"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert os.path.exists(os.path.join(OUT, "unit_tests"))
    assert os.path.exists(os.path.join(OUT, "acceptance"))


def _binary(name):
    path = os.path.join(OUT, name)
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: build it with make -C tests/cpp (needs /root/reference)")
    return path


@pytest.mark.gpu
def test_reference_unit_tests_pass():
    r = subprocess.run([_binary("unit_tests")], capture_output=True, text=True, timeout=1800)
    print(r.stdout[-6000:])
    summary = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert summary, r.stdout[-2000:] + r.stderr[-2000:]
    total, passed, failed = map(int, summary.groups())
    assert total >= 45 and failed == 0 and r.returncode == 0, r.stdout[-4000:]


@pytest.mark.gpu
def test_reference_acceptance_criteria_1_to_8():
    # argv[1] is the reference CLI (criterion 9 only): not built, out of scope
    r = subprocess.run([_binary("acceptance"), "/nonexistent/lpmc-cli"], capture_output=True,
                       text=True, timeout=3600)
    print(r.stdout)
    status = {int(m.group(2)): m.group(1) for m in
              re.finditer(r"^(PASS|FAIL) (\d+):", r.stdout, re.MULTILINE)}
    for c in range(1, 9):
        assert status.get(c) == "PASS", (c, r.stdout[-4000:])
    assert status.get(9) == "FAIL"  # the CLI determinism check needs the absent CLI
