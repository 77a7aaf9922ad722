"""The reference's own doctest suites (/root/reference/proj/tests/test_*.cpp),
compiled unmodified by oracle/Makefile (doctest shim) against
  * the reference library itself   -> oracle/_ref/tests_ref/   (CPU)
  * our drop-in libmoesched.so     -> oracle/_ref/tests_b200/  (B200)
Both must fail exactly the same checks (the reference's own suite fails two
statistical checks of test_trace.cpp:217-219 against its own library)."""
import os
import re
import subprocess

import pytest

from conftest import REPO

REF_DIR = os.path.join(REPO, "oracle", "_ref", "tests_ref")
B200_DIR = os.path.join(REPO, "oracle", "_ref", "tests_b200")
SUITES = ["test_core", "test_trace", "test_router", "test_cache", "test_prefetch", "test_balancer"]
KNOWN_REF_FAILURES = {"test_trace": 2}  # test_trace.cpp:217,219 fail on the reference library too


def run_suite(path):
    out = subprocess.run([path], capture_output=True, text=True, timeout=600)
    m = re.search(r"test cases: (\d+) \| (\d+) failed \| checks: (\d+) \| (\d+) failed", out.stdout)
    assert m, out.stdout + out.stderr
    return tuple(int(x) for x in m.groups()), out.stderr


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_reference_library(suite):
    path = os.path.join(REF_DIR, suite)
    if not os.path.exists(path):
        pytest.skip("reference test binaries not built here (needs /root/reference)")
    (cases, failed_cases, checks, failed), err = run_suite(path)
    assert failed == KNOWN_REF_FAILURES.get(suite, 0), err


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_b200_dropin(gpu, suite):
    path = os.path.join(B200_DIR, suite)
    if not os.path.exists(path):
        pytest.skip("drop-in test binaries not built (oracle/Makefile ref-tests)")
    (cases, failed_cases, checks, failed), err = run_suite(path)
    assert failed == KNOWN_REF_FAILURES.get(suite, 0), err
    ref = os.path.join(REF_DIR, suite)
    if os.path.exists(ref):
        (rc, _, rchecks, _), _ = run_suite(ref)
        assert (cases, checks) == (rc, rchecks)  # same cases, same number of checks executed
