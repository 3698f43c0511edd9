"""The reference's OWN C++ test suites against this repo's drop-in kvrail library.

oracle/Makefile `suites` compiles /root/reference/proj/tests/acceptance.cpp and the
94 doctest unit cases (test_pager, test_transport, test_far_view, test_scenario,
test_concurrency, ... with the doctest shim in oracle/doctest_shim/) UNMODIFIED
against include/kvrail/*.hpp and links them with paper_2605_09735_b200/lib/
libkvrail.so — no reference library in the link. They must pass exactly as they do
against the reference (acceptance.cpp:582-596: 10 criteria; doctest: 94 cases).
With KVRAIL_B200_DEVICE=0 every run_scenario of the acceptance suite runs the B200
path (payload in HBM, the step graph, K-scan, K-gather, K-attn).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = os.path.join(ROOT, "oracle", "_ref", "suites")


def suite(name):
    path = os.path.join(SUITES, name)
    if not os.path.exists(path):
        pytest.skip("reference suites not built (oracle/Makefile suites needs /root/reference)")
    return path


def test_reference_unit_suite_against_our_library():
    out = subprocess.run([suite("unit_tests")], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "test cases: 94 | 94 passed | 0 failed" in out.stdout


def test_reference_acceptance_suite_against_our_library():
    out = subprocess.run([suite("acceptance")], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert out.stdout.count("[PASS]") == 10 and "0 criterion(s) failed" in out.stdout


@pytest.mark.gpu
def test_reference_acceptance_suite_on_the_b200():
    # the variable is honoured: a device that does not exist fails the run
    bad = subprocess.run([suite("acceptance")], capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, KVRAIL_B200_DEVICE="97"))
    assert bad.returncode != 0
    env = dict(os.environ, KVRAIL_B200_DEVICE="0")
    out = subprocess.run([suite("acceptance")], capture_output=True, text=True, timeout=1800, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert out.stdout.count("[PASS]") == 10 and "0 criterion(s) failed" in out.stdout
