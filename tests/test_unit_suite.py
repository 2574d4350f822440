"""The reference's own unit suite (/root/reference/proj/tests/unit/*.cpp,
doctest) compiled unchanged against this repository's
libdreamsched through tests/native/doctest_shim/doctest.h (build/unit_tests,
built by the Makefile where /root/reference exists; the binary travels to the
GPU box).  The same sources against the reference itself
(oracle/_ref/unit_tests_ref) pin the shim: every case passes there.

CPU: every case outside trainer_test.cpp (scheduler, cost model, profile,
schedule, simulator) — the host C++ half of the drop-in library.
GPU: trainer_test.cpp's 17 cases, which run plsgd_step / run_training /
stochastic_gradient through the sm_100a path (trainer_test.cpp:37-268)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = os.path.join(REPO, "build", "unit_tests")
REF = os.path.join(REPO, "oracle", "_ref", "unit_tests_ref")


def _run(binary, *flags):
    if not os.path.exists(binary):
        pytest.skip(f"{os.path.relpath(binary, REPO)} not built (needs /root/reference at build time)")
    p = subprocess.run([binary, *flags], capture_output=True, text=True, timeout=900)
    return p.returncode, p.stdout + p.stderr


def _counts(out):
    line = [ln for ln in out.splitlines() if ln.startswith("[doctest-shim] test cases:")][-1]
    parts = [int(x.split()[0]) for x in line.split(":", 1)[1].split("|")]
    return dict(zip(["run", "passed", "failed", "skipped"], parts))


def test_shim_pinned_on_the_reference():
    rc, out = _run(REF)
    c = _counts(out)
    assert rc == 0 and c["failed"] == 0 and c["run"] == 81, out[-3000:]


def test_reference_unit_suite_host_cases():
    rc, out = _run(OURS, "-sfe=*trainer_test.cpp")
    c = _counts(out)
    assert rc == 0 and c["failed"] == 0 and c["run"] == 64, out[-3000:]


@pytest.mark.gpu
def test_reference_unit_suite_trainer_cases_on_gpu():
    rc, out = _run(OURS, "-sf=*trainer_test.cpp")
    c = _counts(out)
    assert rc == 0 and c["failed"] == 0 and c["run"] == 17, out[-3000:]
