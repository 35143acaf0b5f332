"""The reference's OWN unit tests (/root/reference/proj/tests/test_nepv.cpp,
test_sym_eig.cpp, test_solvers.cpp, test_greedy.cpp, test_tensor.cpp),
compiled unchanged against the drop-in headers include/rank1/ and linked with
librank1_b200.so (tests/cpp/Makefile; doctest replaced by the doctest-
compatible shim tests/cpp/doctest_shim/doctest.h).  On the B200 every test
case must pass: the same assertions, tolerances and exception types the
reference holds itself to, now answered by the device path.

The binaries are built in this container (where /root/reference exists) and
travel to the GPU box; /root/reference is not read at run time."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_ref_unit")
TESTS = ["test_nepv", "test_sym_eig", "test_solvers", "test_greedy", "test_tensor"]


def _exe(name):
    p = os.path.join(BIN, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (make -C tests/cpp needs /root/reference)")
    return p


@pytest.mark.parametrize("name", TESTS)
def test_reference_unit_binary_lists_cases(name):
    """CPU: the binary loads librank1_b200.so and registers the reference's cases."""
    r = subprocess.run([_exe(name), "-ltc"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    assert len([ln for ln in r.stdout.splitlines() if ln.strip()]) >= 5


@pytest.mark.gpu
@pytest.mark.parametrize("name", TESTS)
def test_reference_unit_tests_pass_on_b200(gpu_ctx, name):
    r = subprocess.run([_exe(name)], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert m, out[-3000:]
    assert r.returncode == 0 and int(m.group(3)) == 0, out[-6000:]
