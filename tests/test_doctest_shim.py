"""CPU: the doctest-compatible shim that lets the reference's unit tests compile
unchanged (tests/cpp/doctest_shim/doctest.h) keeps doctest's semantics —
Approx tolerances, SUBCASE re-runs, REQUIRE aborting the case, CHECK_THROWS_AS,
test-case filters and the exit status."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "shim_selftest")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "tests", "cpp", "doctest_shim"),
                    os.path.join(ROOT, "tests", "cpp", "test_doctest_shim.cpp"), "-o", exe], check=True)
    return exe


def test_shim_semantics(tmp_path):
    exe = _build(tmp_path)
    good = subprocess.run([exe, "-tce=bad*"], capture_output=True, text=True)
    assert good.returncode == 0, good.stdout + good.stderr
    assert "4 passed | 0 failed | 4 skipped" in good.stdout
    bad = subprocess.run([exe, "-tc=bad*"], capture_output=True, text=True)
    assert bad.returncode == 1
    assert "4 passed" not in bad.stdout and "| 0 passed | 4 failed |" in bad.stdout
    assert "THREW exception: boom" in bad.stderr
    listed = subprocess.run([exe, "-ltc"], capture_output=True, text=True).stdout.split("\n")
    assert "approx semantics" in listed and len([x for x in listed if x]) == 8
