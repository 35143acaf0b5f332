"""The C++ drop-in: a program written against the reference's rank1:: API
compiles against include/rank1/*.hpp and links librank1_b200.so (CPU suite);
on a B200 it runs and matches the compiled reference (GPU suite)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "test_dropin")
PKG = os.path.join(ROOT, "paper_2403_01778_b200")
REF = os.path.join(ROOT, "oracle", "_ref")


def _compile():
    if not os.path.exists(os.path.join(REF, "librank1_ref.so")):
        pytest.skip("oracle/_ref not built")
    cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), SRC, "-o", OUT,
           "-L" + PKG, "-lrank1_b200", "-L" + REF, "-lrank1_ref",
           f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{REF}"]
    # the product library is named librank1_b200.so: link by path
    cmd = [c if c != "-lrank1_b200" else os.path.join(PKG, "librank1_b200.so") for c in cmd]
    cmd = [c if c != "-lrank1_ref" else os.path.join(REF, "librank1_ref.so") for c in cmd]
    subprocess.run(cmd, check=True)
    return OUT


def test_cpp_dropin_compiles_and_links():
    assert os.path.exists(_compile())


@pytest.mark.gpu
def test_cpp_dropin_runs_on_b200(gpu_ctx):
    exe = _compile()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
