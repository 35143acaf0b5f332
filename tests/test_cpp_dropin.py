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


MULTI = os.path.join(ROOT, "tests", "cpp", "test_multi_gpu.cpp")


def _compile_multi():
    out = os.path.join(ROOT, "tests", "cpp", "test_multi_gpu")
    cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), MULTI, "-o", out,
           os.path.join(PKG, "librank1_b200.so"), f"-Wl,-rpath,{PKG}"]
    subprocess.run(cmd, check=True)
    return out


def test_cpp_multi_gpu_program_compiles():
    assert os.path.exists(_compile_multi())


@pytest.mark.gpu
def test_cpp_multi_gpu_path_matches_single(gpu_ctx):
    """R1_NUM_GPUS=1 takes the sharded C++ path (slab upload, r1_comm_init_all,
    r1_solve_sharded on a thread per GPU) on this one-GPU box: bit-identical to
    the default single-context path."""
    exe = _compile_multi()
    env0 = {k: v for k, v in os.environ.items() if k != "R1_NUM_GPUS"}
    one = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=env0)
    multi = subprocess.run([exe], capture_output=True, text=True, timeout=300,
                           env=dict(env0, R1_NUM_GPUS="1"))
    assert one.returncode == 0, one.stderr
    assert multi.returncode == 0, multi.stderr
    # ncclCommInitAll prints its version banner on stdout
    body = lambda out: [ln for ln in out.splitlines() if not ln.startswith("NCCL")]  # noqa: E731
    assert body(one.stdout) == body(multi.stdout)
    assert one.stdout.count("hoscf") == 2
