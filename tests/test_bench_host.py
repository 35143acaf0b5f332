"""CPU checks of bench.py's host logic: the `--gpus N` self-launch under
torchrun (one rank per GPU, 127.0.0.1 rendezvous), the world-size assertion,
the headline workload (BASELINE config 5) and its algorithmic byte counts."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_torchrun_command_has_one_rank_per_gpu():
    cmd = bench.torchrun_cmd(["--gpus", "8", "--steps", "5"], 8, 29512)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd
    assert "--master-addr=127.0.0.1" in cmd and "--master-port=29512" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "5"]
    assert cmd[-5].endswith("bench.py")


def test_no_relaunch_for_one_gpu_or_under_torchrun(monkeypatch):
    args = bench.parse_args(["--gpus", "1"])
    assert bench.maybe_relaunch(args, []) is False
    monkeypatch.setenv("WORLD_SIZE", "4")
    args = bench.parse_args(["--gpus", "4"])
    assert bench.maybe_relaunch(args, []) is False


def test_world_size_must_match_gpus(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit, match="--gpus 4 but WORLD_SIZE=2"):
        bench.init_dist(4)


def test_headline_is_config5_and_bytes():
    assert bench.HEAD_DIMS == (500, 2000, 4000) and bench.HEAD_CFG == 5
    n = 500 * 2000 * 4000
    assert bench.sweep_bytes(bench.HEAD_DIMS) == 8 * n + 8 * (500 * 2000 + 500 * 4000 + 2000 * 4000) \
        + 8 * 6500
    cfg = bench.head_config()
    assert cfg["dims_reference_order"] == [500, 2000, 4000]
    assert cfg["tensor_bytes"] == 32_000_000_000


def test_defaults_and_warmup_floor():
    a = bench.parse_args([])
    assert a.gpus == 1 and a.steps == 20 and a.warmup == 5 and a.impl == "b200"
    assert bench.parse_args(["--warmup", "1"]).warmup == 3


def test_uniform01_factors_are_the_solver_init():
    """bench's factors = random_unit_factors (solvers.cpp:34-49) = the oracle's."""
    import numpy as np
    from oracle import rank1_oracle as O
    dims = (5, 7, 3)
    got = bench.uniform01_factors(dims, 5)
    want = O.random_unit_factors(dims, 5, 2)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
