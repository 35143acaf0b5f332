#!/usr/bin/env python3
"""Benchmark of the B200 HOSCF hot path: the fused TTVc sweep (all NEPv blocks
of J(u), rank1::build_j) on BASELINE.json config 5 — the largest single-GPU
config and the north star's scaling config: reference dims 500 x 2000 x 4000
(32 GB fp64, smooth rank-3 + 1e-3 N(0,1)) — plus time-to-converge of HOSCF /
iHOSCF on it and on the other BASELINE configs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step = one sweep of the whole tensor (all P = 3 blocks) at the solver's
uniform01 initial factors.  With N > 1 ranks each rank holds a contiguous slab
along the slowest mode (the 4000 mode), sweeps it, and the blocks are
assembled with NCCL all-reduce (partial blocks) and all-gather (blocks touching
the sharded mode): strong scaling of the fixed 32 GB tensor.  `--gpus N`
without a torchrun environment re-launches itself under torchrun with N ranks.
Prints ONE JSON line on rank 0 (contract in the task statement).

`--impl reference` times the reference's own rank1::build_j (the unmodified
reference compiled by oracle/Makefile, OpenMP over all host cores, its default
determinism=true) on the SAME config: the full 32 GB tensor, generated on the
host by the reference-identical generator, one full build_j per step.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HOSCF TTVc sweep GB/s (fraction of HBM/FP64 roofline); time-to-converge @1-8 GPU"
HEAD_NAME, HEAD_CFG, HEAD_DIMS, HEAD_SEED = "C5", 5, (500, 2000, 4000), 5
HEAD_WORKLOAD = ("C5: HOSCF TTVc sweep (all 3 NEPv blocks of J(u), rank1::build_j) of the "
                 "500x2000x4000 fp64 tensor (reference dims; config 4000x2000x500), "
                 "sum_r w_r sin((r+1)pi i/4000) cos(r pi j/2000) exp(-r k/500) + 1e-3 N(0,1), "
                 "at the solver's uniform01 initial factors (seed 5)")


def head_config():
    return {"workload": HEAD_WORKLOAD, "dims_reference_order": list(HEAD_DIMS),
            "tensor_bytes": 8 * int(np.prod(HEAD_DIMS)),
            "algorithmic_bytes_per_step": sweep_bytes(HEAD_DIMS),
            "l2": "inputs (32 GB) far larger than L2 (126 MB); no flush needed"}


def sweep_bytes(dims) -> int:
    """Algorithmic bytes of one sweep: read A once, write all
    blocks, read the factors."""
    d = len(dims)
    n = int(np.prod(dims))
    blocks = sum(dims[m] * dims[k] for m in range(d) for k in range(m + 1, d))
    return 8 * n + 8 * blocks + 8 * sum(dims)


def level0_bytes(dims) -> int:
    """Algorithmic bytes of the dominant kernel (top-level pass): A once plus its
    outputs B01 (I0 I1), C0 (I0 O), C1 (I1 O) and the factors it reads."""
    n = int(np.prod(dims))
    o = n // (dims[0] * dims[1])
    return 8 * n + 8 * (dims[0] * dims[1] + (dims[0] + dims[1]) * o) + 8 * (dims[0] + dims[1] + o)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def fp64_peak():
    """Measured DFMA peak (tools/fp64_peak.cu, profiles/r02_fp64_peak.json)."""
    p = os.path.join(ROOT, "profiles", "r02_fp64_peak.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["dfma_tflops"]), "measured (profiles/r02_fp64_peak.json)"
    return None, "unmeasured"


def profile_traffic():
    """DRAM read+write bytes of one C5 sweep (all its kernels) from the
    committed ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "r02_sweep_c5_wide_ncu_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("dram_bytes_per_sweep")
    return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every ~2 ms during
    the timed region through NVML (nvidia-smi as a fallback)."""

    BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
            0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, cuda_index: int, period_s: float = 0.002):
        self.cuda_index = cuda_index
        self.period = period_s
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = self.cuda_index
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.cuda_index < len(ids):
                v = ids[self.cuda_index]
                if v.isdigit():
                    idx = int(v)
                else:
                    return pynvml, pynvml.nvmlDeviceGetHandleByUUID(v)
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _loop(self):
        nv, h = self._nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for bit, name in self.BITS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        try:
            self._nvml = self._handle()
            nv, h = self._nvml
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        except Exception:
            self._nvml = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml, 2 ms period"}


# ------------------------------------------------------------ launching --

def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_cmd(argv, gpus: int, port: int):
    """The self-launch command for `--gpus N` outside torchrun: one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__)] + list(argv)


def maybe_relaunch(args, argv) -> bool:
    """Re-exec under torchrun when N > 1 GPUs were asked for without a
    torch.distributed environment.  Returns False when no relaunch is needed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    cmd = torchrun_cmd(argv, args.gpus, free_port())
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # keep NCCL's init lines visible to the driver
    rc = subprocess.call(cmd, env=env)
    sys.exit(rc)


def init_dist(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}")
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
    return world, rank, local, dist


def emit(obj):
    print(json.dumps(obj), flush=True)


def max_over_ranks(v, dist):
    if dist is None:
        return v
    import torch
    x = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return float(x.item())


# ---------------------------------------------------------------- b200 arm --

def run_b200(args):
    import ctypes

    import torch

    import paper_2403_01778_b200 as r1
    from paper_2403_01778_b200 import _lib
    from paper_2403_01778_b200.distributed import (build_j_sharded, init_comm, local_dims,
                                                   slab_bounds, solve_distributed)

    world, rank, local, dist = init_dist(args.gpus)
    torch.cuda.set_device(local)
    ctx = r1.Context(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    L = _lib.lib()
    dims = HEAD_DIMS
    d = len(dims)
    lo, hi = slab_bounds(dims[-1], world, rank)
    ldims = local_dims(dims, lo, hi)
    slab_elems = int(np.prod(ldims))
    first = int(np.prod(dims[:-1])) * lo

    # the rank's slab, generated in HBM (counter-based config generator) in
    # torch-owned memory (16-B aligned, padded) wrapped as an r1_tensor
    a_dev = torch.empty(slab_elems + 2, dtype=torch.float64, device="cuda")
    t = r1.DeviceTensor.wrap(a_dev.data_ptr(), ldims, ctx, keepalive=a_dev)
    gdims = _lib.dims_arr(dims)
    _lib.check(L.r1_generate_config(ctx.handle, t.handle, HEAD_CFG, HEAD_SEED, _lib.u64p(gdims), d,
                                    first))
    # factors: the solver's uniform01 init (solvers.cpp:34-49); a slab's sweep
    # reads its slice of the global last factor in place
    fac_full = uniform01_factors(dims, seed=HEAD_SEED)
    fl = np.concatenate(fac_full)
    fac = torch.from_numpy(fl).cuda()
    nb = int(sum(dims[m] * dims[k] for m in range(d) for k in range(m + 1, d)))
    gblocks = torch.empty(nb, dtype=torch.float64, device="cuda")
    comm = init_comm(ctx, dist, world, rank) if world > 1 else None

    def step():
        if world > 1:  # slab sweep + one NCCL group (r1_build_j_sharded)
            build_j_sharded(ctx, t, dims, fac.data_ptr(), gblocks.data_ptr())
        else:
            _lib.check(L.r1_build_j_device(ctx.handle, t.handle, fac.data_ptr(), gblocks.data_ptr(),
                                           None))

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()

    # ---- device-resident timing (value) + live per-kernel timing (roofline)
    L.r1x_time_kernels(ctx.handle, 1)
    ms_k, nk = ctypes.c_double(), ctypes.c_uint64()
    L.r1x_kernel_time(ctx.handle, ctypes.byref(ms_k), ctypes.byref(nk))  # reset
    launches0 = ctx.launch_count
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = ctx.launch_count - launches0
    L.r1x_kernel_time(ctx.handle, ctypes.byref(ms_k), ctypes.byref(nk))
    L.r1x_time_kernels(ctx.handle, 0)
    ms = max_over_ranks(e0.elapsed_time(e1), dist)
    kernel_ms = ms_k.value / max(1, nk.value)
    value = sweep_bytes(dims) * args.steps / (ms * 1e-3) / 1e9

    # ---- end to end through the public host call with host buffers: N = 1 is
    # r1_build_j (the C-ABI behind rank1::build_j(DenseTensor, FactorSet)):
    # tensor H2D from pinned host memory, factors H2D, sweep, blocks D2H, sync.
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    host = torch.empty(slab_elems, dtype=torch.float64, pin_memory=True)
    host.copy_(a_dev[:slab_elems])
    fac_host = torch.from_numpy(fl).pin_memory()
    blocks_host = torch.empty(nb, dtype=torch.float64, pin_memory=True)
    hdims = _lib.dims_arr(ldims)

    if world == 1:
        def e2e_step():
            _lib.check(L.r1_build_j(ctx.handle, ctypes.cast(host.data_ptr(), _lib._dp), None,
                                    _lib.u64p(hdims), d, ctypes.cast(fac_host.data_ptr(), _lib._dp),
                                    ctypes.cast(blocks_host.data_ptr(), _lib._dp)))
        e2e_path = ("r1_build_j (C-ABI of rank1::build_j): pinned host tensor H2D + factors H2D + "
                    "sweep + blocks D2H per step")
    else:
        def e2e_step():
            _lib.check(L.r1_tensor_copy_from_host(ctx.handle, t.handle,
                                                  ctypes.cast(host.data_ptr(), _lib._dp)))
            fac.copy_(fac_host, non_blocking=True)
            step()
            blocks_host.copy_(gblocks, non_blocking=True)
            stream.synchronize()
        e2e_path = ("per rank: pinned host slab H2D + factors H2D + r1_build_j_sharded (slab "
                    "sweep + NCCL exchange) + blocks D2H per step")

    e2e_step()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0, dist)
    e2e_value = sweep_bytes(dims) * e2e_steps / e2e_s / 1e9

    # e2e with the tensor resident (uploaded once, as in a solve): per step the
    # factors go H2D and the blocks come back D2H
    def e2e_resident_step():
        fac.copy_(fac_host, non_blocking=True)
        step()
        blocks_host.copy_(gblocks, non_blocking=True)
        stream.synchronize()

    e2e_resident_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_resident_step()
    barrier()
    e2e_res_s = max_over_ranks(time.perf_counter() - t0, dist)
    e2e_res_value = sweep_bytes(dims) * args.steps / e2e_res_s / 1e9
    del host

    # ---- time to converge on the headline config (tensor resident): HOSCF and
    # iHOSCF at tol 1e-10.  One GPU: the C++ device driver; N GPUs: the
    # slab-sharded driver (sweep per rank + NCCL exchange, replicated eigen /
    # RQI / stopping test)
    ttc = None
    if not args.skip_solve:
        ttc = {}

        def ttc_one(alg):
            o = r1.SolveOptions(tol=1e-10, max_iters=200, seed=HEAD_SEED)
            runs = []
            for _ in range(3):  # first run includes one-time plan / workspace setup
                torch.cuda.synchronize()
                barrier()
                ts = time.perf_counter()
                if world == 1:
                    rep = r1.solve(alg, t, o, ctx)
                else:
                    rep = solve_distributed(alg, t, dims, o, ctx)
                torch.cuda.synchronize()
                runs.append(max_over_ranks(time.perf_counter() - ts, dist))
            return {"seconds": round(statistics.median(runs[1:]), 6),
                    "seconds_first_call": round(runs[0], 6), "iterations": rep.iterations,
                    "iterations_per_s": round(rep.iterations / statistics.median(runs[1:]), 2),
                    "sweeps": rep.total_sweeps, "converged": rep.converged,
                    "lambda": rep.result.lambda_, "t_build_j": round(rep.wall_build_j(), 6),
                    "t_eig": round(rep.wall_eig(), 6)}

        for alg in ("hoscf", "ihoscf"):
            try:
                ttc[alg] = ttc_one(alg)
            except Exception as e:  # keep the sweep line even if a solve fails
                ttc[alg] = {"error": f"{type(e).__name__}: {e}"}

    del t
    a_dev = None
    torch.cuda.empty_cache()

    # ---- the other BASELINE configs (single GPU): sweep throughput and
    # time-to-converge on device-generated inputs
    other = None
    if world == 1 and not args.skip_configs:
        try:
            other = other_configs(r1, _lib, ctx, stream)
        except Exception as e:
            other = {"error": f"{type(e).__name__}: {e}"}

    # ---- CPU baseline: the compiled reference on this host's cores (rank 0, N=1)
    cpu = None
    if world == 1 and rank == 0 and not args.skip_cpu:
        try:
            cpu = cpu_baseline(args, other)
        except Exception as e:
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {type(e).__name__}: {e}"}

    if rank == 0:
        peak, peak_kind = measured_peaks()
        f64_peak, f64_kind = fp64_peak()
        sweep_ms = ms / args.steps
        k_achieved = level0_bytes(ldims) / (kernel_ms * 1e-3) / 1e9 if kernel_ms > 0 else None
        flops = 6.0 * float(np.prod(ldims))  # 3 FMA per element
        f64_achieved = flops / (sweep_ms * 1e-3) / 1e12
        traffic = profile_traffic()
        out = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(sweep_ms, 6),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE config 5, generated in HBM by the counter-based "
                    "generator; the reference arm generates the same config on the host)",
            "config": dict(head_config(),
                           parallelism=(f"slab{world} along the slowest mode (r1_build_j_sharded: "
                                        "NCCL all-reduce + all-gather in one group)")
                           if world > 1 else "single GPU"),
            "roofline": {
                "bound": "hbm",
                "kernel": "the whole sweep: sweep3_box_kernel (fused top-level pass) + "
                          "finish_kernel (fixed-order partial sums)",
                "achieved": round(value / world, 3),
                "peak": peak,
                "unit": "GB/s",
                "frac": round(value / world / peak, 4),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic_bytes_per_sweep": sweep_bytes(ldims),
                "sweep_ms": round(sweep_ms, 6),
                "traffic": traffic,
                "traffic_source": "profiles/r02_sweep_c5_wide_ncu_summary.json (ncu --set full, "
                                  "dram__bytes_read.sum + dram__bytes_write.sum over the "
                                  "sweep's kernels)" if traffic else None,
                "level0_kernel": {
                    "name": "sweep3_box_kernel",
                    "ms_per_launch": round(kernel_ms, 6),
                    "algorithmic_bytes_per_launch": level0_bytes(ldims),
                    "achieved": round(k_achieved, 3) if k_achieved else None,
                    "frac": round(k_achieved / peak, 4) if k_achieved else None,
                    "share_of_sweep": round(kernel_ms / sweep_ms, 4) if kernel_ms else None},
                "fp64": {"flops_per_sweep": flops, "achieved_tflops": round(f64_achieved, 3),
                         "peak_tflops": f64_peak, "peak_source": f64_kind,
                         "frac": round(f64_achieved / f64_peak, 4) if f64_peak else None},
            },
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * slab_elems + 8 * len(fl),
                    "d2h_bytes_per_step": 8 * nb, "steps": e2e_steps, "path": e2e_path},
            "e2e_resident": {"value": round(e2e_res_value, 3), "unit": "GB/s",
                             "h2d_bytes_per_step": 8 * len(fl), "d2h_bytes_per_step": 8 * nb,
                             "steps": args.steps,
                             "path": "tensor resident (one upload per solve); factors H2D + "
                                     "sweep + blocks D2H per step"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if ttc is not None:
            out["time_to_converge"] = ttc
        if other is not None:
            out["configs"] = other
        if cpu is not None:
            out["cpu_baseline"] = cpu
        emit(out)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


OTHER_CONFIGS = [
    # name, cfg, reference dims, solves: (alg, options)
    ("C1", 1, (100, 100, 100), [("hoscf", dict(tol=1e-300, max_iters=500, init="provided",
                                              scf_lambda_rtol=1e-12))]),
    ("C2", 2, (1000, 1000, 1000), [("hoscf", dict(tol=1e-10, max_iters=100)),
                                   ("ihoscf", dict(tol=1e-10, max_iters=100))]),
    ("C3", 3, (200, 200, 200, 200), [("hoscf", dict(tol=1e-300, max_iters=100, record_kkt=False))]),
    ("C4", 4, (60, 60, 60, 60, 60), [("hoscf", dict(tol=1e-10, max_iters=100)),
                                     ("ihoscf", dict(tol=1e-10, max_iters=100))]),
]


def other_configs(r1, _lib, ctx, stream):
    import torch
    res = {}
    L = _lib.lib()
    for name, cfg, dims, solves in OTHER_CONFIGS:
        n = int(np.prod(dims))
        a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
        t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx, keepalive=a)
        gd = _lib.dims_arr(dims)
        _lib.check(L.r1_generate_config(ctx.handle, t.handle, cfg, cfg, _lib.u64p(gd), len(dims), 0))
        fl = np.concatenate(uniform01_factors(dims, cfg))
        fac = torch.from_numpy(fl).cuda()
        nb = int(sum(dims[m] * dims[k] for m in range(len(dims)) for k in range(m + 1, len(dims))))
        blocks = torch.empty(nb, dtype=torch.float64, device="cuda")

        def sweep():
            _lib.check(L.r1_build_j_device(ctx.handle, t.handle, fac.data_ptr(), blocks.data_ptr(),
                                           None))

        for _ in range(3):
            sweep()
        reps = 20
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            sweep()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        entry = {"dims_reference_order": list(dims), "tensor_bytes": 8 * n,
                 "sweep_ms": round(ms, 4), "sweep_gbs": round(sweep_bytes(dims) / ms / 1e6, 2),
                 "sweep_frac": round(sweep_bytes(dims) / ms / 1e6 / measured_peaks()[0], 4)}
        for alg, kw in solves:
            kw = dict(kw)
            init = kw.pop("init", None)
            o = r1.SolveOptions(seed=cfg, **kw)
            if init == "provided":  # C1: normalised all-ones (BASELINE config 1)
                o.init = "provided"
                o.init_factors = [np.ones(v) for v in dims]
                kw["init"] = init
            runs = []
            for _ in range(2 if cfg in (1, 3) else 3):  # first run: one-time setup
                torch.cuda.synchronize()
                ts = time.perf_counter()
                rep = r1.solve(alg, t, o, ctx)
                torch.cuda.synchronize()
                runs.append(time.perf_counter() - ts)
            te = statistics.median(runs[1:])
            entry[alg] = {"seconds": round(te, 6), "seconds_first_call": round(runs[0], 6),
                          "iterations": rep.iterations,
                          "iterations_per_s": round(rep.iterations / te, 2),
                          "sweeps": rep.total_sweeps, "converged": rep.converged,
                          "lambda": rep.result.lambda_, "t_build_j": round(rep.wall_build_j(), 6),
                          "t_eig": round(rep.wall_eig(), 6), "options": kw}
        res[name] = entry
        del t, a, blocks
        torch.cuda.empty_cache()
    return res


def uniform01_factors(dims, seed):
    """random_unit_factors (solvers.cpp:34-49) with CounterRng(seed, 2)."""
    G = 0x9e3779b97f4a7c15
    M = (1 << 64) - 1

    def mix(z):
        z ^= z >> 30
        z = (z * 0xbf58476d1ce4e5b9) & M
        z ^= z >> 27
        z = (z * 0x94d049bb133111eb) & M
        z ^= z >> 31
        return z

    key = mix((seed + G * 3) & M)
    c = 0
    out = []
    for n in dims:
        u = np.empty(n)
        for i in range(n):
            c += 1
            u[i] = (mix((key + G * c) & M) >> 11) * 2.0 ** -53
        s = 0.0
        for v in u.tolist():
            s += v * v
        out.append(u / np.sqrt(s))
    return out


# ------------------------------------------------------- CPU reference arms --

def ref_config_tensor(cfg, dims, seed):
    """The config tensor in the reference's own DenseTensor, filled on the host
    by the oracle's C generator (bit-identical to the reference's generators,
    tests/test_oracle_pins.py; OpenMP over all cores)."""
    import ctypes

    from oracle import rank1_oracle as O
    from oracle import ref
    dd = np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))

    def fill(addr, n):
        rc = O.lib().r1o_gen_config(cfg, dd.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                    len(dims), seed, ctypes.cast(addr, ctypes.POINTER(ctypes.c_double)))
        if rc != 0:
            raise RuntimeError(f"gen_config {cfg} failed")
    return ref.RefTensor(fill, dims)


def cpu_baseline(args, other):
    """The reference's own CPU path on the same workload, rank 0 / N = 1: a
    bounded number of full build_j calls on the full C5 tensor (determinism
    true = the reference default, and false), plus the reference's
    time-to-converge on C1 (HOSCF, the GPU run's iteration count) and C4."""
    from oracle import ref
    if not ref.available():
        return {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    cores = ref.max_threads()
    t = ref_config_tensor(HEAD_CFG, HEAD_DIMS, HEAD_SEED)
    f = uniform01_factors(HEAD_DIMS, HEAD_SEED)
    t.time_build_j(f, reps=1)  # warm (page-in)
    reps = 3
    _, secs = t.time_build_j(f, reps=reps)
    gbs = sweep_bytes(HEAD_DIMS) * reps / float(np.sum(secs)) / 1e9
    _, secs_nd = t.time_build_j(f, reps=1, determinism=False)
    gbs_nd = sweep_bytes(HEAD_DIMS) / float(np.sum(secs_nd)) / 1e9
    t.close()
    out = {"value": round(gbs, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
           "sample": f"rank1::build_j of the compiled reference (OpenMP, {cores} threads, "
                     f"determinism=true: at d = 3 its block-parallel schedule keeps P = 3 "
                     f"threads busy) on the full C5 tensor (32 GB), {reps} timed sweeps",
           "determinism_false": {"value": round(gbs_nd, 3), "unit": "GB/s",
                                 "sample": "same tensor and factors, determinism=false, 1 sweep"}}
    ttc = {}
    c1_iters = None
    try:
        c1_iters = int(other["C1"]["hoscf"]["iterations"])
    except Exception:
        c1_iters = 201
    for name, cfg, dims, alg, kw in (
            ("C1", 1, (100, 100, 100), "hoscf",
             dict(tol=1e-300, max_iters=c1_iters, record_kkt=False,
                  init_factors=[np.ones(100)] * 3)),
            ("C4", 4, (60, 60, 60, 60, 60), "hoscf", dict(tol=1e-10, max_iters=100, seed=4))):
        try:
            rt = ref_config_tensor(cfg, dims, cfg)
            ts = time.perf_counter()
            rep = rt.solve(alg, **kw)
            sec = time.perf_counter() - ts
            rt.close()
            ttc[name] = {"algorithm": alg, "seconds": round(sec, 4), "iterations": rep["iterations"],
                         "lambda": rep["lam"],
                         "t_build_j": round(sum(r["t_build_j"] for r in rep["trace"]), 4),
                         "t_eig": round(sum(r["t_eig"] for r in rep["trace"]), 4),
                         "note": "fixed iteration count = the GPU run's sigma-rule stop "
                                 "(the reference has no sigma rule)" if name == "C1" else
                                 "tol 1e-10 (Eq. 11), seed 4"}
        except Exception as e:
            ttc[name] = {"error": f"{type(e).__name__}: {e}"}
    out["time_to_converge"] = ttc
    return out


def run_reference(args):
    """The reference arm: the reference's own rank1::build_j on the host cores,
    same metric / config / unit as the b200 arm, one full 32 GB sweep per step."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/librank1_ref.so is not built"})
        return
    t0 = time.perf_counter()
    t = ref_config_tensor(HEAD_CFG, HEAD_DIMS, HEAD_SEED)
    gen_s = time.perf_counter() - t0
    f = uniform01_factors(HEAD_DIMS, HEAD_SEED)
    # CPU warm-up: page-in and OpenMP pool start; full sweeps take seconds each,
    # so at most 2 warm-up and args.ref_max_steps timed sweeps keep the run to minutes
    warm = max(1, min(args.warmup, 2))
    t.time_build_j(f, reps=warm)
    steps = max(1, min(args.steps, args.ref_max_steps))
    _, secs = t.time_build_j(f, reps=steps)
    _, secs_nd = t.time_build_j(f, reps=1, determinism=False)
    t.close()
    total = float(np.sum(secs))
    value = sweep_bytes(HEAD_DIMS) * steps / total / 1e9
    cores = ref.max_threads()
    sample = (f"rank1::build_j (compiled reference, C++/OpenMP, {cores} threads, determinism=true) "
              f"on the full C5 tensor (32 GB) per step; {steps} timed full sweeps after {warm} "
              f"warm-up (host generation {gen_s:.1f} s, untimed)")
    emit({
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "timed_sweeps": steps,
        "warmup": warm,
        "ms_per_step": round(total / steps * 1e3, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE config 5, reference-identical host generator)",
        "config": dict(head_config(), parallelism=f"CPU, {cores} OpenMP threads"),
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores,
                         "kind": "reference", "sample": sample,
                         "determinism_false": {
                             "value": round(sweep_bytes(HEAD_DIMS) / float(secs_nd[0]) / 1e9, 3),
                             "unit": "GB/s", "sample": "1 full sweep, determinism=false"}},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    })


def parse_args(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-max-steps", type=int, default=20)
    ap.add_argument("--skip-solve", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-configs", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    return args


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    if args.impl == "reference":
        run_reference(args)
        return
    maybe_relaunch(args, argv)
    run_b200(args)


if __name__ == "__main__":
    main()
