#!/usr/bin/env python3
"""Benchmark of the B200 HOSCF hot path: the fused TTVc sweep (all NEPv blocks
of J(u), rank1::build_j) on BASELINE.json config 2 (1000^3 planted rank-one +
noise, 8 GB fp64), plus time-to-converge of HOSCF / iHOSCF on it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step = one sweep of the whole tensor (all P = 3 blocks).  With N > 1 ranks
(torchrun), each rank holds a contiguous slab along the slowest mode, sweeps it
and the blocks are assembled with NCCL all-reduce (partial blocks) and
all-gather (blocks touching the sharded mode): strong scaling of a fixed
tensor.  Prints ONE JSON line on rank 0 (contract in the task statement).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG2_DIMS = (1000, 1000, 1000)  # reference dims (config dims reversed; cubic)
CONFIG2_SEED = 2
METRIC = "HOSCF TTVc sweep GB/s (fraction of HBM/FP64 roofline); time-to-converge @1-8 GPU"


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


def profile_traffic():
    """dram read+write bytes per launch of the sweep kernel from the committed
    ncu --set full summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "sweep_c2_ncu_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
    return world, rank, local, dist


def emit(obj):
    print(json.dumps(obj), flush=True)


# ---------------------------------------------------------------- b200 arm --

def run_b200(args):
    import torch

    import paper_2403_01778_b200 as r1
    from paper_2403_01778_b200 import _lib
    from paper_2403_01778_b200.distributed import exchange, local_dims, slab_bounds

    world, rank, local, dist = init_dist()
    torch.cuda.set_device(local)
    ctx = r1.Context(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    L = _lib.lib()
    dims = CONFIG2_DIMS
    d = len(dims)
    lo, hi = slab_bounds(dims[-1], world, rank)
    ldims = local_dims(dims, lo, hi)
    slab_elems = int(np.prod(ldims))
    first = int(np.prod(dims[:-1])) * lo

    # the rank's slab, generated in HBM (counter-based config-2 generator) in
    # torch-owned memory (16-B aligned, padded) wrapped as an r1_tensor
    a_dev = torch.empty(slab_elems + 2, dtype=torch.float64, device="cuda")
    t = r1.DeviceTensor.wrap(a_dev.data_ptr(), ldims, ctx, keepalive=a_dev)
    gdims = _lib.dims_arr(dims)
    _lib.check(L.r1_generate_config(ctx.handle, t.handle, 2, CONFIG2_SEED, _lib.u64p(gdims), d,
                                    first))
    # factors: the solver's uniform01 init (solvers.cpp:34-49), sliced for the slab
    fac_full = uniform01_factors(dims, seed=CONFIG2_SEED)
    fl = np.concatenate(fac_full[:-1] + [fac_full[-1][lo:hi]])
    fac = torch.from_numpy(fl).cuda()
    nb_local = int(sum(ldims[m] * ldims[k] for m in range(d) for k in range(m + 1, d)))
    nb = int(sum(dims[m] * dims[k] for m in range(d) for k in range(m + 1, d)))
    lblocks = torch.empty(nb_local, dtype=torch.float64, device="cuda")
    gblocks = torch.empty(nb, dtype=torch.float64, device="cuda") if world > 1 else lblocks

    def step():
        _lib.check(L.r1_build_j_device(ctx.handle, t.handle, fac.data_ptr(), lblocks.data_ptr(),
                                       None))
        if world > 1:
            exchange(lblocks, dims, world, rank, dist, gblocks)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()

    # ---- device-resident timing (value) + live kernel timing (roofline)
    L.r1x_time_kernels(ctx.handle, 1)
    ms_k = ctypes_double()
    nk = ctypes_u64()
    L.r1x_kernel_time(ctx.handle, ctypes_byref(ms_k), ctypes_byref(nk))  # reset
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
    L.r1x_kernel_time(ctx.handle, ctypes_byref(ms_k), ctypes_byref(nk))
    L.r1x_time_kernels(ctx.handle, 0)
    ms = e0.elapsed_time(e1)
    ms = max_over_ranks(ms, dist)
    kernel_ms = ms_k.value / max(1, nk.value)
    total_bytes = sweep_bytes(dims) * args.steps
    value = total_bytes / (ms * 1e-3) / 1e9

    # ---- end-to-end through the C-ABI with host buffers
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    host = torch.empty(slab_elems, dtype=torch.float64, pin_memory=True)
    host.copy_(a_dev[:slab_elems])
    fac_host = torch.from_numpy(fl).pin_memory()
    blocks_host = torch.empty(nb, dtype=torch.float64, pin_memory=True)

    def e2e_step():
        _lib.check(L.r1_tensor_copy_from_host(ctx.handle, t.handle,
                                              _lib.ctypes.cast(host.data_ptr(), _lib._dp)))
        fac.copy_(fac_host, non_blocking=True)
        step()
        blocks_host.copy_(gblocks, non_blocking=True)
        stream.synchronize()

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
    # factors go H2D and the blocks come back D2H through the same C-ABI calls
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
    h2d = 8 * int(np.prod(dims)) + 8 * sum(dims)
    d2h = 8 * nb

    # ---- time to converge (tensor resident): HOSCF and iHOSCF, tol 1e-10.  One
    # GPU: the C++ device driver; N GPUs: the slab-sharded driver (sweep per
    # rank + NCCL exchange, replicated eigen / RQI / stopping test)
    ttc = None
    if not args.skip_solve:
        from paper_2403_01778_b200.distributed import solve_distributed
        ttc = {}
        def ttc_one(alg):
            o = r1.SolveOptions(tol=1e-10, max_iters=100, seed=CONFIG2_SEED)
            runs = []
            for _ in range(3):  # first run includes one-time plan / workspace setup
                torch.cuda.synchronize()
                barrier()
                ts = time.perf_counter()
                if world == 1:
                    rep = r1.solve(alg, t, o, ctx)
                else:
                    rep = solve_distributed(alg, t, dims, o, dist, world, rank, ctx)
                torch.cuda.synchronize()
                runs.append(max_over_ranks(time.perf_counter() - ts, dist))
            return {"seconds": round(statistics.median(runs[1:]), 6),
                    "seconds_first_call": round(runs[0], 6), "iterations": rep.iterations,
                    "sweeps": rep.total_sweeps, "converged": rep.converged,
                    "lambda": rep.result.lambda_, "t_build_j": round(rep.wall_build_j(), 6),
                    "t_eig": round(rep.wall_eig(), 6)}

        for alg in ("hoscf", "ihoscf"):
            try:
                ttc[alg] = ttc_one(alg)
            except Exception as e:  # keep the sweep line even if a solve fails
                ttc[alg] = {"error": f"{type(e).__name__}: {e}"}

    # ---- the other BASELINE configs (single GPU): sweep throughput and
    # time-to-converge on device-generated inputs
    other = None
    if world == 1 and not args.skip_configs:
        del t
        a_dev = None
        torch.cuda.empty_cache()
        try:
            other = other_configs(r1, _lib, ctx, stream)
        except Exception as e:
            other = {"error": f"{type(e).__name__}: {e}"}

    # ---- CPU baseline: the compiled reference on this host (rank 0, N=1)
    cpu = None
    if world == 1 and rank == 0 and not args.skip_cpu:
        cpu = cpu_baseline(args)

    if rank == 0:
        peak, peak_kind = measured_peaks()
        achieved = level0_bytes(ldims) / (kernel_ms * 1e-3) / 1e9 if kernel_ms > 0 else None
        out = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 6),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE config 2, generated in HBM by the counter-based generator)",
            "config": {
                "workload": "C2: HOSCF TTVc sweep (all 3 NEPv blocks) of a 1000x1000x1000 fp64 "
                            "tensor, 10*u1.u2.u3 + 0.01/sqrt(n^3) N(0,1), uniform01 factors",
                "dims_reference_order": list(dims),
                "tensor_bytes": 8 * int(np.prod(dims)),
                "algorithmic_bytes_per_step": sweep_bytes(dims),
                "l2": "inputs (8 GB) far larger than L2 (126 MB); no flush needed",
                "parallelism": f"slab{world} along the slowest mode (NCCL all-reduce + all-gather)"
                               if world > 1 else "single GPU",
            },
            "roofline": {
                "bound": "hbm",
                "kernel": "sweep3_box_kernel (top-level fused pass)",
                "achieved": round(achieved, 3) if achieved else None,
                "peak": peak,
                "unit": "GB/s",
                "frac": round(achieved / peak, 4) if achieved else None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "kernel_ms_per_launch": round(kernel_ms, 6),
                "algorithmic_bytes_per_launch": level0_bytes(ldims),
                "traffic": profile_traffic(),
            },
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "path": "r1_tensor_copy_from_host (pinned) + r1_build_j_device + D2H blocks"},
            "e2e_resident": {"value": round(e2e_res_value, 3), "unit": "GB/s",
                             "h2d_bytes_per_step": 8 * sum(dims), "d2h_bytes_per_step": d2h,
                             "steps": args.steps,
                             "path": "tensor resident (one upload per solve); factors H2D + "
                                     "r1_build_j_device + blocks D2H per step"},
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
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


OTHER_CONFIGS = [
    # name, cfg, reference dims, solves: (alg, options)
    ("C1", 1, (100, 100, 100), [("hoscf", dict(tol=1e-300, max_iters=500, init="provided",
                                              scf_lambda_rtol=1e-12))]),
    ("C3", 3, (200, 200, 200, 200), [("hoscf", dict(tol=1e-300, max_iters=100, record_kkt=False))]),
    ("C4", 4, (60, 60, 60, 60, 60), [("hoscf", dict(tol=1e-10, max_iters=100)),
                                     ("ihoscf", dict(tol=1e-10, max_iters=100))]),
    ("C5", 5, (500, 2000, 4000), [("hoscf", dict(tol=1e-10, max_iters=200)),
                                  ("ihoscf", dict(tol=1e-10, max_iters=200))]),
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
                 "sweep_ms": round(ms, 4), "sweep_gbs": round(sweep_bytes(dims) / ms / 1e6, 2)}
        for alg, kw in solves:
            init = kw.pop("init", None)
            o = r1.SolveOptions(seed=cfg, **kw)
            kw["init"] = init
            if init == "provided":  # C1: normalised all-ones (BASELINE config 1)
                o.init = "provided"
                o.init_factors = [np.ones(d) for d in dims]
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
                          "sweeps": rep.total_sweeps, "converged": rep.converged,
                          "lambda": rep.result.lambda_, "t_build_j": round(rep.wall_build_j(), 6),
                          "t_eig": round(rep.wall_eig(), 6), "options": {k: v for k, v in kw.items()
                                                                         if v is not None}}
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


def max_over_ranks(v, dist):
    if dist is None:
        return v
    import torch
    x = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return float(x.item())


def ctypes_double():
    import ctypes
    return ctypes.c_double()


def ctypes_u64():
    import ctypes
    return ctypes.c_uint64()


def ctypes_byref(x):
    import ctypes
    return ctypes.byref(x)


# ------------------------------------------------------- CPU reference arm --

def _ref_sample(slices):
    """A bounded sample of config 2: the first `slices` slowest-mode slices of
    the same global tensor (bit-identical to the reference's generator), with
    the solver's initial factors."""
    from oracle import rank1_oracle as O
    dims = CONFIG2_DIMS
    n_slab = dims[0] * dims[1] * slices
    # generate only the slab: planted factors + counter-addressed noise
    u = [O.planted_factor(CONFIG2_SEED, k, dims[k]) for k in range(3)]
    noise = O.rng_gaussians(CONFIG2_SEED, 1, n_slab)
    a = np.einsum("i,j,k->ijk", u[0], u[1], u[2][:slices]).reshape(-1, order="F")
    a = 10.0 * a + (0.01 / np.sqrt(float(np.prod(dims)))) * noise
    sdims = (dims[0], dims[1], slices)
    f = uniform01_factors(dims, CONFIG2_SEED)
    f = [f[0], f[1], f[2][:slices] / np.linalg.norm(f[2][:slices])]
    return a, sdims, f


def cpu_baseline(args, steps=None, warmup=None):
    from oracle import ref
    if not ref.available():
        return {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    slices = args.cpu_slices
    a, sdims, f = _ref_sample(slices)
    reps = steps or 3
    ref.time_build_j(a, sdims, f, reps=1)  # warm
    _, secs = ref.time_build_j(a, sdims, f, reps=reps)
    gbs = sweep_bytes(sdims) * reps / float(np.sum(secs)) / 1e9
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": ref.max_threads(),
            "kind": "reference",
            "sample": f"rank1::build_j (reference, OpenMP, determinism=true) on the first {slices} "
                      f"of 1000 slowest-mode slices of config 2 ({sdims[0]}x{sdims[1]}x{slices}, "
                      f"{8 * int(np.prod(sdims)) / 1e9:.2f} GB), {reps} timed sweeps"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/librank1_ref.so is not built"})
        return
    slices = args.cpu_slices
    a, sdims, f = _ref_sample(slices)
    for _ in range(args.warmup):
        ref.time_build_j(a, sdims, f, reps=1)
    _, secs = ref.time_build_j(a, sdims, f, reps=args.steps)
    total = float(np.sum(secs))
    value = sweep_bytes(sdims) * args.steps / total / 1e9
    cores = ref.max_threads()
    sample = (f"rank1::build_j (reference C++/OpenMP, {cores} threads) on the first {slices} of 1000 "
              f"slowest-mode slices of config 2 ({8 * int(np.prod(sdims)) / 1e9:.2f} GB) per step")
    emit({
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE config 2 slab, reference-identical generator)",
        "config": {"workload": "C2: HOSCF TTVc sweep (rank1::build_j), CPU reference",
                   "dims_reference_order": list(sdims)},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    })


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-slices", type=int, default=200)
    ap.add_argument("--skip-solve", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-configs", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
