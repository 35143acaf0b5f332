"""Experiment / scaling harness with the reference's CSV formats
(proj/include/rank1/experiment.hpp:12-87, src/experiment.cpp:48-233), on the
device: the tensor is generated in HBM (r1_generate) or streamed from a .dt1
file straight into HBM (r1_tensor_read_dt1), every (algorithm, seed) cell is a
device solve, and the phase columns are the solver's CUDA-event phase times
(sweep = phase_j_s, eigen step = phase_eig_s).

    python -m paper_2403_01778_b200.experiment --generator exp --algos hoscf,ihoscf \\
        --seeds 10 --csv runs.csv
    python -m paper_2403_01778_b200.experiment --generator file --input a.dt1 --scaling
"""
from __future__ import annotations

import argparse
import math
import sys
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import (Context, DeviceTensor, InvalidArgument, SolveOptions, _lib, check, default_context,
               dims_arr, read_dt1, solve, u64p)

DEFAULT_DIMS = {"gaussian": [10, 10, 10], "exp": [30, 30, 30], "arcsin": [20, 20, 20, 20],
                "tan": [10, 10, 10, 10, 10]}  # generators.cpp:101-107


@dataclass
class ExperimentSpec:
    """experiment.hpp:12-25 (threads: the scaling list; on the device every run
    uses the whole GPU, the column records the requested value)."""
    generator: str = "gaussian"
    dims: List[int] = field(default_factory=list)
    input_path: str = ""
    tensor_seed: int = 0
    base_seed: int = 0
    seeds: int = 50
    algorithms: List[str] = field(default_factory=lambda: ["hoscf"])
    opts: SolveOptions = field(default_factory=SolveOptions)
    threads: List[int] = field(default_factory=lambda: [1])
    scaling_iters: int = 10
    parallel_cells: bool = True


@dataclass
class RunRow:
    generator: str = ""
    dims: str = ""
    algo: str = ""
    seed: int = 0
    lambda_: float = 0.0
    rho: float = 0.0
    iters: int = 0
    converged: bool = False
    wall_s: float = 0.0
    phase_j_s: float = 0.0
    phase_eig_s: float = 0.0


@dataclass
class AlgoSummary:
    algo: str = ""
    runs: int = 0
    converged: int = 0
    mean_lambda: float = 0.0
    std_lambda: float = 0.0
    mean_rho: float = 0.0
    std_rho: float = 0.0
    mean_iters: float = 0.0
    std_iters: float = 0.0


@dataclass
class ExperimentResult:
    rows: List[RunRow] = field(default_factory=list)
    summaries: List[AlgoSummary] = field(default_factory=list)


@dataclass
class ScalingRow:
    generator: str = ""
    dims: str = ""
    threads: int = 0
    iters: int = 0
    phase_j_s: float = 0.0
    phase_eig_s: float = 0.0
    other_s: float = 0.0
    j_fraction: float = 0.0
    lambda_: float = 0.0
    lambda_dev_vs_first: float = 0.0


def format_dims(dims) -> str:
    """experiment.cpp:48-55."""
    return "x".join(str(int(d)) for d in dims)


def parse_dims(text: str) -> List[int]:
    """experiment.cpp:57-70: 'AxBxC' or 'A,B,C'."""
    delim = "x" if "x" in text else ","
    dims = []
    for tok in text.split(delim):
        if not tok:
            continue
        v = int(tok)
        if v < 1:
            raise InvalidArgument("parse_dims: dims must be >= 1")
        dims.append(v)
    if not dims:
        raise InvalidArgument("parse_dims: empty dims")
    return dims


def make_tensor(spec: ExperimentSpec, ctx: Optional[Context] = None) -> DeviceTensor:
    """experiment.cpp:72-79, producing a device tensor: .dt1 straight into
    HBM, or the named generator run on the device."""
    ctx = ctx or default_context()
    if spec.generator == "file":
        if not spec.input_path:
            raise InvalidArgument("make_tensor: file generator needs an input path")
        return read_dt1(spec.input_path, ctx)
    if spec.generator not in DEFAULT_DIMS:
        raise InvalidArgument("unknown generator: " + spec.generator)
    dims = list(spec.dims) or DEFAULT_DIMS[spec.generator]
    d = dims_arr(dims)
    h = _lib.ctypes.c_void_p()
    check(_lib.lib().r1_tensor_create(ctx.handle, u64p(d), len(dims), _lib.ctypes.byref(h)))
    t = DeviceTensor(ctx, h, dims)
    check(_lib.lib().r1_generate(ctx.handle, t.handle, spec.generator.encode(),
                                 _lib.ctypes.c_uint64(spec.tensor_seed)))
    return t


def _frobenius(t: DeviceTensor) -> float:
    out = _lib.ctypes.c_double()
    check(_lib.lib().r1_tensor_frobenius(t.ctx.handle, t.handle, _lib.ctypes.byref(out)))
    return out.value


def _stats(xs):
    """experiment.cpp:29-43 (sample standard deviation)."""
    if not xs:
        return 0.0, 0.0
    mean = sum(xs) / len(xs)
    sd = 0.0
    if len(xs) > 1:
        sd = math.sqrt(sum((x - mean) * (x - mean) for x in xs) / (len(xs) - 1))
    return mean, sd


def run_experiment(spec: ExperimentSpec, a: Optional[DeviceTensor] = None,
                   ctx: Optional[Context] = None) -> ExperimentResult:
    """experiment.cpp:81-159: every (algorithm, seed) cell, algorithm-major.
    Cells run one after another: each device solve already uses the whole GPU."""
    if spec.seeds == 0:
        raise InvalidArgument("run_experiment: seeds must be >= 1")
    if not spec.algorithms:
        raise InvalidArgument("run_experiment: no algorithms selected")
    a = a if a is not None else make_tensor(spec, ctx)
    a_norm = _frobenius(a)
    dims_text = format_dims(a.dims)
    res = ExperimentResult()
    errors = []
    for algo in spec.algorithms:
        for si in range(spec.seeds):
            o = SolveOptions(**{**spec.opts.__dict__, "seed": spec.base_seed + si})
            row = RunRow(spec.generator, dims_text, algo, o.seed)
            try:
                rep = solve(algo, a, o, a.ctx)
                row.lambda_ = rep.result.lambda_
                row.rho = abs(rep.result.lambda_) / a_norm if a_norm > 0 else 0.0
                row.iters = rep.iterations
                row.converged = rep.converged
                row.wall_s = rep.wall_total()
                row.phase_j_s = rep.wall_build_j()
                row.phase_eig_s = rep.wall_eig()
            except Exception as e:  # experiment.cpp:126-128
                errors.append(str(e))
            res.rows.append(row)
    if errors:
        raise RuntimeError("run_experiment: " + errors[0])
    for ai, algo in enumerate(spec.algorithms):
        rows = res.rows[ai * spec.seeds:(ai + 1) * spec.seeds]
        s = AlgoSummary(algo, len(rows), sum(1 for r in rows if r.converged))
        s.mean_lambda, s.std_lambda = _stats([r.lambda_ for r in rows])
        s.mean_rho, s.std_rho = _stats([r.rho for r in rows])
        s.mean_iters, s.std_iters = _stats([float(r.iters) for r in rows])
        res.summaries.append(s)
    return res


def _g(v, spec):
    return spec % v


def experiment_csv(rows: List[RunRow], zero_timings: bool) -> str:
    """experiment.cpp:165-181 (%.10g values, %.3g times)."""
    out = "generator,dims,algo,seed,lambda,rho,iters,converged,wall_s,phase_j_s,phase_eig_s\n"
    for r in rows:
        out += f"{r.generator},{r.dims},{r.algo},{r.seed},"
        out += _g(r.lambda_, "%.10g") + "," + _g(r.rho, "%.10g") + ","
        out += f"{r.iters},{'1' if r.converged else '0'},"
        if zero_timings:
            out += "0,0,0\n"
        else:
            out += ",".join(_g(x, "%.3g") for x in (r.wall_s, r.phase_j_s, r.phase_eig_s)) + "\n"
    return out


def summary_table(summaries: List[AlgoSummary]) -> str:
    """experiment.cpp:183-193."""
    out = "algo         lambda              rho                 iters           conv\n"
    for s in summaries:
        out += "%-12s %9.4f +- %-7.4f %7.4f +- %-7.4f %7.2f +- %-6.2f %d/%d\n" % (
            s.algo, s.mean_lambda, s.std_lambda, s.mean_rho, s.std_rho, s.mean_iters, s.std_iters,
            s.converged, s.runs)
    return out


def run_scaling(spec: ExperimentSpec, a: Optional[DeviceTensor] = None,
                ctx: Optional[Context] = None) -> List[ScalingRow]:
    """experiment.cpp:195-222: fixed-iteration HOSCF runs (tol 1e-300, no KKT
    record), phase split from the device events, lambda agreement vs the first."""
    if not spec.threads:
        raise InvalidArgument("run_scaling: empty thread list")
    a = a if a is not None else make_tensor(spec, ctx)
    rows, first = [], 0.0
    for i, th in enumerate(spec.threads):
        o = SolveOptions(**{**spec.opts.__dict__, "threads": th, "seed": spec.base_seed,
                            "max_iters": spec.scaling_iters, "tol": 1e-300, "record_kkt": False})
        rep = solve("hoscf", a, o, a.ctx)
        tot = rep.wall_total()
        row = ScalingRow(spec.generator, format_dims(a.dims), th, rep.iterations, rep.wall_build_j(),
                         rep.wall_eig())
        row.other_s = tot - row.phase_j_s - row.phase_eig_s
        row.j_fraction = row.phase_j_s / tot if tot > 0 else 0.0
        row.lambda_ = rep.result.lambda_
        if i == 0:
            first = row.lambda_
        row.lambda_dev_vs_first = abs(row.lambda_ - first)
        rows.append(row)
    return rows


def scaling_csv(rows: List[ScalingRow]) -> str:
    """experiment.cpp:224-233."""
    out = ("generator,dims,algo,threads,iters,phase_j_s,phase_eig_s,other_s,j_fraction,lambda,"
           "lambda_dev_vs_first\n")
    for r in rows:
        out += f"{r.generator},{r.dims},hoscf,{r.threads},{r.iters},"
        out += ",".join(_g(x, "%.3g") for x in (r.phase_j_s, r.phase_eig_s, r.other_s)) + ","
        out += "%.4f" % r.j_fraction + "," + _g(r.lambda_, "%.10g") + "," + \
            _g(r.lambda_dev_vs_first, "%.10g") + "\n"
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--generator", default="gaussian")
    ap.add_argument("--dims", default="")
    ap.add_argument("--input", default="")
    ap.add_argument("--tensor-seed", type=int, default=0)
    ap.add_argument("--base-seed", type=int, default=0)
    ap.add_argument("--seeds", type=int, default=50)
    ap.add_argument("--algos", default="hoscf")
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--max-iters", type=int, default=500)
    ap.add_argument("--scaling", action="store_true")
    ap.add_argument("--threads", default="1")
    ap.add_argument("--scaling-iters", type=int, default=10)
    ap.add_argument("--zero-timings", action="store_true")
    ap.add_argument("--csv", default="")
    a = ap.parse_args(argv)
    spec = ExperimentSpec(generator=a.generator, dims=parse_dims(a.dims) if a.dims else [],
                          input_path=a.input, tensor_seed=a.tensor_seed, base_seed=a.base_seed,
                          seeds=a.seeds, algorithms=a.algos.split(","),
                          opts=SolveOptions(tol=a.tol, max_iters=a.max_iters),
                          threads=[int(x) for x in a.threads.split(",")],
                          scaling_iters=a.scaling_iters)
    if a.scaling:
        text = scaling_csv(run_scaling(spec))
    else:
        r = run_experiment(spec)
        text = experiment_csv(r.rows, a.zero_timings)
        sys.stderr.write(summary_table(r.summaries))
    if a.csv:
        with open(a.csv, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)


if __name__ == "__main__":
    main()
