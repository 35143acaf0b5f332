#!/usr/bin/env python3
"""Summarise an ncu capture of the sweep for profiles/: the `--set full`
report of the top-level box kernel plus the per-launch list of one bench run.

    python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT.json [--round N] [--command CMD]
"""
import argparse
import csv
import json
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_requests_srcunit_tex_op_read.sum",
    "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_active.avg", "sm__cycles_active.max",
    "sm__cycles_active.min", "sm__cycles_elapsed.avg",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ik, im, iv, iu = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = defaultdict(lambda: defaultdict(list))
    for r in rows[start + 1:]:
        if len(r) < len(h):
            continue
        name = r[ik].split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("r1::", "")
        val = float(r[iv].replace(",", ""))
        if r[iu] in ("nsecond", "ns"):
            val *= 1e-3  # -> us
        elif r[iu] == "usecond":
            pass
        elif r[iu] in ("msecond", "ms"):
            val *= 1e3
        agg[name][r[im]].append(val)
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("launch_csv")
    ap.add_argument("out")
    ap.add_argument("--round", type=int, default=1)
    ap.add_argument("--command", default="")
    ap.add_argument("--algorithmic-bytes", type=float, default=8024024000)
    a = ap.parse_args()
    d = raw(a.report)
    full = {k: f"{d[k][0]} {d[k][1]}".strip() for k in KEYS if k in d}
    rd = float(d["dram__bytes_read.sum"][0]) * UNIT.get(d["dram__bytes_read.sum"][1], 1.0)
    wr = float(d["dram__bytes_write.sum"][0]) * UNIT.get(d["dram__bytes_write.sum"][1], 1.0)
    agg = launches(a.launch_csv)
    sweep_kernels = {k: v for k, v in agg.items() if "gen_kernel" not in k}
    tot = sum(sum(v["gpu__time_duration.sum"]) / len(v["gpu__time_duration.sum"])
              for v in sweep_kernels.values())
    per = {}
    for k, v in sweep_kernels.items():
        t = v["gpu__time_duration.sum"]
        n = len(t)
        per[k] = {"launches_in_run": n, "us_per_launch": round(sum(t) / n, 3),
                  "share_of_sweep_time": round(sum(t) / n / tot, 4),
                  "dram_read_GB_per_launch": round(sum(v["dram__bytes_read.sum"]) / n / 1e9, 4),
                  "dram_write_GB_per_launch": round(sum(v["dram__bytes_write.sum"]) / n / 1e9, 4)}
    out = {"round": a.round, "command": a.command,
           "kernel": "sweep3_box_kernel<4,4,15,1> (C2 1000^3, top-level fused pass)",
           "ncu_set_full": full, "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd,
           "dram_write_bytes": wr, "algorithmic_bytes_per_launch": a.algorithmic_bytes,
           "traffic_over_algorithmic": round((rd + wr) / a.algorithmic_bytes, 4),
           "launch_list_per_sweep": per,
           "note": "ncu times are cold-cache and serialised (--clock-control none); the kernel's "
                   "share of the sweep is what must agree with the live CUDA-event timing in bench.py"}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("dram_bytes_per_launch", "traffic_over_algorithmic")}))


if __name__ == "__main__":
    main()
