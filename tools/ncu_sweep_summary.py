#!/usr/bin/env python3
"""Summarise an `ncu --set full` capture holding the kernels of ONE sweep (box
kernel + second stage) for profiles/: DRAM bytes per kernel and per sweep, the
FP64 pipe / issue utilisation and the warp instructions per warp DFMA.

    python tools/ncu_sweep_summary.py REPORT.ncu-rep OUT.json --dims 500 2000 4000 --config "C5 ..." --command "ncu ..."
"""
import argparse
import csv
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__inst_executed_pipe_fp64.sum"]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--dims", type=int, nargs="+", required=True)
    ap.add_argument("--config", default="")
    ap.add_argument("--command", default="")
    ap.add_argument("--round", type=int, default=2)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    kernels = []
    total = 0.0
    for v in rows[2:]:
        rec = {h[i]: (v[i], u[i]) for i in range(len(h))}
        m = {}
        for k in KEYS:
            if k in rec and rec[k][0] != "":
                m[k] = {"value": float(rec[k][0].replace(",", "")), "unit": rec[k][1]}
        dram = sum(m[k]["value"] * UNIT.get(m[k]["unit"], 1.0)
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
        total += dram
        kernels.append({"kernel": rec["Kernel Name"][0], "metrics": m, "dram_bytes": dram})
    n = 1
    for d in a.dims:
        n *= d
    nb = sum(a.dims[i] * a.dims[j] for i in range(len(a.dims)) for j in range(i + 1, len(a.dims)))
    alg = 8 * n + 8 * nb + 8 * sum(a.dims)
    box = next((k for k in kernels if "sweep3_box" in k["kernel"]), None)
    ratio = None
    if box:
        ratio = round(box["metrics"]["smsp__inst_executed.sum"]["value"] / (3.0 * n / 32.0), 2)
    json.dump({"config": a.config, "command": a.command, "round": a.round, "kernels": kernels,
               "dram_bytes_per_sweep": total, "algorithmic_bytes_per_sweep": alg,
               "traffic_over_algorithmic": round(total / alg, 4),
               "warp_inst_per_useful_warp_dfma_box": ratio,
               "note": "ncu per-launch times are cold-cache / serialised; traffic = DRAM read + write of the "
                       "kernels of one sweep; useful warp DFMAs = 3 per tensor element / 32"}, open(a.out, "w"),
              indent=1)
    print(a.out, "traffic/alg", round(total / alg, 4), "inst/dfma", ratio)


if __name__ == "__main__":
    main()
