#!/usr/bin/env python3
"""Summarise an ncu `--set full --import-source on` capture of one kernel for
profiles/: launch shape, duration, instruction / issue / stall metrics and the
source lines holding the most warp-stall samples.

    python tools/ncu_kernel_summary.py REPORT.ncu-rep OUT.json [--command CMD] [--note TEXT]
"""
import argparse
import collections
import csv
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__cycles_active.avg",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(report, *args):
    return subprocess.run(["ncu", "-i", report, *args], capture_output=True, text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--command", default="")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rows = list(csv.reader(ncu(a.report, "--page", "raw", "--csv").splitlines()))
    h, u = rows[0], rows[1]
    launches = []
    for v in rows[2:]:
        d = {h[i]: (v[i], u[i]) for i in range(len(h))}
        m = {k: f"{d[k][0]} {d[k][1]}".strip() for k in KEYS if k in d}
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
                  round(float(d[k][0].replace(",", "") or 0), 3)
                  for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("ratio")}
        m["stalls_per_issue"] = {k: x for k, x in sorted(stalls.items(), key=lambda t: -t[1]) if x >= 0.05}
        m["kernel"] = d.get("Kernel Name", ("", ""))[0]
        launches.append(m)
    # source lines by warp-stall samples (innermost frame of each SASS line)
    src = list(csv.reader(ncu(a.report, "--page", "source", "--csv", "--print-source", "cuda,sass").splitlines()))
    per_line, text, cur = collections.Counter(), {}, None
    for x in src:
        if len(x) < 5 or x[0] == "Line No":
            continue
        if x[0].isdigit():
            cur = int(x[0])
            text[cur] = x[1].strip()
        elif x[2] and cur is not None:
            try:
                per_line[cur] += float(x[4] or 0)
            except ValueError:
                pass
    tot = sum(per_line.values()) or 1.0
    top = [{"line": ln, "share": round(c / tot, 4), "source": text.get(ln, "")[:120]}
           for ln, c in per_line.most_common(15)]
    json.dump({"command": a.command, "note": a.note, "launches": launches,
               "top_stall_source_lines": top}, open(a.out, "w"), indent=1)
    print(json.dumps(launches[0], indent=1)[:1500])


if __name__ == "__main__":
    main()
