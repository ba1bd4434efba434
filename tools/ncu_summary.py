"""Summarise an `ncu --set full` report into profiles/ (committed evidence).

    python tools/ncu_summary.py <report.ncu-rep> <config-name> <round-tag> [--kernel REGEX] [--dominant]

Writes profiles/<tag>_<config>_<kernel>.txt (key counters and the warp-stall breakdown of the first
kernel in the report whose name matches REGEX; the file is named after that kernel). With
--dominant, also records the kernel's dram read+write bytes per launch as
traffic_bytes_per_launch[<config>] in profiles/ncu_summary.json (read by bench.py) with the
summary file as its source."""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]
STALL = "smsp__average_warps_issue_stalled_"
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def short_name(kname: str) -> str:
    m = re.search(r"(k_\w+)", kname)
    return m.group(1) if m else "kernel"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("config")
    ap.add_argument("tag")
    ap.add_argument("--kernel", default=".")
    ap.add_argument("--dominant", action="store_true")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    pick = None
    for vals in rows[2:]:
        rec = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        kname = rec.get("Kernel Name", ("?", ""))[0]
        if re.search(a.kernel, kname):
            pick = (kname, rec)
            break
    if pick is None:
        raise SystemExit(f"no kernel matching {a.kernel!r} in {a.report}")
    kname, rec = pick
    got = {k: rec[k] for k in KEYS if k in rec}

    def val(k):
        v, u = rec[k]
        return float(v.replace(",", "")) * SCALE.get(u, 1.0)

    traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    stalls = []
    for k in rec:
        if k.startswith(STALL) and k.endswith("_per_issue_active.ratio"):
            try:
                v = float(rec[k][0].replace(",", ""))
            except ValueError:
                continue
            if v >= 0.05:
                stalls.append((v, k[len(STALL):-len("_per_issue_active.ratio")]))
    short = short_name(kname)
    path = os.path.join(ROOT, "profiles", f"{a.tag}_{a.config}_{short}.txt")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        fh.write(f"# ncu --set full --clock-control none, {kname}, config {a.config}\n")
        fh.write(f"# source report: {os.path.basename(a.report)}\n")
        for k in KEYS:
            if k in got:
                fh.write(f"{k:70s} {got[k][0]:>20s} {got[k][1]}\n")
        fh.write(f"{'traffic_bytes (dram read + write)':70s} {traffic:>20.0f} byte\n")
        fh.write("# warp stalls per issued instruction (>= 0.05)\n")
        for v, name in sorted(stalls, reverse=True):
            fh.write(f"  {name:40s} {v:8.3f}\n")
    if a.dominant:
        sj = os.path.join(ROOT, "profiles", "ncu_summary.json")
        s = json.load(open(sj)) if os.path.exists(sj) else {}
        s.setdefault("traffic_bytes_per_launch", {})[a.config] = traffic
        s.setdefault("source", {})[a.config] = os.path.basename(path)
        json.dump(s, open(sj, "w"), indent=1, sort_keys=True)
    print(open(path).read())


if __name__ == "__main__":
    main()
