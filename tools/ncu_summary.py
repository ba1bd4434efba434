"""Summarise an `ncu --set full` report into profiles/ (committed evidence).

    python tools/ncu_summary.py <report.ncu-rep> <config-name> <round-tag>

Writes profiles/<tag>_<config>_<kernel>.txt (key counters) and merges
traffic_bytes_per_launch[<config>] into profiles/ncu_summary.json (read by bench.py)."""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

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
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def main():
    rep, cfg, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        rec = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        kname = rec.get("Kernel Name", ("?", ""))[0]
        got = {k: rec[k] for k in KEYS if k in rec}
        rb = float(got["dram__bytes_read.sum"][0].replace(",", "")) * SCALE.get(got["dram__bytes_read.sum"][1], 1)
        wb = float(got["dram__bytes_write.sum"][0].replace(",", "")) * SCALE.get(got["dram__bytes_write.sum"][1], 1)
        out.append((kname, got, rb + wb))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    kname, got, traffic = out[0]
    short = "k_accumulate" if "accumulate" in kname else ("k_segments" if "segments" in kname else "kernel")
    path = os.path.join(ROOT, "profiles", f"{tag}_{cfg}_{short}.txt")
    with open(path, "w") as fh:
        fh.write(f"# ncu --set full --clock-control none, {kname}, config {cfg}\n")
        fh.write(f"# source report: {os.path.basename(rep)}\n")
        for k in KEYS:
            if k in got:
                fh.write(f"{k:70s} {got[k][0]:>20s} {got[k][1]}\n")
        fh.write(f"{'traffic_bytes (dram read + write)':70s} {traffic:>20.0f} byte\n")
    sj = os.path.join(ROOT, "profiles", "ncu_summary.json")
    s = json.load(open(sj)) if os.path.exists(sj) else {}
    s.setdefault("traffic_bytes_per_launch", {})[cfg] = traffic
    s.setdefault("source", {})[cfg] = os.path.basename(path)
    json.dump(s, open(sj, "w"), indent=1, sort_keys=True)
    print(open(path).read())


if __name__ == "__main__":
    main()
