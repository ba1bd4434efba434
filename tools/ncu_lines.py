"""Per-source-line warp-instruction counts and stall samples from an ncu report.

    python tools/ncu_lines.py <report.ncu-rep> [top]

Reads `ncu -i --page source --csv --print-source=cuda,sass`: rows with a line number carry
the per-line aggregates (instructions executed, warp-stall samples)."""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    out, fname, hdr = [], "?", None
    for row in csv.reader(raw.splitlines()):
        if not row:
            continue
        if row[0] in ("File Path", "File Name"):
            fname = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0]:
            continue
        rec = dict(zip(hdr, row))
        try:
            ie = int(rec.get("Instructions Executed") or 0)
            smp = int(rec.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            continue
        if ie or smp:
            out.append((ie, smp, fname, row[0], row[1].strip()[:90]))
    tot_i = sum(o[0] for o in out) or 1
    tot_s = sum(o[1] for o in out) or 1
    print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
    for ie, smp, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"{100*ie/tot_i:6.2f}% inst {100*smp/tot_s:6.2f}% smp  {f}:{ln:5s} {src}")


if __name__ == "__main__":
    main()
