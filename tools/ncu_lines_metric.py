#!/usr/bin/env python3
"""Per-source-line value of one ncu source-page metric column (default
'L1 Wavefronts Shared'): ncu_lines_metric.py report.ncu-rep [top_n] [column]"""
import csv
import io
import os
import subprocess
import sys


def main(rep, top=25, col="L1 Wavefronts Shared"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, data = "?", None, []
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or r[2] != "-" or col not in hdr:
            continue
        try:
            data.append((float(r[hdr.index(col)] or 0), f"{fname}:{r[0]}", r[1].strip()[:100]))
        except ValueError:
            pass
    tot = sum(d[0] for d in data) or 1
    print(f"total {col}: {tot:.4g}")
    for s, ln, text in sorted(data, reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}%  {ln:>22}  {text}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         sys.argv[3] if len(sys.argv) > 3 else "L1 Wavefronts Shared")
