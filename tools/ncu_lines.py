#!/usr/bin/env python3
"""Per-source-line warp-stall samples from an ncu report captured with
--import-source on (needs -lineinfo): ncu_lines.py report.ncu-rep [top_n]"""
import csv
import io
import os
import subprocess
import sys


def main(rep, top=30):
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
        if hdr is None or len(r) != len(hdr) or r[2] != "-":
            continue   # keep source-line rows (aggregates), skip per-SASS rows
        try:
            data.append((int(r[4] or 0), f"{fname}:{r[0]}", r[1].strip()[:100]))
        except ValueError:
            pass
    tot = sum(d[0] for d in data) or 1
    for s, ln, text in sorted(data, reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}%  {ln:>22}  {text}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
