#!/usr/bin/env python3
"""Warp-stall samples per CUDA source line of an ncu --set full report (run here, on reports
gpurun brings back):  ncu_lines.py REPORT.ncu-rep [top]   -> the lines with the most samples,
their instruction counts and the dominant stall reasons."""

from __future__ import annotations

import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    iins = hdr.index("Instructions Executed")
    stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]
    recs = []
    for r in rows[hi + 1:]:
        if len(r) <= isamp or not r[0].isdigit():
            continue
        if len(r) != len(hdr):   # a source line with unescaped quotes: metrics are the tail
            r = r[:2] + r[len(r) - len(hdr) + 2:]
        s = int(r[isamp] or 0)
        if not s:
            continue
        st = sorted(((int(r[i] or 0), h[6:]) for i, h in stall_cols), reverse=True)[:3]
        recs.append((s, int(r[0]), int(r[iins] or 0), r[1].strip()[:70], st))
    tot = sum(x[0] for x in recs)
    print(f"total samples {tot}")
    for s, ln, ins, src, st in sorted(recs, reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}% L{ln:<5d} inst {ins:>10d}  {src:70s} {' '.join(f'{h}:{v}' for v, h in st)}")


if __name__ == "__main__":
    main()
