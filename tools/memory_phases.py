#!/usr/bin/env python3
"""Summarise the HBM-bound kernels of one FW solve from an ncu capture
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum):
achieved DRAM GB/s against the measured HBM peak (MEASURED_PEAKS.json).
usage: tools/memory_phases.py capture.csv out.txt"""

from __future__ import annotations

import collections
import csv
import json
import sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    ii, ik, im, iv, iu = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[im]] = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        names[r[ii]] = r[ik].split("(")[0]
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, m in per.items():
        name = names[lid]
        if not any(x in name for x in ("scan", "to_store", "from_store", "max_finite", "copy_idx", "prep_pair")):
            continue
        a = agg[name]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    lines = [f"# HBM-bound kernels of one n=16384 FW solve (ncu, serialised; peak {peak} GB/s measured copy)",
             f"{'kernel':40s} {'launches':>8s} {'ms':>8s} {'GB':>8s} {'GB/s':>8s} {'of peak':>8s}"]
    for name, (cnt, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = b / t / 1e9 if t else 0.0
        lines.append(f"{name[:40]:40s} {cnt:8d} {t * 1e3:8.3f} {b / 1e9:8.3f} {gbs:8.0f} {gbs / peak:8.2f}")
    Path(sys.argv[2]).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
