#!/usr/bin/env python3
"""Summarise ncu captures for profiles/ (run here, on the reports gpurun brings back).

  ncu_summary.py kernel REPORT.ncu-rep UPDATES OUT.txt [OUT.json]
      --set full capture of one min-plus launch: speed-of-light, pipes, occupancy, stalls,
      SASS opcode mix; UPDATES = algorithmic min-plus updates of that launch.
  ncu_summary.py launches LAUNCHES.csv OUT.txt
      launch list (--metrics gpu__time_duration.sum): time share per kernel.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True, check=True).stdout


def kernel(rep, updates, out_txt, out_json=None):
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    d = {h: v for h, v in zip(raw[0], raw[2])}
    u = {h: v for h, v in zip(raw[0], raw[1])}
    keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct"]
    stall = sorted((k for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                   key=lambda k: -float(d[k] or 0))
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hdr = src[1]
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    ops = collections.Counter()
    for r in src[2:]:
        try:
            n = int(r[ia])
        except (ValueError, IndexError):
            continue
        toks = r[isrc].split()
        if toks:
            ops[toks[1] if toks[0].startswith("@") else toks[0]] += n
    tot = sum(ops.values())
    ms = float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "us" else 1.0)
    if u["gpu__time_duration.sum"] == "ns":
        ms = float(d["gpu__time_duration.sum"]) * 1e-6
    rate = updates / (ms * 1e-3)

    def to_bytes(k):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[k]]
        return float(d[k]) * scale

    traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    lines = [f"# ncu --set full --clock-control none, one launch ({rep.split('/')[-1]})"]
    lines += [f"{k:70s} {d.get(k, '')} {u.get(k, '')}" for k in keys]
    lines.append(f"{'algorithmic min-plus updates of the launch':70s} {updates:.4g}")
    lines.append(f"{'achieved (updates / duration)':70s} {rate / 1e12:.2f} T upd/s "
                 f"= {rate / 37.07e12:.3f} of the 37.07 T VIADDMNMX.U16x2 issue ceiling")
    lines.append(f"{'DRAM traffic (read + write)':70s} {traffic / 1e9:.3f} GB "
                 f"({traffic / updates * 1e3:.4f} B per 1000 updates)")
    lines.append("\n# warp stall reasons (per issued instruction)")
    lines += [f"  {k[34:-23]:40s} {float(d[k]):.3f}" for k in stall[:10]]
    lines.append(f"\n# SASS opcode mix ({tot:.4g} warp instructions)")
    lines += [f"  {op:30s} {c:14d} {100 * c / tot:6.2f}%" for op, c in ops.most_common(25)]
    open(out_txt, "w").write("\n".join(lines) + "\n")
    if out_json:
        json.dump({"kernel": d["Kernel Name"], "report": rep.split("/")[-1], "duration_ms": ms, "updates": updates,
                   "achieved_T": rate / 1e12, "frac_of_dpx_ceiling": rate / 37.07e12,
                   "dram_bytes_read": to_bytes("dram__bytes_read.sum"),
                   "dram_bytes_write": to_bytes("dram__bytes_write.sum"), "traffic_bytes": traffic},
                  open(out_json, "w"), indent=1)
    print("\n".join(lines[:25]))


def launches(path, out_txt):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    iu = hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1.0)
        name = r[ik].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list {path.split('/')[-1]}: {sum(v[0] for v in agg.values())} launches, "
             f"{tot:.1f} ms serialised (cold cache; compare shares, not absolutes)",
             f"{'kernel':60s} {'launches':>9s} {'ms':>10s} {'share':>7s}"]
    for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:60]:60s} {n:9d} {ms:10.2f} {100 * ms / tot:6.1f}%")
    open(out_txt, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:15]))


if __name__ == "__main__":
    if sys.argv[1] == "kernel":
        kernel(sys.argv[2], float(sys.argv[3]), sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
