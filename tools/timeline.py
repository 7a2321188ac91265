#!/usr/bin/env python3
"""Concurrent kernel timeline of one FW solve (CUPTI via torch.profiler: real start/end times on
every stream, unlike ncu's serialised replay).  Prints per-kernel-name totals, the busy time of the
union of all kernels, the gaps, and per-round spans; writes the raw events as CSV.
usage: tools/timeline.py n [rho] [out.csv] [block] [host|-] [i32|f32c]"""
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402

n = int(sys.argv[1])
rho = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = sys.argv[3] if len(sys.argv) > 3 else None
block = int(sys.argv[4]) if len(sys.argv) > 4 else 0
host = len(sys.argv) > 5 and sys.argv[5] == "host"   # also list the CUDA runtime calls (host side)
kind = sys.argv[6] if len(sys.argv) > 6 else "i32"   # i32 | f32c (continuous fp32 weights)
if kind == "f32c":
    h = torch.from_numpy(ap.continuous_costs(ap.GenParams(n, rho, 100, 7 + n))).cuda()
else:
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, 7 + n), np.int32)).cuda()
for _ in range(5):
    ap.solve(h, block=block)
torch.cuda.synchronize()
acts = [ProfilerActivity.CUDA] + ([ProfilerActivity.CPU] if host else [])
with profile(activities=acts) as prof:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = ap.solve(h, block=block)
    e1.record()
    torch.cuda.synchronize()
ev, hev = [], []
for e in prof.events():
    if e.device_type.name != "CUDA":
        if host and e.name.startswith("cuda"):
            hev.append((e.time_range.start, e.time_range.end, e.name[:60]))
        continue
    if ("Memcpy" in e.name or "Memset" in e.name) and not host:
        continue
    ev.append((e.time_range.start, e.time_range.end, e.name[:60]))
ev.sort()
t0 = ev[0][0]
tot = defaultdict(lambda: [0, 0.0])
for s, t, nm in ev:
    tot[nm][0] += 1
    tot[nm][1] += t - s
busy, cur_s, cur_t = 0.0, None, None
for s, t, _ in ev:
    if cur_t is None or s > cur_t:
        if cur_t is not None:
            busy += cur_t - cur_s
        cur_s, cur_t = s, t
    else:
        cur_t = max(cur_t, t)
busy += cur_t - cur_s
span = ev[-1][1] - t0
print(f"n={n} tier={r.info['tier']} event {e0.elapsed_time(e1):.3f} ms; kernels span {span / 1e3:.3f} ms, "
      f"union busy {busy / 1e3:.3f} ms, idle {(span - busy) / 1e3:.3f} ms, {len(ev)} launches")
for nm, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"  {d / 1e3:8.3f} ms  {c:5d}x  avg {d / c:7.2f} us  {nm}")
if host:   # merged device / host listing, times relative to the first device op
    for s_, t_, nm in sorted([(s, t, "D " + nm) for s, t, nm in ev] + [(s, t, "H " + nm) for s, t, nm in hev]):
        print(f"{s_ - t0:9.1f} {t_ - s_:8.1f}  {nm}")
if out:
    with open(out, "w") as f:
        f.write("start_us,end_us,name\n")
        for s, t, nm in ev:
            f.write(f"{s - t0:.3f},{t - t0:.3f},{nm}\n")
