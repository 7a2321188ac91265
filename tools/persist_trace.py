#!/usr/bin/env python3
"""Critical path of the persistent small-n FW schedule from an APSP_PERSIST_TRACE CSV.
usage: tools/persist_trace.py trace.csv   (run here or on the box)"""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(open(sys.argv[1])))
t0 = min(int(r["claim"]) for r in rows)
kinds = {0: "close", 1: "row", 2: "col", 3: "upd", 4: "uclose"}
dur = defaultdict(list)
wait = defaultdict(list)
for r in rows:
    k = kinds[int(r["kind"])]
    dur[k].append((int(r["done"]) - int(r["ready"])) / 1e3)
    wait[k].append((int(r["ready"]) - int(r["claim"])) / 1e3)
end = max(int(r["done"]) for r in rows)
print(f"tasks {len(rows)}  span {(end - t0) / 1e3:.1f} us  SMs used {len({r['sm'] for r in rows})}")
for k in dur:
    d, w = dur[k], wait[k]
    print(f"{k:6s} n={len(d):6d} run mean {sum(d) / len(d):7.2f} us max {max(d):7.2f}  wait mean {sum(w) / len(w):7.2f} us")
closes = sorted((int(r["K"]), (int(r["ready"]) - t0) / 1e3, (int(r["done"]) - t0) / 1e3) for r in rows if r["kind"] in ("0", "4"))
print("closures (K, start us, end us):", [(k, round(a, 1), round(b, 1)) for k, a, b in closes[:12]])
