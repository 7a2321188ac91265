#!/usr/bin/env python3
"""Static SASS opcode counts of selected kernels (cuobjdump -sass on the built objects): the
evidence that the tile kernels issue UBLKCP (cp.async.bulk), SYNCS (mbarrier) and the DPX /
FMNMX3 / FADD2 instructions the design relies on.
usage: tools/sass_opcodes.py OUT.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

BUILD = Path(__file__).resolve().parents[1] / "paper_2310_03983_b200" / "csrc" / "build"
KERNELS = {  # object -> kernel-name regex
    "minplus_bulk.o": [r"minplus_nt_kernelILi0ELi0E", r"minplus_nt_kernelILi5ELi0E", r"minplus_w32nt_kernel",
                       r"minplus_f32dm_kernelILi32E"],
    "fw.o": [r"block_close_dpx_kernelILi0ELb1E", r"fw_persist_kernel"],
    "close_blk.o": [r"block_close_blk_kernelILi3E"],
}
WATCH = ("UBLKCP", "SYNCS", "VIADDMNMX", "FMNMX3", "FADD2", "FADD", "LDS", "LDG", "STG", "BAR", "SHFL", "NANOSLEEP")


def main(out):
    lines = []
    for obj, pats in KERNELS.items():
        sass = subprocess.run(["cuobjdump", "-sass", str(BUILD / obj)], capture_output=True, text=True).stdout
        funcs = re.split(r"\n\s*Function : ", sass)
        for pat in pats:
            body = next((f for f in funcs if re.match(r"\S*" + pat, f)), None)
            if body is None:
                lines.append(f"{pat}: not found in {obj}")
                continue
            name = body.split("\n", 1)[0].strip()
            ops = collections.Counter()
            for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", body):
                ops[m.group(1)] += 1
            tot = sum(ops.values())
            lines.append(f"== {name} ({obj}): {tot} SASS instructions")
            for w in WATCH:
                c = sum(v for k, v in ops.items() if k.split(".")[0] == w)
                if c:
                    variants = ", ".join(f"{k} {v}" for k, v in ops.most_common() if k.split(".")[0] == w)
                    lines.append(f"   {w:10s} {c:6d}   ({variants})")
    Path(out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1])
