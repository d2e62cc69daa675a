#!/usr/bin/env python3
"""Opcode census of the kernels in libflashrnn.so (cuobjdump -sass): the
instructions that prove the Blackwell paths -- tcgen05 MMA (UTCHMMA/UTCQMMA),
TMEM loads/stores (LDTM/STTM), TMA (UTMALDG/UTMASTG/UBLKCP), cluster/DSMEM
(SYNCS, ST.ASYNC-style remote stores), mbarrier waits -- per kernel.

    python scripts/sass_summary.py [lib.so] > profiles/r02_sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2412_07752_b200", "libflashrnn.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "SYNCS",
        "FENCE", "MEMBAR", "CCTL", "ELECT", "SHFL", "MUFU", "HMMA", "FFMA", "LDS", "STS", "LDG", "STG", "BAR"]
kern, counts, total = None, {}, collections.Counter()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[\w.]*)?", line)
    if kern and m:
        op = m.group(1)
        counts[kern]["_instr"] += 1
        for k in KEYS:
            if op == k or op.startswith(k):
                counts[kern][k] += 1
                break


def short(n):
    n = re.sub(r"_ZN4frnn\d*(_GLOBAL__N__\w+?_)?", "", n)
    return n[:90]


print(f"# SASS opcode census of {os.path.relpath(lib, ROOT)} (cuobjdump -sass), sm_100a")
print(f"# columns: total instructions, then " + " ".join(KEYS))
for k, c in sorted(counts.items(), key=lambda kv: -kv[1]["_instr"]):
    cols = " ".join(f"{key}={c[key]}" for key in KEYS if c[key])
    print(f"{short(k):90s} n={c['_instr']:6d}  {cols}")
