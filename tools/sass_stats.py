"""Per-kernel SASS statistics of the built library (run here, no GPU):
instruction counts of the mnemonics that matter for this path
(FADD/FADD2, LDS, BRX jump tables, UBLKCP bulk copies, SYNCS mbarriers).

    python tools/sass_stats.py [regex]
"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1601_05052_b200", "libdedisp_b200.so")
pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
func, stats = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        func = m.group(1)
        stats[func] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m and func:
        op = m.group(2).split(".")[0]
        stats[func][op] += 1
        stats[func]["_total"] += 1
keys = ["_total", "FADD", "FADD2", "LDS", "BRX", "UBLKCP", "SYNCS", "STG", "LDG", "BAR"]
for f, c in stats.items():
    if pat.search(f):
        print(f[:70].ljust(70), " ".join(f"{k.strip('_')}={c[k]}" for k in keys if c[k]))
