#!/usr/bin/env python
"""Per-kernel SASS opcode histogram of liblatmap_b200.so (cuobjdump -sass), with the opcodes that
prove the Blackwell paths: UTCHMMA / UTCQMMA (tcgen05.mma), UTCBAR (tcgen05.commit), LDTM
(tcgen05.ld), UTMALDG / UBLKCP (TMA tensor / bulk copies), HMMA (legacy mma.sync), MUFU (SFU).

  python tools/sass_histogram.py [lib.so] > profiles/r02_sass_histogram.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2602_12314_b200/liblatmap_b200.so"
KEY = ("UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "HMMA", "DFMA", "MUFU",
       "LDS", "STS", "LDG", "STG", "RED", "ATOMG", "SHFL", "BAR")

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
kernels = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and cur:
        kernels[cur][m.group(1)] += 1

def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(anonymous namespace\)::|lm::", "", d)
    return d[:110]

print(f"# SASS opcode histogram of {LIB} (cuobjdump -sass; static instruction counts per kernel)")
print("# columns: " + " ".join(KEY) + " | total")
for k, c in kernels.items():
    tot = sum(c.values())
    if tot == 0:
        continue
    print(f"{short(k)}")
    print("    " + " ".join(f"{key}={c.get(key, 0)}" for key in KEY) + f" | total={tot}")
