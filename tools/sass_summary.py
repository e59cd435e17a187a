"""Opcode summary of the built library's SASS (cuobjdump -sass): per kernel, the counts of the
instructions that prove the tensor-core / TMA / TMEM paths (UTCIMMA = tcgen05.mma kind::i8,
UTMALDG = TMA tensor loads, LDTM = tcgen05.ld, DMMA = FP64 mma.sync, UTCBAR = tcgen05.commit,
A_REUSE = collector reuse, .MULTICAST).  python tools/sass_summary.py [lib.so] > profiles/r02_sass_summary.txt"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2402_19147_b200/csrc/libqcur_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCIMMA", "A_REUSE", "UTMALDG", "MULTICAST", "UTMAPF", "LDTM", "UTCBAR", "DMMA", "DFMA", "SYNCS.ARRIVE",
        "ELECT", "UBLKCP", "FFMA2", "LDG.E.ENL2.256"]
per = OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = Counter()
        continue
    if cur is None or "/*" not in line:
        continue
    for k in KEYS:
        if k in line:
            per[cur][k] += 1
tot = Counter()
print(f"# SASS opcode summary of {lib} (sm_100a)")
for fn, c in per.items():
    if not c:
        continue
    tot.update(c)
    short = re.sub(r"_ZN4qcur\d*(_GLOBAL__N__\w+?_\d+)?", "", fn)[:90]
    print(f"{short:92s} " + " ".join(f"{k}={v}" for k, v in sorted(c.items())))
print("TOTAL " + " ".join(f"{k}={v}" for k, v in sorted(tot.items())))
