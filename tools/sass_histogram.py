"""Per-kernel SASS instruction histogram of the built library (cuobjdump -sass): the
mnemonics that prove the tcgen05 / TMA / DMMA paths (UTCHMMA, UTMALDG.*, LDTM, DMMA ...).
usage: python tools/sass_histogram.py [lib.so] > profiles/r2_sass_histogram.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2602_00397_b200/libffwd_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                      check=True).stdout
WATCH = ("UTCHMMA", "UTCBAR", "UTMALDG", "UTMAPF", "UTMACMDFLUSH", "LDTM", "DMMA", "DFMA",
         "SYNCS", "ELECT", "R2UR", "NANOSLEEP", "F2F", "LDGSTS")
kern, counts = None, collections.OrderedDict()
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]+)", line)
    if m and kern:
        op = m.group(1)
        for w in WATCH:
            if op.startswith(w):
                counts[kern][op] += 1
print(f"# SASS histogram of {lib} (cuobjdump -sass), watched mnemonics per kernel")
for k, c in counts.items():
    if not c:
        continue
    short = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    print(f"\n{short[:150]}")
    for op, n in sorted(c.items()):
        print(f"  {op:40s} {n}")
