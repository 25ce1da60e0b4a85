"""Per-opcode counts of cuobjdump -sass listings (make -C paper_1108_5359_b200/csrc sass): the
tcgen05 / TMA / TMEM instructions that prove the tensor-core and TMA paths are in the binary."""
import re
import sys
from collections import Counter

KEY = ("UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "LDTM", "STTM", "UBLKCP", "SYNCS",
       "DFMA", "FFMA", "HMMA", "DMMA", "LDS", "STS", "LDG", "STG", "SHFL", "BAR", "MUFU")
for path in sys.argv[1:]:
    kern, counts = None, {}
    for line in open(path):
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(?:\.[A-Z0-9_.]+)?", line)
        if kern and m:
            counts[kern][m.group(1)] += 1
    print(f"== {path.split('/')[-1]}")
    for k, c in counts.items():
        tot = sum(c.values())
        sel = ", ".join(f"{o} {c[o]}" for o in KEY if c[o])
        print(f"  {k[:110]}\n    {tot} instructions: {sel}")
