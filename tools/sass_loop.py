"""Extract one kernel's SASS and summarise the innermost (hottest) loop body.

usage: python tools/sass_loop.py <lib.so> <kernel-substring> [loop-start-hex loop-end-hex]
Without addresses, picks the smallest backward-branch body (> 40 instructions)
that contains an LDS (the unrolled channel loop).
"""
import re
import subprocess
import sys
from collections import Counter

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
body = next(f for f in funcs if f.split("\n", 1)[0].strip().endswith(pat) or pat in f.split("\n", 1)[0])
ins = []
for line in body.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
need = "LDS"
if "--need" in sys.argv:
    need = sys.argv[sys.argv.index("--need") + 1]
    del sys.argv[sys.argv.index("--need"):sys.argv.index("--need") + 2]
if len(sys.argv) >= 5:
    lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
else:
    best = None
    for addr, txt in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", txt)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < addr:
                seg = [t for a, t in ins if tgt <= a <= addr]
                if any(need in t for t in seg) and len(seg) > 40 and (best is None or len(seg) < best[2]):
                    best = (tgt, addr, len(seg))
    lo, hi = best[0], best[1]
seg = [t for a, t in ins if lo <= a <= hi]
ops = Counter()
for t in seg:
    t = re.sub(r"^@!?U?P\w+\s+", "", t)
    ops[t.split()[0]] += 1
print(f"loop 0x{lo:x}-0x{hi:x}: {len(seg)} instructions")
for k, v in ops.most_common():
    print(f"  {k:24s} {v}")
