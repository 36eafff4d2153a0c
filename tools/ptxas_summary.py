"""Summarise paper_2205_07976_b200/_lib/ptxas.log: kernel -> registers, spills."""
import re
import subprocess
import sys
from pathlib import Path

log = Path(sys.argv[1] if len(sys.argv) > 1 else "paper_2205_07976_b200/_lib/ptxas.log").read_text()
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"nbx::|\(nbx::SpotsParams\)", "", cur)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:60s} regs {m.group(1):>3s}  {spill}")
        cur = None
