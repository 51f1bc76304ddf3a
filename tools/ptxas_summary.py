"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spill bytes.

usage: nvcc ... -Xptxas -v 2>&1 | python tools/ptxas_summary.py [filter]
"""
import re
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
spill = ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = f"spill st {m.group(1)} ld {m.group(2)}"
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and flt in cur:
        print(f"{cur[:60]:60s} regs {m.group(1):>4s}  {spill}")
        cur = None
