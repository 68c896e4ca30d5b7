"""Registers / spills per kernel from build/ptxas.log (make writes it)."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "build/ptxas.log").read().split("\n")
cur = None
for line in log:
    m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = m.group(2)
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        name = re.sub(r"_ZN3cqb\d+", "", cur)[:70]
        print(f"{m2.group(1):>4} regs  spill {spill:>3} B  {name}")
