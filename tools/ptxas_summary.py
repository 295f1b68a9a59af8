"""Summarise build_obj/ptxas.log: registers / spills per kernel (optionally filtered by a regex)."""
import re
import sys

path = sys.argv[2] if len(sys.argv) > 2 else "paper_2512_01678_b200/build_obj/ptxas.log"
pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
cur = None
rows = {}
for line in open(path):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m:
        rows[cur]["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    if pat is None or pat.search(k):
        print(f"{v.get('regs', '?'):>4} regs {v.get('spill', 0):>5} B spill  {k}")
