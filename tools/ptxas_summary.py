"""Summarise `nvcc -Xptxas -v` output: registers / spills / stack per kernel."""
import re
import sys

cur = None
rows = []
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\w+)' for", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["stack"], cur["spill_st"], cur["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
filt = sys.argv[2] if len(sys.argv) > 2 else ""
for r in rows:
    n = r["name"]
    if filt and filt not in n:
        continue
    short = re.sub(r"_ZN3gsb\d*", "", n)[:60]
    print(f"{short:60s} regs={r.get('regs')} stack={r.get('stack')} spill={r.get('spill_st')}")
