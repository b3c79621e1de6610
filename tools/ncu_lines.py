"""Top source lines by warp-stall samples per kernel (ncu --page source, cuda+sass)."""
import collections
import csv
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file = fn = hdr = None
agg = collections.defaultdict(collections.Counter)
text = {}
for r in csv.reader(raw.splitlines()):
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Function Name":
        fn = r[1][:40]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index(col)
        continue
    if not r or hdr is None or not r[0].isdigit() or r[2] != "-":
        continue
    agg[fn][(cur_file, int(r[0]))] += int(r[si]) if r[si].isdigit() else 0
    text[(cur_file, int(r[0]))] = r[1]
for f, c in agg.items():
    tot = sum(c.values())
    print("==", f, tot)
    for k, v in c.most_common(top):
        print(f"{v:7d} {100 * v / tot:5.1f}% {k[0]}:{k[1]}  {text[k].strip()[:70]}")
