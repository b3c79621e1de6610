"""Per-kernel time attribution: run bench.py with GSB_DBG knobs (csrc Ws::dbg;
results are invalid under a knob, only the times matter) and print the
per-kernel ms of each variant.  Usage (GPU box): python tools/attrib.py 0 1 2 4 8"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = {}
for v in sys.argv[1:]:
    env = dict(os.environ, GSB_DBG=v)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "5",
                          "--no-cpu-baseline"], env=env, capture_output=True, text=True)
    try:
        line = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        print(v, "failed", out.stderr[-2000:])
        continue
    rows[v] = {k["kernel"]: k["ms_per_step"] * 1e3 for k in line["roofline"]["kernels"]}
    rows[v]["step"] = line["ms_per_step"] * 1e3
names = sorted({k for r in rows.values() for k in r}, key=lambda k: -rows[sys.argv[1]].get(k, 0))
print("kernel".ljust(22) + "".join(f"dbg={v:>4}".rjust(12) for v in rows))
for n in names:
    print(n.ljust(22) + "".join(f"{rows[v].get(n, 0):12.1f}" for v in rows))
