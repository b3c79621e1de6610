"""Print step time and the per-kernel table of a bench.py JSON line (stdin)."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
d = json.loads([l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1])
ks = d.get("roofline", {}).get("kernels", [])
print(tag, "ms/step %.4f" % d["ms_per_step"], "e2e %.4g" % d.get("e2e", {}).get("value", 0),
      " ".join("%s=%.1f" % (k["kernel"].replace("k_", ""), 1e3 * k["ms_per_step"]) for k in ks))
