"""Repeat test_f32_parity's conditioned case (a fresh pre-fit each time, so
the float32 rounding near kinks varies) and print the worst gradient error
and the kink flips the resolution took.  Usage (GPU box):
python tools/diag_kink.py [case] [tries]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import test_f32_parity as T  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c1"
tries = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for t in range(tries):
    r = T.run_case(case)
    errs = T._grad_errs(r["g"], r["R"], r["model"].param_names())
    worst = max(errs, key=errs.get)
    dr = np.abs(r["R"]["ratio"] - 1.0)
    jump = r["R"]["ratio_jump"]
    ratio_near = int(((dr < T.RATIO_MARGIN) & (dr > 0) & (jump > 1e-3 * jump.max())).sum())
    print(t, "worst", worst, f"{errs[worst]:.3g}", "ok" if errs[worst] <= T.GRAD_TOL else "FAIL",
          "flips", r["flips"], "ratio candidates", ratio_near, flush=True)
