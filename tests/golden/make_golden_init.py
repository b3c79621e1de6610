"""Golden vectors for the sphere pre-fit, by running the REFERENCE's
``decoders.geometric_init`` (gs/decoders.py:102-177).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_init.py

Case "small" of make_golden.py (same dataset, config and
``build_model(skip_init=True)`` parameters), centre/radius as
``build_model`` derives them (gs/optimizer.py:206-213) except radius = 0.3 x
the smallest extent (0.5 touches this scene's box).  Stored per precision:
  * ``K``-step run (max_steps=K, tol huge so it never raises): the geometry
    levels and geometry decoder after K steps, and the returned RMSE;
  * a full run with the default budget/tolerance (double only): the number of
    steps taken (early-exit point) and the final RMSE.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

from gridsurf import decoders, optimizer

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import CASES, render  # noqa: E402

K = 8


def main():
    case = CASES["small"]
    ds = render(case)
    for precision in ("double", "single"):
        cfg = optimizer.TrainConfig(precision=precision, **case["cfg"])
        cfg.weights.smooth_count = case["smooth_count"]
        lo, hi = optimizer.derive_bounds(ds, cfg)
        center = 0.5 * (lo + hi)
        # the default 0.5 x min extent touches this scene's box; 0.3 keeps it inside
        radius = 0.3 * float(np.min(hi - lo))
        model = optimizer.build_model(ds, cfg, skip_init=True)
        rmse_k = decoders.geometric_init(model.grid, model.geom_net, center, radius, seed=cfg.seed,
                                         max_steps=K, tol=1e9)
        arrays = {f"level{i}": l.features.data.copy() for i, l in enumerate(model.grid.levels)}
        for i, (W, b) in enumerate(model.geom_net.layers):
            arrays[f"geom_w{i}"] = W.data.copy()
            arrays[f"geom_b{i}"] = b.data.copy()
        meta = dict(K=K, rmse_k=rmse_k, center=list(map(float, center)), radius=radius,
                    seed=cfg.seed)
        if precision == "double":
            # full run: count the steps the early exit takes
            model2 = optimizer.build_model(ds, cfg, skip_init=True)
            calls = {"n": 0}
            orig = decoders.Adam.step if hasattr(decoders, "Adam") else None
            from gridsurf import optimizer as gopt
            step0 = gopt.Adam.step

            def counting(self, grads):
                calls["n"] += 1
                return step0(self, grads)

            gopt.Adam.step = counting
            try:
                rmse_full = decoders.geometric_init(model2.grid, model2.geom_net, center, radius,
                                                    seed=cfg.seed, max_steps=cfg.init_steps,
                                                    tol=cfg.init_tol)
            finally:
                gopt.Adam.step = step0
            meta.update(full_steps=calls["n"], rmse_full=rmse_full)
            del orig
        arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
        path = os.path.join(HERE, f"init_small_{precision}.npz")
        np.savez_compressed(path, **arrays)
        print(path, meta)


if __name__ == "__main__":
    main()
