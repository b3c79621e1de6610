"""Train SPEC scene #3 on the device (2000 iterations, float32, seed 0) and
print the culled-mesh metrics at 200 / 2000 iterations (2 cm) and at 2000
(1 cm): the numbers tests/test_trained_mesh.py checks.  Usage: python
tools/trained_metrics.py [runs] [seed ...]"""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_trained_mesh import gt_mesh, scene_dataset  # noqa: E402
from paper_2206_14735_b200 import mesher, optimizer  # noqa: E402

seeds = [int(a) for a in sys.argv[2:]] or [0]
for run in range((int(sys.argv[1]) if len(sys.argv) > 1 else 1) * len(seeds)):
    seed = seeds[run % len(seeds)]
    with tempfile.TemporaryDirectory() as d:
        ds = scene_dataset()
        cfg = optimizer.TrainConfig(precision="single", iterations=2000, batch_rays=1024, seed=seed,
                                    checkpoint_every=200)
        t0 = time.time()
        model, _ = optimizer.train(ds, cfg, d)
        t = time.time() - t0
        res = {}
        for it, r in ((200, 0.02), (2000, 0.02), (2000, 0.01)):
            m, _, _, _ = optimizer.load_model(os.path.join(d, f"ckpt_{it:06d}.gsck"))
            gt = gt_mesh(m, r, ds)
            rep = mesher.evaluate(mesher.cull_mesh(mesher.extract_mesh(m, resolution=r), ds), gt)
            res[f"{it}@{r}"] = {k: round(v, 5) for k, v in json.loads(rep.to_json()).items()
                               if k in ("chamfer_l1", "accuracy", "completion", "normal_consistency", "f_score")}
        print(json.dumps({"run": run, "seed": seed, "train_s": round(t, 2), **res}), flush=True)
