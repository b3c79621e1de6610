"""Golden RGB-D frames of the data path, by running the
REFERENCE renderer (gs/scenegen.py:290-368):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_scene.py

* "corrupt": sphere_in_box, 4 orbit frames 64x48, depth noise
  sigma0 = 0.002 z^2 (seed 5), a pixel-rectangle, a world-ball and a
  world-box dropout;
* "slab": thin_slab (1 cm slab), 4 orbit frames 48x36, clean.
(Clean sphere_in_box frames are already in c1_*.npz / small_*.npz.)
"""

from __future__ import annotations

import json
import os

import numpy as np

from gridsurf import scenegen
from gridsurf.camera import Intrinsics

HERE = os.path.dirname(os.path.abspath(__file__))


def intr_of(w, h):
    f = 0.5 * w / np.tan(np.radians(35.0))
    return Intrinsics(fx=f, fy=f, cx=w / 2.0, cy=h / 2.0, width=w, height=h)


def main():
    cases = {
        "corrupt": dict(scene="sphere_in_box", w=64, h=48, frames=4,
                        kw=dict(noise_sigma0=0.002, seed=5, dropout_rect=(5, 4, 20, 12),
                                dropout_world=((0.0, 0.0, -0.5), 0.2),
                                dropout_box=((-1.0, 0.5, -1.0), (1.0, 1.0, 1.0)))),
        "slab": dict(scene="thin_slab", w=48, h=36, frames=4, kw={}),
    }
    arrays = {}
    meta = {}
    for name, c in cases.items():
        intr = intr_of(c["w"], c["h"])
        traj = scenegen.orbit_trajectory(c["frames"])
        ds = scenegen.render_dataset(getattr(scenegen, c["scene"])(), traj, intr, max_t=8.0, **c["kw"])
        arrays[f"{name}_colors_u8"] = np.round(ds.colors * 255.0).astype(np.uint8)
        arrays[f"{name}_depths_u16"] = np.round(ds.depths * 1000.0).astype(np.uint16)
        arrays[f"{name}_poses"] = traj
        kw = {k: (list(map(list, v)) if k == "dropout_box" else
                  [list(v[0]), v[1]] if k == "dropout_world" else list(v) if isinstance(v, tuple) else v)
              for k, v in c["kw"].items()}
        meta[name] = dict(scene=c["scene"], intr=[intr.fx, intr.fy, intr.cx, intr.cy, c["w"], c["h"]], kw=kw)
    arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    path = os.path.join(HERE, "scene_frames.npz")
    np.savez_compressed(path, **arrays)
    print(path, os.path.getsize(path) / 1e3, "kB", {k: int((v > 0).sum()) for k, v in arrays.items() if "depth" in k})


if __name__ == "__main__":
    main()
