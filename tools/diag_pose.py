"""GPU diagnostic (not a test): device pose-gradient intermediates vs the oracle."""
import ctypes as C
import sys
import os
import numpy as np
HERE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")
sys.path.insert(0, os.path.dirname(HERE)); sys.path.insert(0, HERE)
import torch
from test_pose import golden, _device_setup, _intr
from types import SimpleNamespace
from _golden import OracleDataset, cfg_ns
from oracle import gridsurf_oracle as O
from paper_2206_14735_b200 import renderer, sampler, seeds

prec = sys.argv[1] if len(sys.argv) > 1 else "single"
a, meta, ds, cfg, model = _device_setup(prec)
it = 0
batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays, near=cfg.near, far=cfg.max_depth)
total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
eng = renderer.engine_for(model, ds)
M = cfg.batch_rays; N = 132
buf = [v for k, v in eng._ws.items() if isinstance(k, tuple) and k[0] == "pose"][0]
tdt = torch.float32 if prec == "single" else torch.float64
esz = 4 if prec == "single" else 8
xbar = buf[:M * N * 6 * esz].view(tdt).view(M, N, 6).cpu().numpy().astype(np.float64)
off = (M * N * 6 * esz + 255) // 256 * 256
rbar = buf[off:off + M * 6 * 8].view(torch.float64).view(M, 6).cpu().numpy()
ws = [v for k, v in eng._ws.items() if not (isinstance(k, tuple) and k[0] == "pose")][0]
fx, fy, cx, cy, w, h = _intr(meta)
intr = SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
ods = OracleDataset(a["colors_u8"], a["depths_u16"], a["poses"], intr)
c = dict(meta["cfg"]); c["voxel_sizes"] = tuple(c["voxel_sizes"])
ocfg = cfg_ns(precision=prec, **c); ocfg.weights.smooth_count = meta["smooth_count"]
dt = np.float64 if prec == "double" else np.float32
P = O.create_params(meta["lo"], meta["hi"], ods.poses, seed=ocfg.seed, voxel_sizes=ocfg.voxel_sizes, dtype=dt, refine_poses=True)
ob = O.draw_ray_batch(ods, O.substream(ocfg.seed, O.RAYS, it), ocfg.batch_rays, near=ocfg.near, far=ocfg.max_depth)
R = O.train_objective(P, ods, ob, it, ocfg)
pz = R["pose"]
def rel(x, y):
    return float(np.abs(x - y).max() / max(np.abs(y).max(), 1e-300))
print("xbar", rel(xbar[..., :3], pz["xbar"]), "vdir", rel(xbar[..., 3:], pz["vdir_bar"]))
print("o_bar", rel(rbar[:, :3], pz["o_bar"]), "r_bar", rel(rbar[:, 3:], pz["r_bar"]))
for nm, reg in (("pbar", "pbar"), ("ubar", "ubar"), ("cbar", "cbar"), ("color", "color"), ("gphi", "gphi")):
    dv = ws[reg].cpu().numpy().astype(np.float64)[:M * N]
    ref = {"pbar": R["adjoints"]["phi_bar"].reshape(-1), "ubar": R["adjoints"]["u"].reshape(-1, 3),
           "cbar": R["adjoints"]["c_bar"].reshape(-1, 3), "color": R["colors"].reshape(-1, 3),
           "gphi": R["gphi"].reshape(-1, 3)}[nm]
    print(nm, rel(dv, ref))
bad = np.abs(xbar[..., :3] - pz["xbar"]).max(axis=2)
i = np.unravel_index(np.argmax(bad), bad.shape)
print("worst sample", i, xbar[i][:3], pz["xbar"][i])
dep_dev = ws["depths"][:, :N].cpu().numpy()
print("depth max abs diff", np.abs(dep_dev - R["depths"]).max())
pd = ws["pbar"].cpu().numpy().astype(np.float64)[:M * N]
pr = R["adjoints"]["phi_bar"].reshape(-1)
d = np.abs(pd - pr)
print("pbar: n mismatch>1e-3*max", int((d > 1e-3 * np.abs(pr).max()).sum()), "of", pd.size)
k = int(np.argmax(d))
phd = ws["phi"].cpu().numpy()[:M * N]
print("worst pbar", k, pd[k], pr[k], "phi dev/ref", phd[k], R["phi"].reshape(-1)[k],
      "b", (ob.depth_ray[:, None] - R["depths"]).reshape(-1)[k])
