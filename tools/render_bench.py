"""Time gsb_render_frames vs the numpy renderer on config-4 frames (640x480, large_room)."""
import time
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_14735_b200 import scenes, camera

F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
intr = camera.Intrinsics(577.87, 577.87, 319.5, 239.5, 640, 480)
traj = scenes.orbit_trajectory(F, target=(0.0, 0.0, -3.0), radius=3.0, height=-1.5, height_amp=0.5)
sc = scenes.large_room()
scenes.render_frames_device(sc, traj[:2], intr)
torch.cuda.synchronize()
t0 = time.perf_counter()
c, d = scenes.render_frames_device(sc, traj, intr)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
t1 = time.perf_counter()
h = scenes.render_dataset_host(sc, traj[:2], intr, threads=1)
dh = (time.perf_counter() - t1) / 2
same = bool((c[:2].cpu().numpy() == h.colors_u8).all() and (d[:2].cpu().numpy().view(np.uint16) == h.depths_mm).all())
print(f"device: {F} frames 640x480 in {dt*1e3:.1f} ms ({F/dt:.0f} frames/s); numpy: {dh:.2f} s/frame "
      f"(1 thread); first 2 frames identical: {same}")
