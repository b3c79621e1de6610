"""Pinhole camera and poses, host side (gs/camera.py).

Conventions as the reference: camera looks down +z, image origin top-left,
camera-to-world matrices, depth images store z-depth.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Intrinsics:
    """gs/camera.py:37-50."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0 <= self.cx <= self.width and 0 <= self.cy <= self.height):
            raise ValueError("principal point must lie inside the image")


_SMALL_ANGLE = 1e-4


def exp_so3_data(nu):
    """gs/camera.py:125-139."""
    nu = np.asarray(nu, dtype=np.float64)
    th2 = float(nu @ nu)
    K = np.array([[0.0, -nu[2], nu[1]], [nu[2], 0.0, -nu[0]], [-nu[1], nu[0], 0.0]])
    if np.sqrt(th2) < _SMALL_ANGLE:
        a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0
        b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0
    else:
        th = np.sqrt(th2)
        a = np.sin(th) / th
        b = (1.0 - np.cos(th)) / th2
    return np.eye(3) + a * K + b * (K @ K)


# the graph form's values (gs/camera.py:96-122): the device step evaluates the
# graph itself (gsb_pose_table); on the host the array form serves both
exp_so3 = exp_so3_data


class PoseParam:
    """Camera-to-world pose R = R0 exp(nu^), t (gs/camera.py:53-90).

    Frozen poses keep nu = 0 and t as host arrays in the model dtype, exactly
    as the reference stores non-trainable poses.  Trainable poses (pose
    refinement) hold nu and t as views into the parameter
    arena (``Param``), so the fused Adam updates them with the rest; R0 stays
    on the host (f64) and is folded by ``refresh``."""

    def __init__(self, R0, t, trainable=False, dtype=np.float64, nu_param=None, t_param=None):
        self.R0 = np.asarray(R0, dtype=np.float64).copy()
        self.version = 0  # bumped by refresh (device copies of R0 follow it)
        self.trainable = bool(trainable)
        if self.trainable:
            if nu_param is None or t_param is None:
                raise ValueError("trainable poses live in the parameter arena (nu_param, t_param)")
            self.nu, self.t = nu_param, t_param
            self.t.set(np.asarray(t, dtype=dtype))
        else:
            self.nu = np.zeros(3, dtype=dtype)
            self.t = np.asarray(t, dtype=dtype).copy()

    @classmethod
    def from_matrix(cls, c2w, trainable=False, dtype=np.float64, nu_param=None, t_param=None):
        c2w = np.asarray(c2w, dtype=np.float64)
        return cls(c2w[:3, :3], c2w[:3, 3], trainable=trainable, dtype=dtype, nu_param=nu_param,
                   t_param=t_param)

    def nu_data(self):
        return self.nu.numpy() if self.trainable else self.nu

    def t_data(self):
        return self.t.numpy() if self.trainable else self.t

    def rotation_data(self):
        return self.R0 @ exp_so3_data(self.nu_data())

    def matrix(self):
        """gs/camera.py:75-80."""
        m = np.eye(4)
        m[:3, :3] = self.rotation_data()
        m[:3, 3] = np.asarray(self.t_data(), dtype=np.float64)
        return m

    def refresh(self):
        """Fold exp(nu) into R0 and zero nu (gs/camera.py:82-87)."""
        if not self.trainable:
            return
        self.R0 = self.R0 @ exp_so3_data(self.nu_data())
        self.nu.set(np.zeros(3))
        self.version += 1

    def parameters(self):
        return [self.nu, self.t] if self.trainable else []


def pixel_rays(intr, pixels, dtype=np.float64):
    """Unit camera-space directions through pixel (u, v) (gs/camera.py:142-157)."""
    px = np.atleast_2d(np.asarray(pixels, dtype=np.float64))
    if np.any(px[:, 0] < 0) or np.any(px[:, 0] >= intr.width) or np.any(
            px[:, 1] < 0) or np.any(px[:, 1] >= intr.height):
        raise ValueError("pixel outside image bounds")
    d = np.stack([(px[:, 0] - intr.cx) / intr.fx, (px[:, 1] - intr.cy) / intr.fy,
                  np.ones(px.shape[0])], axis=1)
    return (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(dtype)


def ray_to_z_scale(intr, pixels):
    """gs/camera.py:160-171."""
    px = np.atleast_2d(np.asarray(pixels, dtype=np.float64))
    d = np.stack([(px[:, 0] - intr.cx) / intr.fx, (px[:, 1] - intr.cy) / intr.fy,
                  np.ones(px.shape[0])], axis=1)
    return np.linalg.norm(d, axis=1)


def load_poses(path):
    """gs/camera.py:251-262."""
    vals = np.atleast_2d(np.loadtxt(path, dtype=np.float64))
    if vals.shape[1] != 16:
        raise ValueError(f"pose file {path}: expected 16 numbers per line, got {vals.shape[1]}")
    poses = vals.reshape(-1, 4, 4)
    for i, p in enumerate(poses):
        if not np.allclose(p[3], [0, 0, 0, 1], atol=1e-6):
            raise ValueError(f"pose {i} in {path} has a malformed last row")
    return poses


def save_poses(path, poses):
    np.savetxt(path, np.asarray(poses, dtype=np.float64).reshape(-1, 16), fmt="%.17g")


def load_intrinsics(path):
    vals = np.loadtxt(path, dtype=np.float64).ravel()
    if vals.size != 6:
        raise ValueError(f"intrinsics file {path}: expected 6 values")
    return Intrinsics(vals[0], vals[1], vals[2], vals[3], int(vals[4]), int(vals[5]))


def save_intrinsics(path, intr):
    with open(path, "w") as f:
        f.write(f"{intr.fx:.17g} {intr.fy:.17g} {intr.cx:.17g} {intr.cy:.17g} "
                f"{intr.width} {intr.height}\n")


def project(intr, c2w, points):
    """World points into one camera -> (u, v, z_cam) (gs/camera.py:201-210):
    p_cam = (p - t) R, pixel = f * p / z + c (z guarded away from 0)."""
    c2w = np.asarray(c2w, dtype=np.float64)
    R, t = c2w[:3, :3], c2w[:3, 3]
    pc = (np.asarray(points, dtype=np.float64) - t) @ R
    z = pc[:, 2]
    safe = np.where(np.abs(z) > 1e-12, z, 1e-12)
    return intr.fx * pc[:, 0] / safe + intr.cx, intr.fy * pc[:, 1] / safe + intr.cy, z


def backproject(intr, pose, pixels):
    """World-space rays through pixels of one camera (gs/camera.py:174-210):
    (origins, unit directions) as (N, 3) arrays; `pose` is a PoseParam or a
    4x4 camera-to-world matrix."""
    if isinstance(pose, PoseParam):
        m = pose.matrix()
    else:
        m = np.asarray(pose, dtype=np.float64)
    d_cam = pixel_rays(intr, pixels)
    dirs = d_cam @ m[:3, :3].T
    origins = np.broadcast_to(m[:3, 3], dirs.shape).copy()
    return origins, dirs


def pose_errors(estimated, ground_truth):
    """Mean translation error (m) and mean geodesic rotation error (degrees)
    between two (F, 4, 4) camera-to-world stacks (gs/camera.py:213-227)."""
    est = np.asarray(estimated, dtype=np.float64)
    gt = np.asarray(ground_truth, dtype=np.float64)
    if est.shape != gt.shape:
        raise ValueError("pose count mismatch")
    trans = np.linalg.norm(est[:, :3, 3] - gt[:, :3, 3], axis=1)
    rel = np.einsum("fij,fik->fjk", est[:, :3, :3], gt[:, :3, :3])  # R_est^T R_gt
    cos = np.clip((np.trace(rel, axis1=1, axis2=2) - 1.0) / 2.0, -1.0, 1.0)
    return float(trans.mean()), float(np.degrees(np.arccos(cos)).mean())


def perturb_pose(c2w, trans_mag, rot_mag_deg, rng):
    """A pose offset by exactly `trans_mag` metres and `rot_mag_deg` degrees in
    random directions (gs/camera.py:230-243): the translation direction, then
    the rotation axis, each drawn as a normalised 3-vector of normals."""
    out = np.asarray(c2w, dtype=np.float64).copy()
    step = rng.normal(size=3)
    step /= np.linalg.norm(step)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    out[:3, 3] += trans_mag * step
    out[:3, :3] = out[:3, :3] @ exp_so3_data(axis * np.radians(rot_mag_deg))
    return out
