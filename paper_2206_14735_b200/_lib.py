"""ctypes binding of the C ABI in include/gsb.h (the in-tree ``_gsb.so``).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_gsb.so")

GSB_OK = 0
GSB_E_ARG, GSB_E_CUDA, GSB_E_BOUNDS, GSB_E_NONFINITE = -1, -2, -3, -4
MAX_LEVELS, MAX_ROUNDS, KMAX, AMAX = 8, 8, 256, 32
ST_BOUNDS, ST_NONFINITE, ST_OVERFLOW, ST_VIEWDIR, ST_ADAM_BAD, ST_DIVERGED = 0, 1, 2, 3, 4, 5
N_STATUS = 8
PART_NAMES = ("total", "rgb", "depth", "sdf", "fs", "eik", "smooth", "s")
N_PARTS = 8
C_VALID, C_TR, C_FS, C_EIK = 0, 1, 2, 3

# every function include/gsb.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "gsb_version", "gsb_step_workspace_size", "gsb_step_workspace_layout", "gsb_train_step",
    "gsb_adam_step", "gsb_pcg64_random", "gsb_ray_batch", "gsb_gather_weighted",
    "gsb_scatter_weighted", "gsb_grid_sample", "gsb_importance_round",
    "gsb_step_workspace_regions", "gsb_importance_refine", "gsb_launch_count",
    "gsb_timing_enable", "gsb_timing_collect",
    "gsb_sdf_workspace_size", "gsb_sdf_points", "gsb_sdf_fit_step", "gsb_smooth_points",
    "gsb_sdf_volume_workspace_size", "gsb_sdf_volume", "gsb_mc_workspace_size", "gsb_mc_count",
    "gsb_mc_emit", "gsb_nn_workspace_size", "gsb_nearest_neighbors", "gsb_raster_zbuffer",
    "gsb_pose_table", "gsb_pose_scratch_size", "gsb_pose_grad", "gsb_render_frames", "gsb_det_scratch_size",
)
REGIONS = ("parts", "counts", "status", "depths", "weights", "phi", "gphi", "color", "pbar",
           "ubar", "cbar", "ray_o", "ray_r", "ray_far")


class Level(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("channels", C.c_int32),
                ("ox", C.c_double), ("oy", C.c_double), ("oz", C.c_double),
                ("voxel", C.c_double), ("offset", C.c_int64)]


class Model(C.Structure):
    _fields_ = [("precision", C.c_int32), ("n_levels", C.c_int32),
                ("levels", Level * MAX_LEVELS), ("color", Level),
                ("mlp_offset", C.c_int64), ("log_s_offset", C.c_int64), ("n_params", C.c_int64),
                ("lo_c", C.c_double * 3), ("hi_c", C.c_double * 3),
                ("params", C.c_void_p), ("grads", C.c_void_p)]


class Dataset(C.Structure):
    _fields_ = [("colors", C.c_void_p), ("depth_mm", C.c_void_p),
                ("n_frames", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("poses", C.c_void_p)]


SCENE_MAX_PRIMS, SCENE_MAX_OPS, SCENE_MAX_STACK = 16, 32, 8


class Scene(C.Structure):
    _fields_ = [("n_prims", C.c_int32), ("n_ops", C.c_int32),
                ("prim", (C.c_double * 16) * SCENE_MAX_PRIMS),
                ("op", (C.c_int32 * 2) * SCENE_MAX_OPS),
                ("light", C.c_double * 3), ("background", C.c_double * 3)]


class RenderOpts(C.Structure):
    _fields_ = [("rect", C.c_int32 * 4), ("world_c", C.c_double * 3), ("world_r", C.c_double),
                ("has_box", C.c_int32), ("box_lo", C.c_double * 3), ("box_hi", C.c_double * 3)]


class Pose(C.Structure):
    _fields_ = [("n_frames", C.c_int32), ("R0", C.c_void_p), ("nu_offset", C.c_void_p),
                ("t_offset", C.c_void_p), ("t_fixed", C.c_void_p)]


class Pcg64(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64),
                ("inc_hi", C.c_uint64), ("inc_lo", C.c_uint64)]

    @classmethod
    def from_generator(cls, gen):
        st = gen.bit_generator.state
        if st["bit_generator"] != "PCG64":
            raise ValueError("expected a PCG64 generator")
        s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
        m = (1 << 64) - 1
        return cls(s >> 64, s & m, inc >> 64, inc & m)


class Step(C.Structure):
    _fields_ = [("ray_ids", C.c_void_p), ("n_rays", C.c_int32), ("ray_base", C.c_int32),
                ("m_global", C.c_double),
                ("n_coarse", C.c_int32), ("n_rounds", C.c_int32), ("n_add", C.c_int32),
                ("has_fixed_far", C.c_int32),
                ("near", C.c_double), ("max_depth", C.c_double), ("fixed_far", C.c_double),
                ("rng_stratify", Pcg64), ("rng_importance", Pcg64 * MAX_ROUNDS),
                ("w_rgb", C.c_double), ("w_depth", C.c_double), ("w_sdf", C.c_double),
                ("w_fs", C.c_double), ("w_eik", C.c_double), ("w_smooth", C.c_double),
                ("truncation", C.c_double), ("fs_alpha", C.c_double),
                ("smooth_pts", C.c_void_p), ("n_smooth", C.c_int32),
                ("smooth_global", C.c_double),
                ("exact_gather", C.c_int32), ("phases", C.c_int32),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("pose_work", C.c_void_p), ("pose_work_bytes", C.c_size_t),
                ("det_work", C.c_void_p), ("det_work_bytes", C.c_size_t)]


class GsbError(RuntimeError):
    pass


_lib = None


def lib():
    """Load _gsb.so (raises if absent: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise GsbError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, D, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t
    sig = {
        "gsb_version": ([], I32),
        "gsb_launch_count": ([], C.c_uint64),
        "gsb_sdf_workspace_size": ([C.POINTER(Model), I64, C.POINTER(SZ)], I32),
        "gsb_sdf_volume_workspace_size": ([C.POINTER(Model), C.POINTER(SZ)], I32),
        "gsb_sdf_volume": ([C.POINTER(Model), P, D, I64, I64, I64, P, P, SZ, P], I32),
        "gsb_mc_workspace_size": ([I64, I64, I64, C.POINTER(SZ)], I32),
        "gsb_mc_count": ([P, I64, I64, I64, C.c_float, P, P, SZ, P, P, P], I32),
        "gsb_mc_emit": ([P, I64, I64, I64, C.c_float, D, D, D, D, P, P, SZ, P, P, P], I32),
        "gsb_nn_workspace_size": ([I64, I64, I64, I64, C.POINTER(SZ)], I32),
        "gsb_raster_zbuffer": ([P, P, P, P, I64, I32, I32, P, P], I32),
        "gsb_nearest_neighbors": ([P, I64, P, I64, P, D, I64, I64, I64, P, SZ, P, P, P], I32),
        "gsb_smooth_points": ([C.POINTER(Model), C.POINTER(Dataset), P, P, P, P, P, P, I32, D, P, P], I32),
        "gsb_sdf_points": ([C.POINTER(Model), P, I64, P, P, SZ, P], I32),
        "gsb_render_frames": ([C.POINTER(Scene), P, I32, I32, I32, D, D, D, D, D, P, D,
                               C.POINTER(RenderOpts), P, P, P], I32),
        "gsb_det_scratch_size": ([C.POINTER(Model), I32, I32, I32, I32, I32, C.POINTER(SZ)], I32),
        "gsb_pose_table": ([C.POINTER(Model), C.POINTER(Pose), P, P, P], I32),
        "gsb_pose_scratch_size": ([C.POINTER(Model), I32, I32, I32, I32, C.POINTER(SZ)], I32),
        "gsb_pose_grad": ([C.POINTER(Model), C.POINTER(Dataset), C.POINTER(Step), C.POINTER(Pose), P, SZ,
                           P], I32),
        "gsb_sdf_fit_step": ([C.POINTER(Model), P, P, I64, I64, P, SZ, P, P], I32),
        "gsb_timing_enable": ([I32], I32),
        "gsb_timing_collect": ([I32, C.c_char_p, C.POINTER(D), C.POINTER(I64), C.POINTER(I32)], I32),
        "gsb_step_workspace_size": ([C.POINTER(Model), I32, I32, I32, I32, I32, C.POINTER(SZ)], I32),
        "gsb_step_workspace_layout": ([C.POINTER(Model), I32, I32, I32, I32, I32,
                                       C.POINTER(I64), C.POINTER(I64), C.POINTER(I64),
                                       C.POINTER(I64), C.POINTER(I64), C.POINTER(I32)], I32),
        "gsb_step_workspace_regions": ([C.POINTER(Model), I32, I32, I32, I32, I32,
                                        C.POINTER(I64)], I32),
        "gsb_importance_refine": ([I32, I32, I32, I32, P, P, P, P, P, P, P, P], I32),
        "gsb_train_step": ([C.POINTER(Model), C.POINTER(Dataset), C.POINTER(Step), P], I32),
        "gsb_adam_step": ([I32, P, P, P, P, I64, C.POINTER(I64), C.POINTER(D), I32, D, D, D, D, D,
                           P, D, P, P, P], I32),
        "gsb_pcg64_random": ([C.POINTER(Pcg64), I64, I64, P, P], I32),
        "gsb_ray_batch": ([C.POINTER(Dataset), P, I32, P, P], I32),
        "gsb_gather_weighted": ([I32, P, I32, P, P, I64, P, P], I32),
        "gsb_scatter_weighted": ([I32, P, P, P, I32, I64, P, P], I32),
        "gsb_grid_sample": ([I32, C.POINTER(Level), P, P, I64, P, P, P], I32),
        "gsb_importance_round": ([I32, I32, I32, I32, P, P, D, P, P, P, C.POINTER(Pcg64), P, P, P,
                                  P], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def check(rc, what=""):
    if rc != GSB_OK:
        names = {GSB_E_ARG: "bad argument / unsupported configuration", GSB_E_CUDA: "CUDA error",
                 GSB_E_BOUNDS: "grid bounds", GSB_E_NONFINITE: "non-finite"}
        raise GsbError(f"{what}: {names.get(rc, rc)}")
    return rc


def ptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def kernel_times(max_kernels=32):
    """Collect gsb_timing marks -> {kernel name: (total_ms, launches)}."""
    L = lib()
    names = C.create_string_buffer(64 * max_kernels)
    ms = (C.c_double * max_kernels)()
    cnt = (C.c_int64 * max_kernels)()
    n = C.c_int32(0)
    check(L.gsb_timing_collect(max_kernels, names, ms, cnt, C.byref(n)), "timing_collect")
    out = {}
    for k in range(n.value):
        nm = names.raw[64 * k:64 * k + 64].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[k]), int(cnt[k]))
    return out
