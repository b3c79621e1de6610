"""Mesh extraction, visibility culling and reconstruction metrics
(gs/mesher.py), with the heavy parts on the device.

Same public API as the reference module: TriangleMesh, MetricsReport,
EmptyLevelSetError, extract_mesh, sdf_volume, mesh_from_sdf, cull_mesh,
subdivide_to_edge_length, sample_surface, nearest_neighbors, evaluate,
save_mesh, load_mesh.

Device: the dense SDF decode (gsb_sdf_volume), marching cubes
(gsb_mc_count / gsb_mc_emit, generated 256-case table of mc_table.py), the
per-frame z-buffers of cull_mesh (gsb_raster_zbuffer) and the exact
nearest-neighbour search of the metrics (gsb_nearest_neighbors).  Host
(numpy): the RNG-driven surface sampling (bit-exact streams), the
subdivision bookkeeping and I/O.

Differences from the reference: marching cubes emits three vertices per
triangle (scikit-image welds shared edge vertices); faces, areas and every
metric are unaffected.  ``threads`` arguments are accepted and ignored.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib, camera, seeds
from .mc_table import EDGE_CORNERS, NTRI, TABLE

__all__ = [
    "TriangleMesh", "MetricsReport", "EmptyLevelSetError",
    "extract_mesh", "cull_mesh", "evaluate", "subdivide_to_edge_length",
    "sample_surface", "save_mesh", "load_mesh", "mesh_from_sdf", "sdf_volume",
    "nearest_neighbors",
]

MAX_EDGE = 0.015
OCCLUSION_TOL = 0.01
EVAL_DENSITY = 1e4  # points per m^2 = 1 per cm^2
EVAL_SEED = 90210


class EmptyLevelSetError(RuntimeError):
    pass


@dataclass
class TriangleMesh:
    vertices: np.ndarray  # (V, 3) float64
    faces: np.ndarray     # (F, 3) int64

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=np.float64).reshape(-1, 3)
        self.faces = np.asarray(self.faces, dtype=np.int64).reshape(-1, 3)
        if self.faces.size and self.faces.max() >= len(self.vertices):
            raise ValueError("face index out of range")

    def _edges(self):
        v = self.vertices
        return v[self.faces[:, 1]] - v[self.faces[:, 0]], v[self.faces[:, 2]] - v[self.faces[:, 0]]

    def face_areas(self):
        a, b = self._edges()
        return 0.5 * np.linalg.norm(np.cross(a, b), axis=1)

    def face_normals(self):
        a, b = self._edges()
        n = np.cross(a, b)
        return n / np.maximum(np.linalg.norm(n, axis=1, keepdims=True), 1e-300)

    def area(self):
        return float(self.face_areas().sum())

    def drop_degenerate(self, min_area=1e-14):
        return TriangleMesh(self.vertices, self.faces[self.face_areas() > min_area])


@dataclass
class MetricsReport:
    accuracy: float
    completion: float
    chamfer_l1: float
    normal_consistency: float
    f_score: float
    precision: float
    recall: float
    threshold: float
    n_pred_points: int
    n_gt_points: int

    def to_json(self):
        return json.dumps(asdict(self), indent=2, sort_keys=True)

    def table(self):
        rows = [("accuracy [m]", self.accuracy), ("completion [m]", self.completion),
                ("chamfer-l1 [m]", self.chamfer_l1),
                ("normal consistency", self.normal_consistency),
                (f"f-score @ {self.threshold:g} m", self.f_score)]
        w = max(len(r[0]) for r in rows)
        return "\n".join(f"{n:<{w}}  {v:.6f}" for n, v in rows)


# ---------------------------------------------------------------------------
# device helpers


def _torch():
    import torch
    return torch


_TABLES = {}


def _mc_table(device):
    key = str(device)
    if key not in _TABLES:
        torch = _torch()
        packed = np.concatenate([NTRI.astype(np.int8), TABLE[:, :16].reshape(-1).astype(np.int8),
                                 EDGE_CORNERS.reshape(-1).astype(np.int8)])
        assert TABLE.shape[1] <= 16 + 1 and packed.size == 256 + 256 * 16 + 24
        _TABLES[key] = torch.from_numpy(packed).to(device)
    return _TABLES[key]


def _device(default=None):
    torch = _torch()
    return default if default is not None else torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------------------
# extraction (gs/mesher.py:108-151)


def volume_dims(model, resolution):
    """World box shrunk by half the finest voxel, and the vertex counts."""
    margin = 0.5 * model.grid.finest_voxel
    lo = model.grid.lo + margin
    hi = model.grid.hi - margin
    dims = np.maximum(np.floor((hi - lo) / resolution).astype(int) + 1, 2)
    return lo, dims


def sdf_volume_device(model, resolution):
    """(vol (nx, ny, nz) float32 device tensor, lo, resolution)."""
    from .engine import model_struct
    torch = _torch()
    lo, dims = volume_dims(model, resolution)
    dev = model.arena.device
    vol = torch.empty(tuple(int(d) for d in dims), dtype=torch.float32, device=dev)
    ms = model_struct(model)
    lib = _lib.lib()
    nb = C.c_size_t(0)
    _lib.check(lib.gsb_sdf_volume_workspace_size(C.byref(ms), C.byref(nb)), "sdf_volume_ws")
    ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
    lo_h = (C.c_double * 3)(*map(float, lo))
    _lib.check(lib.gsb_sdf_volume(C.byref(ms), lo_h, float(resolution), int(dims[0]), int(dims[1]),
                                  int(dims[2]), vol.data_ptr(), ws.data_ptr(), ws.numel(),
                                  _lib.stream_handle()), "gsb_sdf_volume")
    return vol, lo, resolution


def sdf_volume(model, resolution, threads=1):
    """Decode the SDF on a dense grid over the model's world box
    (gs/mesher.py:114-133): (vol float32 numpy, lo, resolution)."""
    vol, lo, res = sdf_volume_device(model, resolution)
    return vol.cpu().numpy(), lo, res


def mesh_from_sdf(vol, origin, resolution, level=0.0, device=None):
    """Marching cubes on a dense SDF volume (numpy or device tensor); raises
    EmptyLevelSetError if there is no zero crossing (gs/mesher.py:136-146)."""
    torch = _torch()
    if isinstance(vol, torch.Tensor) and vol.is_cuda:
        v = vol.to(torch.float32).contiguous()
    else:
        v = torch.from_numpy(np.ascontiguousarray(vol, dtype=np.float32)).to(_device(device))
    nx, ny, nz = (int(s) for s in v.shape)
    lib = _lib.lib()
    tab = _mc_table(v.device)
    nb = C.c_size_t(0)
    _lib.check(lib.gsb_mc_workspace_size(nx, ny, nz, C.byref(nb)), "mc_workspace")
    ws = torch.empty(nb.value, dtype=torch.uint8, device=v.device)
    total = torch.zeros(1, dtype=torch.int64, device=v.device)
    minmax = torch.zeros(2, dtype=torch.float32, device=v.device)
    s = _lib.stream_handle()
    _lib.check(lib.gsb_mc_count(v.data_ptr(), nx, ny, nz, float(level), tab.data_ptr(), ws.data_ptr(),
                                ws.numel(), total.data_ptr(), minmax.data_ptr(), s), "gsb_mc_count")
    lo_v, hi_v = (float(x) for x in minmax.cpu())
    if lo_v > level or hi_v < level:
        raise EmptyLevelSetError("SDF volume has no zero crossing")
    n = int(total.item())
    verts = torch.empty((3 * n, 3), dtype=torch.float64, device=v.device)
    keys = torch.empty(3 * n, dtype=torch.int64, device=v.device)
    if n:
        o = np.asarray(origin, dtype=np.float64)
        _lib.check(lib.gsb_mc_emit(v.data_ptr(), nx, ny, nz, float(level), float(o[0]), float(o[1]),
                                   float(o[2]), float(resolution), tab.data_ptr(), ws.data_ptr(),
                                   ws.numel(), verts.data_ptr(), keys.data_ptr(), s), "gsb_mc_emit")
    vw, faces = weld(verts.cpu().numpy(), keys.cpu().numpy())
    return TriangleMesh(vw, faces).drop_degenerate()


def weld(verts, keys):
    """One vertex per lattice edge (marching cubes emits it once per
    incident triangle): vertices in order of first use, faces re-indexed.
    Welding by the edge key is welding by identical coordinates, as
    scikit-image's marching cubes returns its mesh."""
    if len(keys) == 0:
        return verts.reshape(0, 3), np.zeros((0, 3), dtype=np.int64)
    _, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    return verts[first[order]], rank[inv.reshape(-1)].reshape(-1, 3).astype(np.int64)


def extract_mesh(model, resolution=0.01, threads=1):
    """Zero level set of the decoded SDF as a triangle mesh (gs/mesher.py:149-151)."""
    vol, lo, res = sdf_volume_device(model, resolution)
    return mesh_from_sdf(vol, lo, res)


# ---------------------------------------------------------------------------
# culling (gs/mesher.py:157-272)


def subdivide_to_edge_length(mesh, max_edge=MAX_EDGE):
    """4-way subdivide faces until every edge is at most max_edge.

    Vectorised; the output (vertex order: midpoints appended in first-use
    order over the split faces' edges ab, bc, ca; face order: kept faces, then
    four children per split face) is the reference loop's, exactly."""
    varr = mesh.vertices.copy()
    faces = mesh.faces
    for _ in range(32):
        v = varr
        e = np.stack([np.linalg.norm(v[faces[:, 1]] - v[faces[:, 0]], axis=1),
                      np.linalg.norm(v[faces[:, 2]] - v[faces[:, 1]], axis=1),
                      np.linalg.norm(v[faces[:, 0]] - v[faces[:, 2]], axis=1)], axis=1)
        needs = e.max(axis=1) > max_edge
        if not needs.any():
            break
        sf = faces[needs]
        a, b, c = sf[:, 0], sf[:, 1], sf[:, 2]
        # the three edge keys of each split face in the reference's call order
        pa = np.stack([a, b, c], axis=1).reshape(-1)
        pb = np.stack([b, c, a], axis=1).reshape(-1)
        lo_, hi_ = np.minimum(pa, pb), np.maximum(pa, pb)
        key = lo_ * len(varr) + hi_
        uk, first, inv = np.unique(key, return_index=True, return_inverse=True)
        rank = np.empty(len(uk), dtype=np.int64)  # first-use order
        rank[np.argsort(first, kind="stable")] = np.arange(len(uk))
        mid_idx = len(varr) + rank[inv].reshape(-1, 3)
        ordered = np.argsort(rank, kind="stable")
        new_rows = 0.5 * (varr[pa[first[ordered]]] + varr[pb[first[ordered]]])
        ab, bc, ca = mid_idx[:, 0], mid_idx[:, 1], mid_idx[:, 2]
        quads = np.stack([np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
                          np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)], axis=1).reshape(-1, 3)
        faces = np.concatenate([faces[~needs], quads], axis=0)
        varr = np.concatenate([varr, new_rows], axis=0)
    return TriangleMesh(varr, faces)


def cull_mesh(mesh, dataset, thin_mode=False, max_edge=MAX_EDGE, occlusion_tol=OCCLUSION_TOL,
              threads=1):
    """Remove faces never observed by the dataset's cameras (gs/mesher.py:232-272):
    a (subdivided) face survives if any vertex, in any frame, projects inside
    the image with positive depth, within occlusion_tol of the mesh's own
    z-buffer (rasterised on the device), and (unless thin_mode) on a pixel with
    valid depth."""
    torch = _torch()
    fine = subdivide_to_edge_length(mesh, max_edge)
    intr = dataset.intrinsics
    verts = fine.vertices
    valid = (dataset.depths_mm > 0) if hasattr(dataset, "depths_mm") else (dataset.depths > 0)
    visible = np.zeros(len(verts), dtype=bool)
    dev = _device()
    lib = _lib.lib()
    faces_d = torch.from_numpy(np.ascontiguousarray(fine.faces)).to(dev)
    zbuf_d = torch.empty((intr.height, intr.width), dtype=torch.float64, device=dev)
    for f in range(len(dataset.poses)):
        u, v, z = camera.project(intr, dataset.poses[f], verts)
        inside = (z > 1e-9) & (u >= 0) & (u <= intr.width - 1) & (v >= 0) & (v <= intr.height - 1)
        if not inside.any():
            continue
        uvz = torch.from_numpy(np.stack([u, v, z])).to(dev)
        _lib.check(lib.gsb_raster_zbuffer(uvz[0].data_ptr(), uvz[1].data_ptr(), uvz[2].data_ptr(),
                                          faces_d.data_ptr(), len(fine.faces), intr.height, intr.width,
                                          zbuf_d.data_ptr(), _lib.stream_handle()), "gsb_raster_zbuffer")
        zbuf = zbuf_d.cpu().numpy()
        ui = np.clip(np.round(u).astype(np.int64), 0, intr.width - 1)
        vi = np.clip(np.round(v).astype(np.int64), 0, intr.height - 1)
        ok = inside & (z <= zbuf[vi, ui] + occlusion_tol)
        if not thin_mode:
            ok &= valid[f][vi, ui]
        visible |= ok
    keep = visible[fine.faces].any(axis=1)
    return _compact(TriangleMesh(fine.vertices, fine.faces[keep]))


def _compact(mesh):
    """Drop unreferenced vertices and reindex faces."""
    used = np.unique(mesh.faces.ravel()) if mesh.faces.size else np.empty(0, np.int64)
    remap = np.full(len(mesh.vertices), -1, dtype=np.int64)
    remap[used] = np.arange(used.size)
    return TriangleMesh(mesh.vertices[used], remap[mesh.faces])


# ---------------------------------------------------------------------------
# metrics (gs/mesher.py:278-400)


def sample_surface(mesh, density=EVAL_DENSITY, seed=EVAL_SEED):
    """Area-weighted uniform surface samples with face normals; N =
    round(area * density).  Same RNG stream and calls as the reference."""
    areas = mesh.face_areas()
    total = areas.sum()
    if total <= 0:
        raise ValueError("mesh has no area to sample")
    n = max(int(round(total * density)), 1)
    rng = np.random.default_rng(np.random.SeedSequence((seed, seeds.EVAL_SAMPLES)))
    tri = rng.choice(len(areas), size=n, p=areas / total)
    r1 = np.sqrt(rng.random(n))
    r2 = rng.random(n)
    v = mesh.vertices
    a, b, c = v[mesh.faces[tri, 0]], v[mesh.faces[tri, 1]], v[mesh.faces[tri, 2]]
    pts = (1 - r1)[:, None] * a + (r1 * (1 - r2))[:, None] * b + (r1 * r2)[:, None] * c
    return pts, mesh.face_normals()[tri]


def nearest_neighbors(query, ref, cell):
    """Exact nearest neighbour (distance, index) from query into ref points,
    on the device with the reference's cell hash (gs/mesher.py:348-363)."""
    torch = _torch()
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    query = np.ascontiguousarray(query, dtype=np.float64)
    lo = np.minimum(ref.min(axis=0), query.min(axis=0)) - cell
    hi = np.maximum(ref.max(axis=0), query.max(axis=0)) + cell
    dims = np.maximum(((hi - lo) / cell).astype(np.int64) + 1, 1)
    nx, ny, nz = (int(d) for d in dims)
    dev = _device()
    lib = _lib.lib()
    nb = C.c_size_t(0)
    _lib.check(lib.gsb_nn_workspace_size(len(ref), nx, ny, nz, C.byref(nb)), "nn_workspace")
    ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
    q_d = torch.from_numpy(query).to(dev)
    r_d = torch.from_numpy(ref).to(dev)
    out_d = torch.empty(len(query), dtype=torch.float64, device=dev)
    out_i = torch.empty(len(query), dtype=torch.int64, device=dev)
    lo_h = (C.c_double * 3)(*map(float, lo))
    _lib.check(lib.gsb_nearest_neighbors(q_d.data_ptr(), len(query), r_d.data_ptr(), len(ref), lo_h,
                                         float(cell), nx, ny, nz, ws.data_ptr(), ws.numel(),
                                         out_d.data_ptr(), out_i.data_ptr(), _lib.stream_handle()),
               "gsb_nearest_neighbors")
    return out_d.cpu().numpy(), out_i.cpu().numpy()


def evaluate(pred_mesh, gt_mesh, threshold=0.05, density=EVAL_DENSITY, seed=EVAL_SEED):
    """Accuracy, completion, chamfer-l1, normal consistency and F-score
    between two meshes (gs/mesher.py:366-400)."""
    if pred_mesh.faces.size == 0 or gt_mesh.faces.size == 0:
        raise ValueError("cannot evaluate an empty mesh")
    p_pts, p_nrm = sample_surface(pred_mesh, density, seed)
    g_pts, g_nrm = sample_surface(gt_mesh, density, seed)
    d_pg, i_pg = nearest_neighbors(p_pts, g_pts, threshold)
    d_gp, i_gp = nearest_neighbors(g_pts, p_pts, threshold)
    acc = float(d_pg.mean())
    comp = float(d_gp.mean())
    nc_pg = np.abs(np.sum(p_nrm * g_nrm[i_pg], axis=1)).mean()
    nc_gp = np.abs(np.sum(g_nrm * p_nrm[i_gp], axis=1)).mean()
    precision = float((d_pg < threshold).mean())
    recall = float((d_gp < threshold).mean())
    f = 2 * precision * recall / (precision + recall) if precision + recall > 0 else 0.0
    return MetricsReport(accuracy=acc, completion=comp, chamfer_l1=0.5 * (acc + comp),
                         normal_consistency=float(0.5 * (nc_pg + nc_gp)), f_score=float(f),
                         precision=precision, recall=recall, threshold=float(threshold),
                         n_pred_points=len(p_pts), n_gt_points=len(g_pts))


# ---------------------------------------------------------------------------
# I/O: PLY (ascii / binary little-endian) and OBJ (gs/mesher.py:406-485)


def save_mesh(path, mesh, binary=True):
    path = str(path)
    if path.endswith(".obj"):
        with open(path, "w") as f:
            f.writelines(f"v {x:.9g} {y:.9g} {z:.9g}\n" for x, y, z in mesh.vertices)
            f.writelines(f"f {a + 1} {b + 1} {c + 1}\n" for a, b, c in mesh.faces)
        return
    nv, nf = len(mesh.vertices), len(mesh.faces)
    header = (f"ply\nformat {'binary_little_endian' if binary else 'ascii'} 1.0\n"
              f"element vertex {nv}\nproperty float x\nproperty float y\nproperty float z\n"
              f"element face {nf}\nproperty list uchar int vertex_indices\nend_header\n")
    if binary:
        rec = np.empty(nf, dtype=[("n", "u1"), ("idx", "<i4", (3,))])
        rec["n"] = 3
        rec["idx"] = mesh.faces.astype("<i4")
        with open(path, "wb") as f:
            f.write(header.encode("ascii"))
            f.write(mesh.vertices.astype("<f4").tobytes())
            f.write(rec.tobytes())
    else:
        with open(path, "w") as f:
            f.write(header)
            f.writelines(f"{x:.9g} {y:.9g} {z:.9g}\n" for x, y, z in mesh.vertices)
            f.writelines(f"3 {a} {b} {c}\n" for a, b, c in mesh.faces)


def load_mesh(path):
    path = str(path)
    if path.endswith(".obj"):
        verts, faces = [], []
        with open(path) as f:
            for line in f:
                p = line.split()
                if p and p[0] == "v":
                    verts.append([float(x) for x in p[1:4]])
                elif p and p[0] == "f":
                    faces.append([int(t.split("/")[0]) - 1 for t in p[1:4]])
        return TriangleMesh(np.asarray(verts), np.asarray(faces, dtype=np.int64))
    with open(path, "rb") as f:
        if f.readline().strip() != b"ply":
            raise ValueError(f"{path}: not a PLY file")
        fmt, nv, nf = None, 0, 0
        while True:
            tok = f.readline().split()
            if not tok:
                raise ValueError(f"{path}: truncated PLY header")
            if tok[0] == b"format":
                fmt = tok[1].decode()
            elif tok[0] == b"element":
                if tok[1] == b"vertex":
                    nv = int(tok[2])
                else:
                    nf = int(tok[2])
            elif tok[0] == b"end_header":
                break
        if fmt == "ascii":
            verts = np.loadtxt(f, max_rows=nv).reshape(nv, -1)[:, :3]
            faces = np.loadtxt(f, max_rows=nf).reshape(nf, -1)[:, 1:4].astype(np.int64)
        elif fmt == "binary_little_endian":
            verts = np.frombuffer(f.read(nv * 12), dtype="<f4").reshape(nv, 3).astype(np.float64)
            rec = np.frombuffer(f.read(nf * 13), dtype=[("n", "u1"), ("idx", "<i4", (3,))])
            faces = rec["idx"].astype(np.int64)
        else:
            raise ValueError(f"{path}: unsupported PLY format {fmt}")
    return TriangleMesh(np.asarray(verts, dtype=np.float64), faces)
