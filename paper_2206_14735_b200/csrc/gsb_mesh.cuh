// gsb_mesh.cuh -- mesh extraction and reconstruction metrics on the device
// (mesher.extract_mesh / evaluate, gs/mesher.py:114-151, 287-400).
//
//  * marching cubes over a dense float32 SDF volume: a count pass (cell ->
//    triangle count from the 256-case table), an exclusive scan (CUB), and an
//    emit pass writing three f64 vertices per triangle plus the lattice-edge
//    key of each (the host welds equal keys into one vertex); the table is
//    the generated one of mc_table.py (watertight; see there);
//  * exact nearest neighbours with the reference's grid hash: ref points
//    bucketed by cell (stable radix sort), each query searches Chebyshev
//    rings of cells in the reference's order with its early-out rule, so
//    distances and tie-breaking indices are the reference's.
#pragma once

#include <cub/cub.cuh>

#include "gsb_common.cuh"

namespace gsb {
namespace mesh {

// packed table: ntri[256] | tri[256][16] (edge ids, -1 padded) | edge corners[12][2]
constexpr int kTabNtri = 0, kTabTri = 256, kTabEdge = 256 + 256 * 16, kTabBytes = kTabEdge + 24;

__device__ __forceinline__ int cube_index(const float* __restrict__ vol, int64_t i, int64_t j, int64_t k,
                                          int64_t ny, int64_t nz, float level, float (&v)[8]) {
  int m = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    v[c] = vol[((i + ((c >> 2) & 1)) * ny + (j + ((c >> 1) & 1))) * nz + (k + (c & 1))];
    m |= (v[c] < level ? 1 : 0) << c;
  }
  return m;
}

// order-preserving float <-> int for atomic min/max
__device__ __forceinline__ int f2o(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}

__global__ void k_mc_count(const float* __restrict__ vol, int64_t nx, int64_t ny, int64_t nz, float level,
                           const int8_t* __restrict__ tab, int32_t* __restrict__ counts,
                           int* __restrict__ minmax) {
  const int64_t cells = (nx - 1) * (ny - 1) * (nz - 1);
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int lo = INT_MAX, hi = INT_MIN;
  if (c < cells) {
    const int64_t k = c % (nz - 1), j = (c / (nz - 1)) % (ny - 1), i = c / ((nz - 1) * (ny - 1));
    float v[8];
    counts[c] = tab[kTabNtri + cube_index(vol, i, j, k, ny, nz, level, v)];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      lo = min(lo, f2o(v[q]));
      hi = max(hi, f2o(v[q]));
    }
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(minmax, lo);
    atomicMax(minmax + 1, hi);
  }
}

__global__ void k_mc_emit(const float* __restrict__ vol, int64_t nx, int64_t ny, int64_t nz, float level,
                          double ox, double oy, double oz, double res, const int8_t* __restrict__ tab,
                          const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                          double* __restrict__ verts, int64_t* __restrict__ keys) {
  const int64_t cells = (nx - 1) * (ny - 1) * (nz - 1);
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= cells || counts[c] == 0) return;
  const int64_t k = c % (nz - 1), j = (c / (nz - 1)) % (ny - 1), i = c / ((nz - 1) * (ny - 1));
  float v[8];
  const int m = cube_index(vol, i, j, k, ny, nz, level, v);
  const int nt = tab[kTabNtri + m];
  double* out = verts + (int64_t)offsets[c] * 9;
  const double o[3] = {ox, oy, oz};
  const int64_t base[3] = {i, j, k};
  for (int q = 0; q < 3 * nt; ++q) {
    const int e = tab[kTabTri + m * 16 + q];
    const int a = tab[kTabEdge + 2 * e], b = tab[kTabEdge + 2 * e + 1];
    const double va = v[a], vb = v[b];
    const double t = ((double)level - va) / (vb - va);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double pa = (double)(base[d] + ((a >> (2 - d)) & 1));
      const double pb = (double)(base[d] + ((b >> (2 - d)) & 1));
      out[q * 3 + d] = o[d] + (pa + t * (pb - pa)) * res;
    }
    if (keys) {  // the lattice edge (lower end point, axis) the vertex lies on: equal
                 // keys are bit-identical vertices (a < b along the axis in every cell)
      const int ax = (a ^ b) == 4 ? 0 : ((a ^ b) == 2 ? 1 : 2);
      const int64_t li = i + ((a >> 2) & 1), lj = j + ((a >> 1) & 1), lk = k + (a & 1);
      keys[(int64_t)offsets[c] * 3 + q] = ((li * ny + lj) * nz + lk) * 3 + ax;
    }
  }
}

// ---------------------------------------------------------------------------
// nearest neighbours (gs/mesher.py:302-363)

__global__ void k_nn_cells(const double* __restrict__ ref, int64_t n, double lx, double ly, double lz,
                           double cell, int64_t nx, int64_t ny, int64_t nz, int64_t* __restrict__ cid,
                           int64_t* __restrict__ idx) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  // cidx = clip(((ref - lo) / cell).astype(int64), 0, dims - 1)
  int64_t ci[3];
  const double lo3[3] = {lx, ly, lz};
  const int64_t dims[3] = {nx, ny, nz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int64_t q = (int64_t)((ref[r * 3 + a] - lo3[a]) / cell);
    q = q < 0 ? 0 : q;
    ci[a] = q > dims[a] - 1 ? dims[a] - 1 : q;
  }
  cid[r] = (ci[0] * ny + ci[1]) * nz + ci[2];
  idx[r] = r;
}

// starts[c] = #(sorted cids < c) for c in [0, ncells]
__global__ void k_nn_starts(const int64_t* __restrict__ sorted_cid, int64_t n, int64_t ncells,
                            int64_t* __restrict__ starts) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > ncells) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted_cid[mid] < c) lo = mid + 1; else hi = mid;
  }
  starts[c] = lo;
}

__global__ void k_nn_query(const double* __restrict__ q, int64_t nq, const double* __restrict__ ref,
                           const int64_t* __restrict__ order, const int64_t* __restrict__ starts,
                           double lx, double ly, double lz, double cell, int64_t nx, int64_t ny,
                           int64_t nz, double* __restrict__ out_d, int64_t* __restrict__ out_i) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nq) return;
  const double px = q[t * 3], py = q[t * 3 + 1], pz = q[t * 3 + 2];
  // int((p - lo) / cell) truncates toward zero, then clamp (gs/mesher.py:311-313)
  int64_t cx = (int64_t)((px - lx) / cell), cy = (int64_t)((py - ly) / cell), cz = (int64_t)((pz - lz) / cell);
  cx = cx < 0 ? 0 : (cx > nx - 1 ? nx - 1 : cx);
  cy = cy < 0 ? 0 : (cy > ny - 1 ? ny - 1 : cy);
  cz = cz < 0 ? 0 : (cz > nz - 1 ? nz - 1 : cz);
  double best = INFINITY;
  int64_t besti = -1;
  const int64_t rmax = nx > ny ? (nx > nz ? nx : nz) : (ny > nz ? ny : nz);
  for (int64_t r = 0; r <= rmax; ++r) {
    if (besti >= 0 && r >= 1 && best <= ((double)(r - 1) * cell) * ((double)(r - 1) * cell)) break;
    const int64_t x0 = cx - r > 0 ? cx - r : 0, x1 = cx + r < nx - 1 ? cx + r : nx - 1;
    const int64_t y0 = cy - r > 0 ? cy - r : 0, y1 = cy + r < ny - 1 ? cy + r : ny - 1;
    const int64_t z0 = cz - r > 0 ? cz - r : 0, z1 = cz + r < nz - 1 ? cz + r : nz - 1;
    for (int64_t ix = x0; ix <= x1; ++ix)
      for (int64_t iy = y0; iy <= y1; ++iy)
        for (int64_t iz = z0; iz <= z1; ++iz) {
          const int64_t ax = ix - cx < 0 ? cx - ix : ix - cx;
          const int64_t ay = iy - cy < 0 ? cy - iy : iy - cy;
          const int64_t az = iz - cz < 0 ? cz - iz : iz - cz;
          if (r > 0 && ax != r && ay != r && az != r) continue;  // only the shell at radius r
          const int64_t cid = (ix * ny + iy) * nz + iz;
          for (int64_t kk = starts[cid]; kk < starts[cid + 1]; ++kk) {
            const int64_t j = order[kk];
            const double dx = ref[j * 3] - px, dy = ref[j * 3 + 1] - py, dz = ref[j * 3 + 2] - pz;
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < best) {
              best = d2;
              besti = j;
            }
          }
        }
  }
  out_d[t] = sqrt(best);
  out_i[t] = besti;
}

// ---------------------------------------------------------------------------
// min-z rasterisation with perspective-correct depth (mesher._raster_zbuffer,
// gs/mesher.py:198-229): one thread per face over its pixel bounding box; the
// per-pixel arithmetic is the reference's, and since every written depth is
// positive, the minimum is an integer atomicMin on the f64 bit pattern.
__global__ void k_raster_zbuffer(const double* __restrict__ u, const double* __restrict__ v,
                                 const double* __restrict__ z, const int64_t* __restrict__ faces,
                                 int64_t nf, int H, int W, unsigned long long* __restrict__ zbuf) {
  const int64_t fi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (fi >= nf) return;
  const int64_t i0 = faces[fi * 3], i1 = faces[fi * 3 + 1], i2 = faces[fi * 3 + 2];
  const double z0 = z[i0], z1 = z[i1], z2 = z[i2];
  if (z0 <= 1e-9 || z1 <= 1e-9 || z2 <= 1e-9) return;
  const double x0 = u[i0], y0 = v[i0], x1 = u[i1], y1 = v[i1], x2 = u[i2], y2 = v[i2];
  const int xmin = max((int)floor(fmin(x0, fmin(x1, x2))), 0);
  const int xmax = min((int)ceil(fmax(x0, fmax(x1, x2))), W - 1);
  const int ymin = max((int)floor(fmin(y0, fmin(y1, y2))), 0);
  const int ymax = min((int)ceil(fmax(y0, fmax(y1, y2))), H - 1);
  if (xmin > xmax || ymin > ymax) return;
  const double det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0);
  if (fabs(det) < 1e-18) return;
  const double iz0 = 1.0 / z0, iz1 = 1.0 / z1, iz2 = 1.0 / z2;
  for (int py = ymin; py <= ymax; ++py)
    for (int px = xmin; px <= xmax; ++px) {
      const double w1 = ((px - x0) * (y2 - y0) - (x2 - x0) * (py - y0)) / det;
      const double w2 = ((x1 - x0) * (py - y0) - (px - x0) * (y1 - y0)) / det;
      const double w0 = 1.0 - w1 - w2;
      if (w0 < -1e-9 || w1 < -1e-9 || w2 < -1e-9) continue;
      const double iz = w0 * iz0 + w1 * iz1 + w2 * iz2;
      const double zz = 1.0 / iz;
      atomicMin(zbuf + (int64_t)py * W + px, (unsigned long long)__double_as_longlong(zz));
    }
}

}  // namespace mesh
}  // namespace gsb
