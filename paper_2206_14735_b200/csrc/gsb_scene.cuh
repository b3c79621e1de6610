// gsb_scene.cuh -- synthetic RGB-D rendering on the device:
// the analytic CSG scene of gs/scenegen.py sphere-traced per pixel, shaded and
// quantised straight into the u8 colour / u16 millimetre dataset layout.
//
// The CSG tree is flattened on the host into a postfix program (gsb_scene_t):
// PUSH k evaluates primitive k, NEG negates the top (Complement), MIN n
// replaces the top n entries by the first minimal one (Union, numpy argmin
// tie order).  Each stack entry carries (value, primitive, sign) so the
// winning primitive's gradient / albedo is what Union.grad / albedo_at pick.
//
// Arithmetic mirrors numpy's float64 op for op (no FMA contraction: explicit
// __dmul_rn / __dadd_rn where nvcc could fuse) except the two BLAS products
// of gs/scenegen.py:297 / 154, whose OpenBLAS orders were measured here:
//   dirs = d_cam @ R.T (dgemm):        fma(a2, b2, fma(a1, b1, a0 b0))
//   n @ light_dir     (dgemv):        fma(n2, l2, fma(n0, l0, n1 l1))
#pragma once

#include <cstdint>

#include "gsb_common.cuh"

namespace gsb {

enum { kPrimSphere = 0, kPrimBox = 1 };
enum { kOpPush = 0, kOpNeg = 1, kOpMin = 2 };

struct SdfHit {
  double v;
  int prim;
  double sign;
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double norm3(double a, double b, double c) {
  return sqrt(dadd(dadd(dmul(a, a), dmul(b, b)), dmul(c, c)));
}

// prim row: [0] type, [1..3] centre, [4] radius | [4..6] half, [7..9] albedo,
// [10..12] albedo2, [13] checker
__device__ __forceinline__ double prim_sdf(const double* P, const double (&x)[3]) {
  if ((int)P[0] == kPrimSphere)
    return dsub(norm3(dsub(x[0], P[1]), dsub(x[1], P[2]), dsub(x[2], P[3])), P[4]);
  double q[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) q[a] = dsub(fabs(dsub(x[a], P[1 + a])), P[4 + a]);
  const double outside = norm3(fmax(q[0], 0.0), fmax(q[1], 0.0), fmax(q[2], 0.0));
  const double inside = fmin(fmax(fmax(q[0], q[1]), q[2]), 0.0);
  return dadd(outside, inside);
}

__device__ __forceinline__ void prim_grad(const double* P, const double (&x)[3], double (&g)[3]) {
  if ((int)P[0] == kPrimSphere) {
    const double d[3] = {dsub(x[0], P[1]), dsub(x[1], P[2]), dsub(x[2], P[3])};
    const double n = fmax(norm3(d[0], d[1], d[2]), 1e-300);
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = d[a] / n;
    return;
  }
  double q[3], s[3], pos[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double d = dsub(x[a], P[1 + a]);
    q[a] = dsub(fabs(d), P[4 + a]);
    s[a] = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 1.0);  // np.sign, 0 -> 1
    pos[a] = fmax(q[a], 0.0);
  }
  if (q[0] < 0.0 && q[1] < 0.0 && q[2] < 0.0) {  // inside: axis of the nearest face
    const int ax = (q[1] > q[0]) ? ((q[2] > q[1]) ? 2 : 1) : ((q[2] > q[0]) ? 2 : 0);
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = (a == ax ? 1.0 : 0.0) * s[a];
    return;
  }
  const double n = fmax(norm3(pos[0], pos[1], pos[2]), 1e-300);
#pragma unroll
  for (int a = 0; a < 3; ++a) g[a] = dmul(s[a], pos[a]) / n;
}

__device__ __forceinline__ void prim_albedo(const double* P, const double (&x)[3], double (&c)[3]) {
  bool odd = false;
  if ((int)P[0] == kPrimBox && P[13] > 0.0) {
    const double k = dadd(dadd(floor(x[0] / P[13]), floor(x[1] / P[13])), floor(x[2] / P[13]));
    const long long ki = (long long)k;
    odd = (((ki % 2) + 2) % 2) == 1;  // numpy floor-mod
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) c[a] = odd ? P[10 + a] : P[7 + a];
}

__device__ __forceinline__ SdfHit scene_eval(const gsb_scene_t& S, const double (&x)[3]) {
  SdfHit st[GSB_SCENE_MAX_STACK];
  int sp = 0;
  for (int i = 0; i < S.n_ops; ++i) {
    const int op = S.op[i][0], arg = S.op[i][1];
    if (op == kOpPush) {
      st[sp].v = prim_sdf(S.prim[arg], x);
      st[sp].prim = arg;
      st[sp].sign = 1.0;
      ++sp;
    } else if (op == kOpNeg) {
      st[sp - 1].v = -st[sp - 1].v;
      st[sp - 1].sign = -st[sp - 1].sign;
    } else {  // kOpMin over the top `arg` entries, first minimum wins
      const int b = sp - arg;
      int best = b;
      for (int j = b + 1; j < sp; ++j)
        if (st[j].v < st[best].v) best = j;
      st[b] = st[best];
      sp = b + 1;
    }
  }
  return st[0];
}

// one thread per pixel of frame f0 + (pixel / HW)
__global__ void __launch_bounds__(128) k_render_frames(gsb_scene_t S, const double* __restrict__ poses,
                                                       int64_t n_pix, int H, int W, double fx, double fy,
                                                       double cx, double cy, double max_t,
                                                       const double* __restrict__ noise, double sigma0,
                                                       gsb_render_opts_t O, uint8_t* __restrict__ colors,
                                                       uint16_t* __restrict__ depth) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_pix) return;
  const int64_t hw = (int64_t)H * W;
  const int64_t f = i / hw;
  const int rem = (int)(i % hw), v = rem / W, u = rem % W;
  // gs/camera.py:142-171
  const double dx = ((double)u - cx) / fx, dy = ((double)v - cy) / fy;
  const double scale = norm3(dx, dy, 1.0);
  const double dc[3] = {dx / scale, dy / scale, 1.0 / scale};
  const double* P = poses + f * 16;  // row-major 4x4 camera-to-world
  double d[3], o[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    d[j] = fma(dc[2], P[j * 4 + 2], fma(dc[1], P[j * 4 + 1], dmul(dc[0], P[j * 4 + 0])));
    o[j] = P[j * 4 + 3];
  }
  // sphere_trace, gs/scenegen.py:223-252
  double t = 0.0;
  bool hit = false;
  for (int it = 0; it < 256; ++it) {
    const double x[3] = {dadd(o[0], dmul(t, d[0])), dadd(o[1], dmul(t, d[1])), dadd(o[2], dmul(t, d[2]))};
    const double s = scene_eval(S, x).v;
    if (fabs(s) < 1e-6) {
      hit = true;
      break;
    }
    t = dadd(t, s);
    if (t > max_t) break;
  }
  const double xh[3] = {dadd(o[0], dmul(t, d[0])), dadd(o[1], dmul(t, d[1])), dadd(o[2], dmul(t, d[2]))};
  double col[3] = {S.background[0], S.background[1], S.background[2]};
  if (hit) {  // AnalyticScene.shade, gs/scenegen.py:151-155
    const SdfHit h = scene_eval(S, xh);
    double g[3], alb[3];
    prim_grad(S.prim[h.prim], xh, g);
    prim_albedo(S.prim[h.prim], xh, alb);
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = h.sign * g[a];
    const double nl = fma(g[2], S.light[2], fma(g[0], S.light[0], dmul(g[1], S.light[1])));
    const double lam = fmax(-nl, 0.0);
    const double k = dadd(0.35, dmul(0.65, lam));
#pragma unroll
    for (int a = 0; a < 3; ++a) col[a] = fmin(fmax(dmul(alb[a], k), 0.0), 1.0);
  }
  double z = hit ? t / scale : 0.0;
  if (sigma0 > 0.0) {  // gs/scenegen.py:303-306
    z = hit ? dadd(z, dmul(dmul(noise[i], sigma0), dmul(z, z))) : 0.0;
    z = fmax(z, 0.0);
  }
  if (O.world_r > 0.0 && hit && norm3(dsub(xh[0], O.world_c[0]), dsub(xh[1], O.world_c[1]),
                                      dsub(xh[2], O.world_c[2])) < O.world_r)
    z = 0.0;
  if (O.has_box && hit && xh[0] >= O.box_lo[0] && xh[0] <= O.box_hi[0] && xh[1] >= O.box_lo[1] &&
      xh[1] <= O.box_hi[1] && xh[2] >= O.box_lo[2] && xh[2] <= O.box_hi[2])
    z = 0.0;
  uint16_t dm = (uint16_t)(long long)rint(dmul(z, 1000.0));
  if (O.rect[2] > O.rect[0] && u >= O.rect[0] && u < O.rect[2] && v >= O.rect[1] && v < O.rect[3]) dm = 0;
  depth[i] = dm;
#pragma unroll
  for (int a = 0; a < 3; ++a) colors[i * 3 + a] = (uint8_t)(int)rint(dmul(col[a], 255.0));
}

}  // namespace gsb
