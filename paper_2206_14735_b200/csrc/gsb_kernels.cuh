// gsb_kernels.cuh -- the GO-Surf training-step kernels (templated on the
// storage/compute type T and the grid shape S).
//
// Step data flow (all on one stream, no host round trips):
//   k_ray_setup      rays + stratified depths      gs/sampler.py:58-107, gs/renderer.py:302-321
//                    (float32: k_setup, with the decoder weight tiles in its trailing blocks)
//   k_sdf_eval       no-grad phi at listed samples gs/renderer.py:323-326, 236-240
//   k_importance     one importance round per ray  gs/renderer.py:329-342, gs/sampler.py:128-197
//   k_counts         tr/fs/eik partition counts    gs/renderer.py:384-412
//   k_fwd            phi, grad phi, colour          gs/renderer.py:348-365
//   k_render         alphas/composite/losses/adjoints (warp per ray)
//                                                  gs/renderer.py:112-159, 372-414
//                    + smoothness loss/adjoints in its trailing blocks  gs/renderer.py:416-434
//   k_bwd_geom       grid scatter + geometry MLP grads
//   k_bwd_color      colour grid scatter + colour MLP grads
//   k_finalize       deterministic reductions of the per-CTA MLP partials and the losses
//   k_adam           dense Adam over the arena       gs/optimizer.py:38-55
#pragma once

#include <type_traits>

#include "gsb_common.cuh"
#include "gsb_mlp.cuh"

namespace gsb {

template <typename T>
struct Ws {
  // per ray
  T* o;
  T* r;
  double* od;
  double* rd;
  double* nearv;
  double* farv;
  T* col;
  double* dray;
  int32_t* valid;
  int32_t* cnt;  // [M][3] tr, fs, eik
  double* dep[2];
  double* phi[2];
  int ld;
  int32_t* evl;
  int32_t* evl_count;
  int64_t evl_cap;
  // per sample (M*N taped + 2*S smoothness points)
  T* sphi;
  T* sgphi;
  T* scol;
  T* scolf;             // float32 tcgen05 path: [MN][CC] colour-grid features of the taped samples
                        // (k_fwd_t5 writes them, k_bwd_color_t5 reads them instead of re-gathering)
  T* pbar;
  T* ubar;
  T* cbar;
  T* wts;
  double* ray_part;     // [M][8]
  double* smooth_part;  // [S]
  T* mlp_part;          // [nb_max][NMLP]
  uint4* wfrag;         // float32: per-lane tf32 hi/lo B fragments of the MLP (gsb_tc.cuh)
  int mlp_slots;        // float32 taped backward: >0 = CTAs red.add into slot blockIdx % mlp_slots
  int sweep;            // tcgen05 taped kernels: bit 0 fwd, 1 geometry bwd, 2 colour bwd sweep the tiles backward
  int dbg;              // GSB_DBG time-attribution knobs (results invalid when set): 1 no scatter,
                        // 2 no outer products, 4 no CTA reduction, 8 no feature loads, 16 no MMAs,
                        // 64 no grad-phi corner re-reads (forward)
  uint64_t* det_keys;   // deterministic scatter mode: [NS][NL+1][8] grad-row addresses, or null
  T* det_vals;          // ... and their [8] values (C used); reduced in sample order (k_det_reduce)
  T* pose_g;            // pose refinement, float32: [MN][IN_G] dphi/dz (k_fwd_tc), or null
  T* pose_fb;           // pose refinement, float32: [MN][12] colour-input cotangent (k_bwd_color_tc)
  double* fin_red;      // [FIN_SPLIT][NMLP] chunk totals of k_finalize_mlp2
  unsigned* fin_cnt;    // [ceil(NMLP/32)] tickets (self-resetting; zeroed per step)
  double* loss_red;     // [ceil(max(M, S) / 256)][8] block partials of k_finalize_loss
  unsigned* loss_cnt;   // its ticket (zeroed per step)
  int nb_max;
  long long* counts;
  double* parts;
  int32_t* status;
  uint64_t* imp_state;  // [GSB_MAX_ROUNDS][M][2]: importance-round PCG64 state at row (ray_base + ray) * A
};

// the importance rounds' generators (one substream per round) and A, for
// k_ray_setup's per-row jump-ahead
struct PcgRounds {
  gsb_pcg64_t r[GSB_MAX_ROUNDS];
  int n, A;
};

struct Geo {
  LevelDev lv[GSB_MAX_LEVELS];
  LevelDev col;
  double lo[3], hi[3];
};

// ---------------------------------------------------------------------------
// per-level gather / gradient helpers

template <typename T, int C, bool EXACT>
__device__ __forceinline__ void gather_level(const LevelDev& L, const Loc& q, T* out) {
  const T* F = reinterpret_cast<const T*>(L.feat) + q.base * C;
  if constexpr (EXACT) {
    // _nb_gather_weighted (gs/diffcore.py:816-827): f64 weight times the
    // stored feature, added to the storage-dtype accumulator per corner.
    double wx[2] = {1.0 - q.fx, q.fx}, wy[2] = {1.0 - q.fy, q.fy}, wz[2] = {1.0 - q.fz, q.fz};
    T acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = T(0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double w = (wx[(k >> 2) & 1] * wy[(k >> 1) & 1]) * wz[k & 1];
      T row[C];
      load_row<T, C>(F + corner_off(L, k) * C, row);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = (T)((double)acc[c] + w * (double)row[c]);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) out[c] = acc[c];
  } else {
    T wx[2] = {(T)(1.0 - q.fx), (T)q.fx}, wy[2] = {(T)(1.0 - q.fy), (T)q.fy},
      wz[2] = {(T)(1.0 - q.fz), (T)q.fz};
    T acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = T(0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      T w = (wx[(k >> 2) & 1] * wy[(k >> 1) & 1]) * wz[k & 1];
      T row[C];
      load_row<T, C>(F + corner_off(L, k) * C, row);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = fma(w, row[c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) out[c] = acc[c];
  }
}

// d/dx <interp(theta, x), g> (gs/diffcore.py:844-871), added to grad
template <typename T, int C>
__device__ __forceinline__ void level_dx(const LevelDev& L, const Loc& q, const T* gl, T (&gr)[3]) {
  const T* F = reinterpret_cast<const T*>(L.feat) + q.base * C;
  T e[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    T row[C];
    load_row<T, C>(F + corner_off(L, k) * C, row);
    T a = T(0);
#pragma unroll
    for (int c = 0; c < C; ++c) a = fma(row[c], gl[c], a);
    e[k] = a;
  }
  T x1 = (T)q.fx, y1 = (T)q.fy, z1 = (T)q.fz;
  T x0 = (T)(1.0 - q.fx), y0 = (T)(1.0 - q.fy), z0 = (T)(1.0 - q.fz);
  T iv = (T)L.inv_vs;
  gr[0] += ((e[4] - e[0]) * (y0 * z0) + (e[5] - e[1]) * (y0 * z1) + (e[6] - e[2]) * (y1 * z0) +
            (e[7] - e[3]) * (y1 * z1)) * iv;
  gr[1] += ((e[2] - e[0]) * (x0 * z0) + (e[3] - e[1]) * (x0 * z1) + (e[6] - e[4]) * (x1 * z0) +
            (e[7] - e[5]) * (x1 * z1)) * iv;
  gr[2] += ((e[1] - e[0]) * (x0 * y0) + (e[3] - e[2]) * (x0 * y1) + (e[5] - e[4]) * (x1 * y0) +
            (e[7] - e[6]) * (x1 * y1)) * iv;
}

// ---------------------------------------------------------------------------
// ray setup: draw_ray_batch (given ids) + realized rays + box exit + stratify

template <typename T>
__device__ __forceinline__ void rotate(const double* P, double dx, double dy, double dz, T (&r)[3]) {
  // r = R (M,3,3) @ dir_cam (M,3,1) in the model dtype (gs/renderer.py:307-309).
  // float64: OpenBLAS's stacked dgemm sums sequentially without FMA.  float32:
  // rows 0/1 sequential, row 2 as fma(R22, d2, fma(R20, d0, R21*d1)) -- the
  // pattern measured for numpy's float32 stacked matmul on x86-64 OpenBLAS.
  T d0 = (T)dx, d1 = (T)dy, d2 = (T)dz;
  T R[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = (T)P[i];
  r[0] = (R[0] * d0 + R[1] * d1) + R[2] * d2;
  r[1] = (R[3] * d0 + R[4] * d1) + R[5] * d2;
  if constexpr (sizeof(T) == 4)
    r[2] = fmaf(R[8], d2, fmaf(R[6], d0, R[7] * d1));
  else
    r[2] = (R[6] * d0 + R[7] * d1) + R[8] * d2;
}

struct PixelRay {
  int64_t frame;
  int u, v;
  double dir[3];
  double scale;
  double col[3];
  double depth_ray;
  int valid;
};

// gs/sampler.py:70-88, gs/camera.py:142-171
__device__ __forceinline__ PixelRay pixel_ray(const gsb_dataset_t& D, int64_t flat) {
  PixelRay R;
  int64_t hw = (int64_t)D.height * D.width;
  R.frame = flat / hw;
  int64_t rem = flat % hw;
  R.v = (int)(rem / D.width);
  R.u = (int)(rem % D.width);
  double dx = ((double)R.u - D.cx) / D.fx;
  double dy = ((double)R.v - D.cy) / D.fy;
  double dz = 1.0;
  double nrm = sqrt((dx * dx + dy * dy) + dz * dz);
  R.dir[0] = dx / nrm;
  R.dir[1] = dy / nrm;
  R.dir[2] = dz / nrm;
  R.scale = nrm;
  int64_t pix = (R.frame * D.height + R.v) * D.width + R.u;
  const uint8_t* c = D.colors + pix * 3;
  R.col[0] = (double)c[0] / 255.0;
  R.col[1] = (double)c[1] / 255.0;
  R.col[2] = (double)c[2] / 255.0;
  double z = (double)D.depth_mm[pix] / 1000.0;
  R.valid = z > 0.0;
  R.depth_ray = z * R.scale;
  return R;
}

// rays per block of k_ray_setup: 16 rays x 8 threads (384 blocks at c2)
constexpr int kRaySetupRays = 16;

template <typename T>
__device__ __forceinline__ void ray_setup_block(const gsb_dataset_t& D, const int64_t* __restrict__ ids, int M,
                                                int ray_base, const Ws<T>& w, const Geo& G, int Nc, double nearv,
                                                double max_depth, int has_ff, double ff, const gsb_pcg64_t& rng,
                                                const PcgRounds& imp, int blk, int nfin) {
  // RPB rays per block: threads 0..RPB-1 set the rays up, then all 128
  // threads fill the stratified depths, TPR threads per ray (each jumps its
  // own PCG stream to its first sample)
  constexpr int RPB = kRaySetupRays, TPR = 128 / RPB;  // rays per block, threads per ray
  static_assert(TPR >= GSB_MAX_ROUNDS, "one thread per importance round");
  __shared__ double s_near[RPB], s_span[RPB];
  const int t = threadIdx.x;
  const int i = blk * RPB + t;
  if (blk == 0) {  // the step's counters (first kernel of the step): no memset launches
    if (t < 8) w.counts[t] = 0;
    if (t < GSB_MAX_ROUNDS) w.evl_count[t] = 0;
    if (t == 0) *w.loss_cnt = 0u;
    for (int k = t; k < nfin; k += 128) w.fin_cnt[k] = 0u;  // k_finalize_mlp2 tickets
  }
  if (t < RPB && i < M) {
    PixelRay P = pixel_ray(D, ids[i]);
    const double* pose = D.poses + P.frame * 12;
    T r[3];
    rotate<T>(pose, P.dir[0], P.dir[1], P.dir[2], r);
    T o[3] = {(T)pose[9], (T)pose[10], (T)pose[11]};
    double od[3], rd[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      w.o[i * 3 + a] = o[a];
      w.r[i * 3 + a] = r[a];
      od[a] = (double)o[a];
      rd[a] = (double)r[a];
      w.od[i * 3 + a] = od[a];
      w.rd[i * 3 + a] = rd[a];
      w.col[i * 3 + a] = (T)P.col[a];
    }
    // decode_color's unit view-direction check (gs/decoders.py:96-98), in dtype
    T n2 = (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
    if (fabs((double)sqrt(n2) - 1.0) > 1e-6) atomicOr(w.status + GSB_ST_VIEWDIR, 1);
    w.dray[i] = P.depth_ray;
    w.valid[i] = P.valid;
    double farv;
    if (has_ff) {
      farv = ff;
    } else {  // _box_exit, gs/renderer.py:228-233
      double ex = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double rr = fabs(rd[a]) < 1e-12 ? 1e-12 : rd[a];
        double t1 = (G.lo[a] - od[a]) / rr;
        double t2 = (G.hi[a] - od[a]) / rr;
        double tm = t1 >= t2 ? t1 : t2;
        ex = (a == 0 || tm < ex) ? tm : ex;
      }
      farv = ex <= max_depth ? ex : max_depth;
    }
    double nf = nearv + 0.05;
    farv = farv >= nf ? farv : nf;
    w.nearv[i] = nearv;
    w.farv[i] = farv;
    s_near[t] = nearv;
    s_span[t] = farv - nearv;
  }
  // the generator work does not depend on the rays: it runs before the
  // barrier, under the setup threads' dataset reads and float64 math
  const int rl = t / TPR, q = t % TPR, ray = blk * RPB + rl;
  const bool live = ray < M;
  if (live && q < imp.n && w.imp_state) {  // importance round q: this row's first-uniform state
    Pcg g;
    g.init(imp.r[q]);
    g.advance((uint64_t)(ray_base + ray) * (uint64_t)imp.A);
    uint64_t* o = w.imp_state + ((int64_t)q * M + ray) * 2;
    o[0] = (uint64_t)(g.state >> 64);
    o[1] = (uint64_t)g.state;
  }
  // stratified_coarse (gs/sampler.py:91-107) with uniform row (ray_base + ray)
  constexpr int kU = 16;  // uniforms drawn ahead of the barrier
  const int chunk = (Nc + TPR - 1) / TPR, j0 = q * chunk, j1 = min(Nc, j0 + chunk);
  Pcg g;
  double u[kU];
  if (live && j0 < j1) {
    g.init(rng);
    g.advance((uint64_t)(ray_base + ray) * (uint64_t)Nc + (uint64_t)j0);
#pragma unroll
    for (int k = 0; k < kU; ++k)
      if (j0 + k < j1) u[k] = g.next_double();
  }
  __syncthreads();
  if (!live || j0 >= j1) return;
  const double nv = s_near[rl], span = s_span[rl];
  double* dep = w.dep[0] + (int64_t)ray * w.ld;
#pragma unroll
  for (int k = 0; k < kU; ++k)
    if (j0 + k < j1) dep[j0 + k] = nv + span * (((double)(j0 + k) + u[k]) / (double)Nc);
  for (int j = j0 + kU; j < j1; ++j) {  // long rows (Nc > 8 kU): the rest after the barrier
    const double uu = g.next_double();
    dep[j] = nv + span * (((double)j + uu) / (double)Nc);
  }
}
template <typename T>
__global__ void __launch_bounds__(128) k_ray_setup(gsb_dataset_t D, const int64_t* __restrict__ ids, int M,
                                                   int ray_base, Ws<T> w, Geo G, int Nc, double nearv,
                                                   double max_depth, int has_ff, double ff, gsb_pcg64_t rng,
                                                   PcgRounds imp, int nfin) {
  ray_setup_block<T>(D, ids, M, ray_base, w, G, Nc, nearv, max_depth, has_ff, ff, rng, imp, blockIdx.x, nfin);
}

// ---------------------------------------------------------------------------
// no-grad SDF at listed samples (importance passes)

template <typename T, class S, bool EXACT>
__global__ void __launch_bounds__(128) k_sdf_eval(Ws<T> w, Geo G, int M, int Nc,
                                                  const double* __restrict__ dep,
                                                  double* __restrict__ phi,
                                                  const int32_t* __restrict__ list,
                                                  const int32_t* __restrict__ list_count,
                                                  const T* __restrict__ mlp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sw = reinterpret_cast<T*>(smem_raw);
  stage_weights<T, S>(sw, mlp, 0, S::NG);
  __syncthreads();
  const int64_t total = list ? (int64_t)(*list_count) : (int64_t)M * Nc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int ray, slot;
    if (list) {
      const int32_t e = list[t];
      ray = e / GSB_KMAX;
      slot = e % GSB_KMAX;
    } else {
      ray = (int)((uint32_t)t / (uint32_t)Nc);
      slot = (int)((uint32_t)t % (uint32_t)Nc);
    }
    const double d = dep[(int64_t)ray * w.ld + slot];
    // phi_at: clip(o + d r) in float64, then cast (gs/renderer.py:323-326)
    T p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double x = w.od[ray * 3 + a] + d * w.rd[ray * 3 + a];
      x = x >= G.lo[a] ? x : G.lo[a];
      x = x <= G.hi[a] ? x : G.hi[a];
      p[a] = (T)x;
    }
    T z[S::IN_G];
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      const Loc q = locate<EXACT>(G.lv[l], (double)p[0], (double)p[1], (double)p[2], w.status);
      gather_fast<T, S::CG>(G.lv[l], compact<T>(q), z + l * S::CG);
    }
    T h0[GSB_HID], h1[GSB_HID];
    dense_fwd<T, S::IN_G>(sw + S::oGW0, sw + S::oGb0, z, h0);
    relu_mask(h0);
    dense_fwd<T, GSB_HID>(sw + S::oGW1, sw + S::oGb1, h0, h1);
    relu_mask(h1);
    const T f = dot32(sw + S::oGW2, h1) + sw[S::oGb2];
    phi[(int64_t)ray * w.ld + slot] = (double)f;
  }
}

// ---------------------------------------------------------------------------
// one importance round, thread per ray (render_weights_data +
// importance_refine_with_sources + enforce_separation)

static __device__ void separation_fallback(double* row, int32_t* src, int k) {
  // gs/sampler.py:172-197 for one row: collapse near-duplicates, then
  // re-split the largest gaps (first maximum) until k samples again.
  double kept[GSB_KMAX];
  int n = 1;
  kept[0] = row[0];
  for (int i = 1; i < k; ++i)
    if (row[i] - kept[n - 1] >= 1e-9) kept[n++] = row[i];
  while (n < k) {
    int j = 0;
    double best = kept[1] - kept[0];
    for (int t = 1; t < n - 1; ++t) {
      double dlt = kept[t + 1] - kept[t];
      if (dlt > best) {
        best = dlt;
        j = t;
      }
    }
    for (int t = n; t > j + 1; --t) kept[t] = kept[t - 1];
    kept[j + 1] = kept[j] + best / 2.0;
    ++n;
  }
  for (int i = 0; i < k; ++i) {
    if (!(kept[i] == row[i])) src[i] = -1;
    row[i] = kept[i];
  }
}

// ---------------------------------------------------------------------------
// smoothness points (renderer.draw_smooth_points, gs/renderer.py:243-276)
// from the host's RNG draws: pick = integers(0, n_valid, S), jitter =
// uniform(-t, t, S), nrm = normal((S, 8, 3)).  Same f64 operations in the
// same order (the build disables FMA contraction); poses are the f64
// ModelState.pose_matrices() rows (R0 exact, t rounded through the dtype).

template <typename T>
__global__ void k_smooth_points(gsb_dataset_t D, const double* __restrict__ poses,
                                const int64_t* __restrict__ row_cum, int64_t n_rows,
                                const int16_t* __restrict__ valid_u,
                                const int64_t* __restrict__ pick, const double* __restrict__ jitter,
                                const double* __restrict__ nrm, int S, double delta, Geo G,
                                T* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  // k-th valid pixel in np.nonzero order: row by the inclusive prefix counts,
  // then the r-th valid column of that row
  const int64_t k = pick[i];
  int64_t lo = 0, hi = n_rows;  // first row with cum > k
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (row_cum[mid] > k) hi = mid; else lo = mid + 1;
  }
  const int64_t row = lo;
  const int64_t r = k - (row > 0 ? row_cum[row - 1] : 0);
  const int64_t f = row / D.height;
  const int v = (int)(row % D.height);
  const uint16_t* drow = D.depth_mm + row * D.width;
  const int u = valid_u[row * D.width + r];  // r-th valid column (per-row compacted index)
  // pixel ray and z -> ray-distance scale (gs/camera.py:142-171)
  const double dx = ((double)u - D.cx) / D.fx;
  const double dy = ((double)v - D.cy) / D.fy;
  const double dz = 1.0;
  const double n0 = sqrt((dx * dx + dy * dy) + dz * dz);
  const double dc[3] = {dx / n0, dy / n0, dz / n0};
  const double depth_ray = ((double)drow[u] / 1000.0) * n0 + jitter[i];
  const double* P = poses + f * 12;
  double x[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    // np.einsum("nij,nj->ni") sums this 3-term contraction as (t0 + t2) + t1
    // (numpy 2.3 two-accumulator loop; measured, 100% of 180k cases)
    const double dir = (P[3 * a] * dc[0] + P[3 * a + 2] * dc[2]) + P[3 * a + 1] * dc[1];
    double xa = P[9 + a] + depth_ray * dir;
    xa = xa >= G.lo[a] ? xa : G.lo[a];
    x[a] = xa <= G.hi[a] ? xa : G.hi[a];
  }
  // first of 8 unit directions whose delta-step stays in the box, else the first
  double xe[3];
  bool found = false;
  for (int j = 0; j < 8; ++j) {
    const double* e = nrm + ((int64_t)i * 8 + j) * 3;
    const double en = sqrt((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2]);
    double c[3];
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c[a] = x[a] + delta * (e[a] / en);
      ok = ok && c[a] >= G.lo[a] && c[a] <= G.hi[a];
    }
    if (j == 0 || (ok && !found)) {
#pragma unroll
      for (int a = 0; a < 3; ++a) xe[a] = c[a];
    }
    if (ok && !found) found = true;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double c = xe[a] >= G.lo[a] ? xe[a] : G.lo[a];
    c = c <= G.hi[a] ? c : G.hi[a];
    out[(int64_t)i * 3 + a] = (T)x[a];
    out[((int64_t)S + i) * 3 + a] = (T)c;
  }
}

// ---------------------------------------------------------------------------
// one importance round (render_weights_data + importance_refine_with_sources
// + enforce_separation, gs/renderer.py:162-173, gs/sampler.py:128-197) for a
// ray handled by a group of G lanes of a warp (32 / G rays per warp).  The
// two float64 recurrences (cumprod of the transmittance, cumsum of the CDF)
// run serially on the group's first lane so they round exactly like numpy;
// the G-lane groups of a warp run their serial chains side by side, so a
// warp retires 32 / G of them at once.  Everything else is lane-parallel
// within the group: sigmoid ratios, CDF normalisation, inverse-CDF draws, the
// stable merge (by rank), the separation test and provenance.

// per-ray scratch in shared memory, `ld` >= K + A entries per array
struct ImpRow {
  double* a;    // sigmoid values, then om, then the CDF (in place)
  double* out;  // merged depths
  double* d;    // the input depth row, staged once
  double* nw;   // new depths (A), in draw order
  double* ns;   // the same, sorted (stable)
  int32_t* src; // provenance (-1 = new / moved)
};
__host__ __device__ constexpr size_t imp_row_bytes(int ld, int A) {
  return (size_t)ld * 8 * 3 + (size_t)((A + 1) / 2 * 2) * 8 * 2 + (size_t)(ld + 3) / 4 * 4 * 4;
}
__device__ __forceinline__ ImpRow imp_row(unsigned char* base, int ld, int A) {
  ImpRow r;
  r.a = reinterpret_cast<double*>(base);
  r.out = r.a + ld;
  r.d = r.out + ld;
  r.nw = r.d + ld;
  r.ns = r.nw + (A + 1) / 2 * 2;
  r.src = reinterpret_cast<int32_t*>(r.ns + (A + 1) / 2 * 2);
  return r;
}

template <int G>
struct LaneGroup {
  int gl;        // lane in the group
  unsigned gm;   // the group's lanes
  __device__ __forceinline__ LaneGroup() {
    const int lane = threadIdx.x & 31;
    gl = lane % G;
    gm = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
  }
  __device__ __forceinline__ void sync() const { __syncwarp(gm); }
  template <typename V>
  __device__ __forceinline__ V bcast(V v) const { return __shfl_sync(gm, v, 0, G); }
  __device__ __forceinline__ bool all(bool p) const { return (__ballot_sync(gm, p) & gm) == gm; }
  __device__ __forceinline__ bool any(bool p) const { return (__ballot_sync(gm, p) & gm) != 0u; }
  __device__ __forceinline__ int sum(int v) const {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gm, v, o, G);
    return v;
  }
};

// d, ph: (K) input row; win: optional given weights (K); uni: optional
// uniforms (A) else PCG64 at row * A (row_state: that state precomputed);
// writes R.out / R.src (K + A).  WOUT: also the rendering weights to wout.
template <int G, bool WOUT>
static __device__ void importance_group(const LaneGroup<G>& grp, const ImpRow& R, int K, int A,
                                        const double* __restrict__ d, const double* __restrict__ ph,
                                        const double* __restrict__ win, double s, double nearv,
                                        double farv, const gsb_pcg64_t& rng, uint64_t row,
                                        const double* __restrict__ uni, double* __restrict__ wout,
                                        const uint64_t* __restrict__ row_state = nullptr) {
  const int gl = grp.gl;
  double total = 0.0;
  double* cdf = R.a;
  for (int i = gl; i < K; i += G) R.d[i] = d[i];  // read the row once
  d = R.d;
  if (win) {
    if (gl == 0) {
      double c = 0.0;
      for (int i = 0; i < K - 1; ++i) {
        c = (i == 0) ? win[i] : c + win[i];
        cdf[i] = c;
      }
      total = c;
    }
  } else {
    // om_i = min(sig_{i+1} / max(sig_i, 1e-12), 1): sigmoids into out, om into a
    for (int i = gl; i < K; i += G) R.out[i] = sigmoid_raw(s * ph[i]);
    grp.sync();
    for (int i = gl; i < K - 1; i += G) {
      const double den = R.out[i] >= 1e-12 ? R.out[i] : 1e-12;
      const double ratio = R.out[i + 1] / den;
      R.a[i] = ratio <= 1.0 ? ratio : 1.0;
    }
    grp.sync();
    if (gl == 0) {  // sequential cumprod / cumsum, as numpy; the CDF overwrites om in place
      double trans = 1.0, c = 0.0;
      int i = 0;
      for (; i + 4 <= K - 1; i += 4) {
        const double2 o01 = *reinterpret_cast<const double2*>(R.a + i);
        const double2 o23 = *reinterpret_cast<const double2*>(R.a + i + 2);
        const double om4[4] = {o01.x, o01.y, o23.x, o23.y};
        double c4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double wi = trans * (1.0 - om4[q]);
          if constexpr (WOUT) wout[i + q] = wi;
          c = (i + q == 0) ? wi : c + wi;
          c4[q] = c;
          trans = trans * om4[q];
        }
        *reinterpret_cast<double2*>(cdf + i) = make_double2(c4[0], c4[1]);
        *reinterpret_cast<double2*>(cdf + i + 2) = make_double2(c4[2], c4[3]);
      }
      for (; i < K - 1; ++i) {
        const double om = R.a[i];
        const double wi = trans * (1.0 - om);
        if constexpr (WOUT) wout[i] = wi;
        c = (i == 0) ? wi : c + wi;
        cdf[i] = c;
        trans = trans * om;
      }
      if constexpr (WOUT) wout[K - 1] = trans * (1.0 - 1.0);
      total = c;
    }
  }
  total = grp.bcast(total);
  grp.sync();
  const bool dead = total <= 0.0;
  if (dead)
    for (int i = gl; i < K - 1; i += G) cdf[i] = (double)(i + 1);
  grp.sync();
  const double last = cdf[K - 2];
  grp.sync();
  for (int i = gl; i < K - 1; i += G) cdf[i] = cdf[i] / last;
  grp.sync();
  // inverse-CDF draws
  for (int a = gl; a < A; a += G) {
    double u;
    if (uni) {
      u = uni[a];
    } else {
      Pcg g;
      g.init(rng);
      if (row_state) {  // state at row * A precomputed (k_ray_setup): a short jump
        g.state = ((u128)row_state[0] << 64) | (u128)row_state[1];
        g.advance((uint64_t)a);
      } else {
        g.advance(row * (uint64_t)A + (uint64_t)a);
      }
      u = g.next_double();
    }
    int lo = 0, hi = K - 1;  // idx = #(cdf <= u): upper bound on a non-decreasing array
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
    }
    const int idx = lo < K - 2 ? lo : K - 2;
    const double clo = idx > 0 ? cdf[idx - 1] : 0.0, chi = cdf[idx];
    double frac;
    if (chi > clo) {
      double den = chi - clo;
      den = den >= 1e-300 ? den : 1e-300;
      frac = (u - clo) / den;
    } else {
      frac = 0.5;
    }
    double v = d[idx] + frac * (d[idx + 1] - d[idx]);
    if (dead) v = nearv + u * (farv - nearv);
    R.nw[a] = v;
  }
  grp.sync();
  // stable merge (np.argsort kind="stable": old columns precede new on ties)
  bool sorted = true;
  for (int i = gl; i + 1 < K; i += G)
    if (!(d[i] <= d[i + 1])) sorted = false;
  sorted = grp.all(sorted);
  const int n = K + A;
  if (sorted) {
    // new samples: stable rank among themselves (the draw index breaks
    // ties) and #(old <= v); then the sorted copy for the old samples' counts
    for (int a = gl; a < A; a += G) {
      const double v = R.nw[a];
      int lo = 0, hi = K;  // #(old <= v)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (d[mid] <= v) lo = mid + 1; else hi = mid;
      }
      int r = 0;
      for (int b = 0; b < A; ++b) r += (R.nw[b] < v) || (R.nw[b] == v && b < a);
      R.ns[r] = v;
      R.out[lo + r] = v;
      R.src[lo + r] = -1;
    }
    grp.sync();
    for (int i = gl; i < K; i += G) {
      const double di = d[i];
      int lo = 0, hi = A;  // #(new < di) over the sorted new samples
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (R.ns[mid] < di) lo = mid + 1; else hi = mid;
      }
      R.out[i + lo] = di;
      R.src[i + lo] = i;
    }
  } else if (gl == 0) {  // general stable insertion sort (unsorted input rows)
    for (int t = 0; t < n; ++t) {
      const double v = t < K ? d[t] : R.nw[t - K];
      const int sv = t < K ? t : -1;
      int q = t;
      while (q > 0 && R.out[q - 1] > v) {
        R.out[q] = R.out[q - 1];
        R.src[q] = R.src[q - 1];
        --q;
      }
      R.out[q] = v;
      R.src[q] = sv;
    }
  }
  grp.sync();
  bool bad = false;
  for (int i = gl; i + 1 < n; i += G)
    if (R.out[i + 1] - R.out[i] < 1e-9) bad = true;
  if (grp.any(bad) && gl == 0) separation_fallback(R.out, R.src, n);
  grp.sync();
}

constexpr int kImpG = 16;             // lanes per ray of the twin (2 rays per warp)
constexpr int kImpRaysPerBlock = 128 / kImpG;

template <typename T, int G>
__global__ void __launch_bounds__(128) k_importance_dev(Ws<T> w, int M, int K, int A, int ray_base,
                                                        const double* __restrict__ dep,
                                                        const double* __restrict__ phi,
                                                        double* __restrict__ dep_out,
                                                        double* __restrict__ phi_out,
                                                        const T* __restrict__ log_s,
                                                        gsb_pcg64_t rng, int32_t* __restrict__ evl,
                                                        int32_t* __restrict__ evl_count, int64_t cap,
                                                        int want_list, int count_final, double trunc,
                                                        const uint64_t* __restrict__ row_states) {
  extern __shared__ __align__(16) unsigned char imp_smem[];
  const LaneGroup<G> grp;
  const int gid = threadIdx.x / G;  // ray slot in the block
  const int i = blockIdx.x * (128 / G) + gid;
  const int n = K + A;
  if (i >= M) return;  // group-uniform
  const ImpRow R = imp_row(imp_smem + (size_t)gid * imp_row_bytes(n, A), n, A);
  // ModelState.s_value() = float(np.exp(log_s)) in the model dtype
  const double s = (double)exp(log_s[0]);
  const double* d = dep + (int64_t)i * w.ld;
  const double* ph = phi + (int64_t)i * w.ld;
  importance_group<G, false>(grp, R, K, A, d, ph, nullptr, s, w.nearv[i], w.farv[i], rng,
                             (uint64_t)(ray_base + i), nullptr, nullptr,
                             row_states ? row_states + (int64_t)i * 2 : nullptr);
  const int gl = grp.gl;
  double* out = dep_out + (int64_t)i * w.ld;
  double* po = phi_out + (int64_t)i * w.ld;
  int nnew = 0;
  for (int t = gl; t < n; t += G) {
    out[t] = R.out[t];
    const int sv = R.src[t];
    if (sv >= 0) po[t] = ph[sv];
    else ++nnew;
  }
  if (count_final) {  // partition counts of the final samples (as k_counts)
    const int valid = w.valid[i];
    const double D = w.dray[i];
    int ntr = 0, nfs = 0, neik = 0;
    for (int t = gl; t < n; t += G) {
      const double b = D - R.out[t];
      const bool tr = valid && fabs(b) <= trunc;
      const bool fs = valid && b > trunc;
      const bool bh = valid && b < -trunc;
      ntr += tr;
      nfs += fs;
      neik += (fs || bh || !valid);
    }
    ntr = grp.sum(ntr);
    nfs = grp.sum(nfs);
    neik = grp.sum(neik);
    if (gl == 0) {
      w.cnt[i * 3 + 0] = ntr;
      w.cnt[i * 3 + 1] = nfs;
      w.cnt[i * 3 + 2] = neik;
      atomicAdd((unsigned long long*)&w.counts[GSB_C_VALID], (unsigned long long)valid);
      atomicAdd((unsigned long long*)&w.counts[GSB_C_TR], (unsigned long long)ntr);
      atomicAdd((unsigned long long*)&w.counts[GSB_C_FS], (unsigned long long)nfs);
      atomicAdd((unsigned long long*)&w.counts[GSB_C_EIK], (unsigned long long)neik);
    }
  }
  if (!want_list) return;
  const int tot = grp.sum(nnew);
  int base = 0;
  if (gl == 0) base = atomicAdd(evl_count, tot);
  base = grp.bcast(base);
  if (base + tot > cap) {
    if (gl == 0) atomicOr(w.status + GSB_ST_OVERFLOW, 1);
    return;
  }
  // compact the new slots in order
  for (int t0 = 0; t0 < n; t0 += G) {
    const int t = t0 + gl;
    const bool isnew = t < n && R.src[t] < 0;
    const unsigned bal = __ballot_sync(grp.gm, isnew) & grp.gm;
    const unsigned below = bal & ((1u << (threadIdx.x & 31)) - 1u);
    if (isnew) evl[base + __popc(below)] = i * GSB_KMAX + t;
    base += __popc(bal);
  }
}

// twin: explicit weights or phi, explicit uniforms or generator; the same
// G-lane groups as the step kernel
static __global__ void __launch_bounds__(128) k_importance_twin(int M, int K, int A, int ld,
                                                         const double* dep, const double* phi,
                                                         const double* win, double s,
                                                         const double* nearv, const double* farv,
                                                         const double* uni, gsb_pcg64_t rng,
                                                         int use_rng, double* out, int32_t* src,
                                                         double* wts) {
  constexpr int G = kImpG;
  extern __shared__ __align__(16) unsigned char imp_smem[];
  const LaneGroup<G> grp;
  const int gid = threadIdx.x / G;
  const int i = blockIdx.x * kImpRaysPerBlock + gid;
  if (i >= M) return;
  const int n = K + A;
  const ImpRow R = imp_row(imp_smem + (size_t)gid * imp_row_bytes(n, A), n, A);
  const double* d = dep + (int64_t)i * ld;
  const double* ph = phi ? phi + (int64_t)i * ld : nullptr;
  const double* wi = win ? win + (int64_t)i * ld : nullptr;
  const double* ui = use_rng ? nullptr : uni + (int64_t)i * A;
  if (wts)
    importance_group<G, true>(grp, R, K, A, d, ph, wi, s, nearv[i], farv[i], rng, (uint64_t)i, ui,
                              wts + (int64_t)i * ld);
  else
    importance_group<G, false>(grp, R, K, A, d, ph, wi, s, nearv[i], farv[i], rng, (uint64_t)i, ui, nullptr);
  for (int t = grp.gl; t < n; t += G) {
    out[(int64_t)i * ld + t] = R.out[t];
    src[(int64_t)i * ld + t] = R.src[t];
  }
}

// ---------------------------------------------------------------------------
// partition counts (gs/renderer.py:384-412)

template <typename T>
__global__ void k_counts(Ws<T> w, int M, int N, const double* __restrict__ dep, double trunc) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  long long ntr = 0, nfs = 0, neik = 0, nval = 0;
  if (i < M) {
    int valid = w.valid[i];
    double D = w.dray[i];
    const double* d = dep + (int64_t)i * w.ld;
    for (int j = 0; j < N; ++j) {
      double b = D - d[j];
      bool tr = valid && fabs(b) <= trunc;
      bool fs = valid && b > trunc;
      bool bh = valid && b < -trunc;
      ntr += tr;
      nfs += fs;
      neik += (fs || bh || !valid);
    }
    nval = valid;
    w.cnt[i * 3 + 0] = (int32_t)ntr;
    w.cnt[i * 3 + 1] = (int32_t)nfs;
    w.cnt[i * 3 + 2] = (int32_t)neik;
  }
  ntr = warp_sum(ntr);
  nfs = warp_sum(nfs);
  neik = warp_sum(neik);
  nval = warp_sum(nval);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd((unsigned long long*)&w.counts[GSB_C_VALID], (unsigned long long)nval);
    atomicAdd((unsigned long long*)&w.counts[GSB_C_TR], (unsigned long long)ntr);
    atomicAdd((unsigned long long*)&w.counts[GSB_C_FS], (unsigned long long)nfs);
    atomicAdd((unsigned long long*)&w.counts[GSB_C_EIK], (unsigned long long)neik);
  }
}

// taped forward: phi, grad phi (gs/renderer.py:356-358), colour (:360-365)
template <typename T, class S>
struct FwdRow {
  static constexpr int oZ = 0;                              // z (IN_G) / colour input (IN_C)
  static constexpr int ZP = ((S::IN_G > S::IN_C ? S::IN_G : S::IN_C) + 3) / 4 * 4;
  static constexpr int oH = ZP;                             // hidden layer 0
  static constexpr int oD = oH + GSB_HID;                   // delta0
  static constexpr int ROW = oD + GSB_HID;
};

template <typename T, class S, bool EXACT>
__global__ void __launch_bounds__(128) k_fwd(Ws<T> w, Geo G, int M, int N,
                                             const double* __restrict__ dep,
                                             const T* __restrict__ spts, int nsp,
                                             const T* __restrict__ mlp) {
  using R = FwdRow<T, S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sw = reinterpret_cast<T*>(smem_raw);
  T* myrow = sw + (S::NMLP + 3) / 4 * 4 + (size_t)threadIdx.x * R::ROW;
  stage_weights<T, S>(sw, mlp, 0, S::NMLP);
  __syncthreads();
  const int64_t MN = (int64_t)M * N;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= MN + nsp) return;
  T p[3];
  int ray = -1;
  if (s < MN) {
    ray = (int)((uint32_t)s / (uint32_t)N);
    taped_point<T>(w.o + ray * 3, w.r + ray * 3,
                   dep[(int64_t)ray * w.ld + (int)((uint32_t)s % (uint32_t)N)], G.lo, G.hi, p);
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) p[a] = spts[(s - MN) * 3 + a];
  }
  LocT<T> loc[S::NL];
#pragma unroll
  for (int l = 0; l < S::NL; ++l) {
    loc[l] = compact<T>(locate<EXACT>(G.lv[l], (double)p[0], (double)p[1], (double)p[2], w.status));
    T f[S::CG];
    gather_fast<T, S::CG>(G.lv[l], loc[l], f);
#pragma unroll
    for (int c = 0; c < S::CG; ++c) myrow[R::oZ + l * S::CG + c] = f[c];
  }
  uint32_t m0, m1;
  T phi;
  {
    T h[GSB_HID];
    dense_f_row<T, S::IN_G>(sw + S::oGW0, myrow + R::oZ, h);
    add_bias(sw + S::oGb0, h);
    m0 = relu_mask(h);
    store32(myrow + R::oH, h);
    dense_f_row<T, GSB_HID>(sw + S::oGW1, myrow + R::oH, h);
    add_bias(sw + S::oGb1, h);
    m1 = relu_mask(h);
    phi = dot32(sw + S::oGW2, h) + sw[S::oGb2];
  }
  // grad phi: g = W0 ((W1 (W2 . m1)) . m0), then sum_l J_l^T g_l
  T gz[S::IN_G];
  {
    T d[GSB_HID];
#pragma unroll
    for (int j = 0; j < GSB_HID; ++j) d[j] = ((m1 >> j) & 1u) ? sw[S::oGW2 + j] : T(0);
    dense_d_row<T, GSB_HID>(sw + S::oGW1, d, m0, myrow + R::oD);
    load32(myrow + R::oD, d);
    dense_d_reg<T, S::IN_G>(sw + S::oGW0, d, gz);
  }
  T gr[3] = {T(0), T(0), T(0)};
#pragma unroll
  for (int l = 0; l < S::NL; ++l) level_dx_fast<T, S::CG>(G.lv[l], loc[l], gz + l * S::CG, gr);
  w.sphi[s] = phi;
#pragma unroll
  for (int a = 0; a < 3; ++a) w.sgphi[s * 3 + a] = gr[a];
  if (ray < 0) return;
  // colour: sigmoid(MLP_c([f_c, r]))  (gs/decoders.py:86-99)
  const Loc qc = locate<EXACT>(G.col, (double)p[0], (double)p[1], (double)p[2], w.status);
  {
    T f[S::CC];
    gather_fast<T, S::CC>(G.col, compact<T>(qc), f);
#pragma unroll
    for (int c = 0; c < S::CC; ++c) myrow[R::oZ + c] = f[c];
#pragma unroll
    for (int a = 0; a < 3; ++a) myrow[R::oZ + S::CC + a] = w.r[ray * 3 + a];
  }
  T h[GSB_HID];
  dense_f_row<T, S::IN_C>(sw + S::oCW0, myrow + R::oZ, h);
  add_bias(sw + S::oCb0, h);
  relu_mask(h);
  store32(myrow + R::oH, h);
  dense_f_row<T, GSB_HID>(sw + S::oCW1, myrow + R::oH, h);
  add_bias(sw + S::oCb1, h);
  relu_mask(h);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    T a = T(0);
#pragma unroll
    for (int j = 0; j < GSB_HID; ++j) a = fma(h[j], sw[S::oCW2 + j * 3 + c], a);
    w.scol[s * 3 + c] = sigmoid_fast(a + sw[S::oCb2 + c]);
  }
}

// ---------------------------------------------------------------------------
// smoothness (gs/renderer.py:428-434): loss partial + grad-phi adjoints

template <typename T>
__device__ __forceinline__ void smooth_item(Ws<T> w, int64_t MN, int S, T scale, int j) {
  if (j >= S) return;
  int64_t a = MN + j, b = MN + S + j;
  T acc = T(0);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    T dlt = w.sgphi[a * 3 + c] - w.sgphi[b * 3 + c];
    acc += dlt * dlt;
    w.ubar[a * 3 + c] = scale * dlt;
    w.ubar[b * 3 + c] = -(scale * dlt);
  }
  w.pbar[a] = T(0);
  w.pbar[b] = T(0);
  w.smooth_part[j] = (double)acc;
}

// ---------------------------------------------------------------------------
// rendering + losses + per-sample adjoints, thread per ray

struct LossW {
  double rgb, depth, sdf, fs, eik, smooth, trunc, alpha, m_global, smooth_global;
};

// ---------------------------------------------------------------------------
// rendering + losses + per-sample adjoints, one warp per ray
// (gs/renderer.py:112-159 alphas/composite, :372-414 losses)

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

template <typename T>
__device__ __forceinline__ T warp_allsum(T v) {
  return warp_sum(v);
}

constexpr int kRenderRows = 6;  // per-warp shared arrays of N values

// The smoothness pairs (k_smooth's work, nsm > 0) ride in trailing blocks
// of the same launch: one launch fewer per step.
template <typename T>
__global__ void __launch_bounds__(128, 11) k_render(Ws<T> w, int M, int N, const double* __restrict__ dep,
                                                const T* __restrict__ params, int64_t log_s_off,
                                                LossW L, int nsm = 0, int64_t MN = 0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int rblocks = (M + 3) / 4;
  if ((int)blockIdx.x >= rblocks) {  // block-uniform
    const T scale = (T)(2.0 * L.smooth) / (T)L.smooth_global;
    smooth_item<T>(w, MN, nsm, scale, ((int)blockIdx.x - rblocks) * 128 + (int)threadIdx.x);
    return;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T* sig = reinterpret_cast<T*>(smem_raw) + (size_t)wid * kRenderRows * N;
  T* trn = sig + N;
  T* xb = trn + N;
  T* yb = xb + N;
  T* alp = yb + N;  // alpha_j, kept from the forward pass
  T* rat = alp + N; // sigma_{j+1} / max(sigma_j, 1e-12), kept from the forward pass
  const int ray = blockIdx.x * (blockDim.x >> 5) + wid;
  if (ray >= M) return;  // warp-uniform
  const T s = exp(params[log_s_off]);  // ModelState.s_tensor (gs/renderer.py:83-84)
  const T SF = (T)1e-12, TF = (T)1e-15;
  const int64_t s0 = (int64_t)ray * N;
  const double* d = dep + (int64_t)ray * w.ld;
  for (int j = lane; j < N; j += 32) sig[j] = sigmoid_raw(w.sphi[s0 + j] * s);
  __syncwarp();
  // ---- forward: alphas, transmittance (exclusive scan of log(1 - alpha)), composite
  T carry = T(0), ch0 = T(0), ch1 = T(0), ch2 = T(0), dh = T(0);
  for (int j0 = 0; j0 < N; j0 += 32) {
    const int j = j0 + lane;
    T al = T(0), Lj = T(0), ratio = T(0);
    if (j < N - 1) {
      const T den = sig[j] >= SF ? sig[j] : SF;
      ratio = sig[j + 1] / den;
      al = T(1) - (ratio <= T(1) ? ratio : T(1));
    }
    if (j < N) {
      const T om = T(1) - al;
      Lj = log(om >= TF ? om : TF);
      alp[j] = al;
      rat[j] = ratio;
    }
    const T incl = warp_incl_scan(Lj);
    const T Tj = (j == 0) ? T(1) : exp(carry + (incl - Lj));
    carry += __shfl_sync(0xffffffffu, incl, 31);
    if (j < N) {
      trn[j] = Tj;
      const T wj = Tj * al;
      w.wts[s0 + j] = wj;
      const T* cj = w.scol + (s0 + j) * 3;
      ch0 = fma(wj, cj[0], ch0);
      ch1 = fma(wj, cj[1], ch1);
      ch2 = fma(wj, cj[2], ch2);
      dh = fma(wj, (T)d[j], dh);
    }
  }
  ch0 = warp_sum(ch0);
  ch1 = warp_sum(ch1);
  ch2 = warp_sum(ch2);
  dh = warp_sum(dh);
  // ---- losses
  const int valid = w.valid[ray];
  const double D = w.dray[ray];
  const T err0 = ch0 - w.col[ray * 3], err1 = ch1 - w.col[ray * 3 + 1], err2 = ch2 - w.col[ray * 3 + 2];
  const T lrgb = sqrt(((err0 * err0 + err1 * err1) + err2 * err2) + (T)1e-24);
  const T dT = (T)D;
  const T lde = valid ? fabs(dh - dT) : T(0);
  const long long nvalid = w.counts[GSB_C_VALID];
  const long long neik = w.counts[GSB_C_EIK];
  const T inv_nv = T(1) / (T)(nvalid > 1 ? nvalid : 1);
  const T inv_ne = T(1) / (T)(neik > 1 ? neik : 1);
  const T ntr = (T)max(w.cnt[ray * 3 + 0], 1), nfs = (T)max(w.cnt[ray * 3 + 1], 1);
  const T alpha = (T)(-L.alpha);
  T sdf = T(0), fsv = T(0), eik = T(0);
  for (int j = lane; j < N; j += 32) {
    const double b = D - d[j];
    const T bc = (T)b, ph = w.sphi[s0 + j];
    const bool tr = valid && fabs(b) <= L.trunc;
    const bool fs = valid && b > L.trunc;
    const bool bh = valid && b < -L.trunc;
    if (tr) sdf += fabs(ph - bc);
    if (fs) {
      const T e = exp(ph * alpha);
      T inner = e - T(1);
      inner = T(0) >= inner ? T(0) : inner;
      const T lin = ph - bc;
      fsv += inner >= lin ? inner : lin;
    }
    if (fs || bh || !valid) {
      const T* gp = w.sgphi + (s0 + j) * 3;
      const T nn = sqrt(((gp[0] * gp[0] + gp[1] * gp[1]) + gp[2] * gp[2]) + (T)1e-20);
      const T df = T(1) - nn;
      eik += df * df;
    }
  }
  sdf = warp_sum(sdf);
  fsv = warp_sum(fsv);
  eik = warp_sum(eik);
  // ---- backward seeds
  const T Mg = (T)L.m_global;
  const T chb0 = ((T)L.rgb / Mg) * err0 / lrgb, chb1 = ((T)L.rgb / Mg) * err1 / lrgb,
          chb2 = ((T)L.rgb / Mg) * err2 / lrgb;
  const T dhb = valid ? (T)L.depth * sgn(dh - dT) * inv_nv : T(0);
  const T ksdf = ((T)L.sdf / Mg) / ntr, kfs = ((T)L.fs / Mg) / nfs;
  const T keik = (T)(-2.0 * L.eik) * inv_ne;
  // pass A: w_bar, c_bar, T_bar T; suffix sums L_bar_j = sum_{i>j} T_bar_i T_i
  T tot = T(0);
  for (int j0 = 0; j0 < N; j0 += 32) {
    const int j = j0 + lane;
    T tt = T(0);
    if (j < N) {
      const T al = alp[j];
      const T Tj = trn[j];
      const T wj = Tj * al;
      const T* cj = w.scol + (s0 + j) * 3;
      const T wbar = ((chb0 * cj[0] + chb1 * cj[1]) + chb2 * cj[2]) + dhb * (T)d[j];
      T* cb = w.cbar + (s0 + j) * 3;
      cb[0] = wj * chb0;
      cb[1] = wj * chb1;
      cb[2] = wj * chb2;
      tt = (wbar * al) * Tj;
      xb[j] = wbar;  // keep w_bar for pass B
    }
    const T incl = warp_incl_scan(tt);
    if (j < N) yb[j] = tot + incl;  // inclusive prefix P_j
    tot += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
  // pass B: sigma_bar contributions (own D-bar part, and r_bar_j / D_j to j+1)
  for (int j0 = 0; j0 < N; j0 += 32) {
    const int j = j0 + lane;
    T own = T(0), fwd = T(0);
    if (j < N) {
      const T al = alp[j], ratio = rat[j];
      const T den = (j < N - 1) ? (sig[j] >= SF ? sig[j] : SF) : T(1);
      const T om = T(1) - al;
      const T Lbar = tot - yb[j];
      const T ombar = om >= TF ? Lbar / om : T(0);
      const T abar = xb[j] * trn[j] - ombar;
      if (j < N - 1) {
        const T rbar = ratio <= T(1) ? -abar : T(0);
        fwd = rbar / den;
        own = sig[j] >= SF ? -(rbar * sig[j + 1]) / (den * den) : T(0);
      }
    }
    __syncwarp();
    if (j < N) {
      xb[j] = fwd;   // contribution to sigma_bar_{j+1}
      yb[j] = own;   // contribution to sigma_bar_j
    }
  }
  __syncwarp();
  // pass C: phi_bar, u (eikonal), log_s partial
  T logs = T(0);
  for (int j = lane; j < N; j += 32) {
    const T sg = sig[j];
    const T sbar = yb[j] + (j > 0 ? xb[j - 1] : T(0));
    const T zb = sbar * (sg * (T(1) - sg));
    const T ph = w.sphi[s0 + j];
    logs += zb * ph;
    const double b = D - d[j];
    T pb = zb * s;
    if (valid && fabs(b) <= L.trunc) pb += ksdf * sgn(ph - (T)b);
    const bool fs = valid && b > L.trunc, bh = valid && b < -L.trunc;
    if (fs) {
      const T e = exp(ph * alpha);
      const T inner = e - T(1);
      const T inner0 = T(0) >= inner ? T(0) : inner;
      const T dfs = inner0 >= ph - (T)b ? (inner > T(0) ? e * alpha : T(0)) : T(1);
      pb += kfs * dfs;
    }
    w.pbar[s0 + j] = pb;
    const T* gp = w.sgphi + (s0 + j) * 3;
    T* ub = w.ubar + (s0 + j) * 3;
    if (fs || bh || !valid) {
      const T nn = sqrt(((gp[0] * gp[0] + gp[1] * gp[1]) + gp[2] * gp[2]) + (T)1e-20);
      const T k = keik * (T(1) - nn) / nn;
      ub[0] = k * gp[0];
      ub[1] = k * gp[1];
      ub[2] = k * gp[2];
    } else {
      ub[0] = T(0);
      ub[1] = T(0);
      ub[2] = T(0);
    }
  }
  logs = warp_sum(logs);
  if (lane == 0) {
    double* part = w.ray_part + (int64_t)ray * 8;
    part[0] = (double)lrgb;
    part[1] = (double)lde;
    part[2] = (double)(sdf / ntr);
    part[3] = (double)(fsv / nfs);
    part[4] = (double)eik;
    part[5] = (double)logs;
  }
}

// ---------------------------------------------------------------------------
// backward, geometry: grid scatter + geometry MLP weight gradients.
// Thread per sample.  Each thread's shared-memory row holds its activations
// and, at the end, its outer-product factors; every warp then accumulates
// the 32 samples' outer products with lane j owning output column j.
// One round of corner loads per sample: z = sum_k w_k theta_k and
// v = sum_k ju_k theta_k are formed together (p, u are known up front).

template <typename T, class S>
struct GeoRow {
  static constexpr int A0 = S::IN_G + 1;            // z, then [p z + v, p]
  static constexpr int A0P = (A0 + 3) / 4 * 4;
  static constexpr int oA0 = 0;
  static constexpr int oB0 = oA0 + A0P;             // delta0
  static constexpr int oA1 = oB0 + GSB_HID;         // h0, then [p h0 + q0, p]
  static constexpr int A1P = (GSB_HID + 1 + 3) / 4 * 4;
  static constexpr int oV2 = oA1 + A1P;             // p h1 + dd1 (.) m1
  static constexpr int oQ = oV2 + GSB_HID;          // v (IN_G), then q0 (32)
  static constexpr int oM = oQ + GSB_HID;           // m1 bits
  static constexpr int ROW = oM + 4;
};

// Grid scatter theta[idx_k] += g (coef_k) for one level, reduced within the
// warp first: samples of a ray are depth-ordered, so lanes sharing a cell
// form contiguous runs; each run is summed with a segmented shuffle scan and
// its first lane issues one vector red per corner.  Inactive lanes form
// their own (empty) runs.
// Deterministic mode: entry slot (sample, level) records its 8 corner rows
// (address key + C values); k_det_reduce sums each row's entries in slot
// order after a stable sort, so the result does not depend on scheduling.
template <typename T, int C>
__device__ __forceinline__ void det_put(uint64_t* keys, T* vals, int64_t slot, const LevelDev& L,
                                        int64_t base, const T* gl, const T (&coef)[8], bool active) {
  if (!active) return;  // unused slots keep the ~0 key they were initialised with
  T* Gp = reinterpret_cast<T*>(L.grad) + base * C;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t e = slot * 8 + k;
    keys[e] = (uint64_t)(uintptr_t)(Gp + corner_off(L, k) * C);
#pragma unroll
    for (int c = 0; c < C; ++c) vals[e * 8 + c] = gl[c] * coef[k];
  }
}

template <typename T, int C>
__device__ __forceinline__ void scatter_level(const LevelDev& L, const LocT<T>& q, const T* gl,
                                              const T (&coef)[8], bool active, bool no_merge,
                                              uint64_t* dkeys = nullptr, T* dvals = nullptr,
                                              int64_t dslot = 0) {
  if (dkeys) {
    det_put<T, C>(dkeys, dvals, dslot, L, (int64_t)q.base, gl, coef, active);
    return;
  }
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int key = active ? q.base : (-2 - lane);
  const int prev = __shfl_up_sync(full, key, 1);
  const bool head = lane == 0 || key != prev;
  const unsigned heads = no_merge ? full : __ballot_sync(full, head);
  T* Gp = reinterpret_cast<T*>(L.grad) + (int64_t)q.base * C;
  if (heads == full) {  // no shared cells in this warp (or no_merge): one red per lane
    if (!active) return;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      T v[C];
#pragma unroll
      for (int c = 0; c < C; ++c) v[c] = gl[c] * coef[k];
      red_row<T, C>(Gp + corner_off(L, k) * C, v);
    }
    return;
  }
  if (heads == 1u) {  // one cell for the whole warp (coarse levels): butterfly
    // reduce-scatters of the 8 x C values in chunks of 32 (31 shuffles per
    // chunk instead of 5 x 8C for the scan); lane l then adds value
    // 32 chunk + l = (corner, channel).  Extending this to 2-3 long runs per
    // warp measured slower (379 vs 372 us bwd_geom).
    constexpr int V = 8 * C;
#pragma unroll
    for (int ch = 0; ch < (V + 31) / 32; ++ch) {
      T v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int j = ch * 32 + i;
        v[i] = j < V ? gl[j % C] * coef[j / C] : T(0);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
          const T send = up ? v[i] : v[i + o];
          v[i] = (up ? v[i + o] : v[i]) + __shfl_xor_sync(full, send, o);
        }
      }
      if constexpr (C == 4 && sizeof(T) == 4) {
        // lanes 4k..4k+3 hold corner k's four channels: one 16-byte red per
        // corner from lane 4k (a vector red costs about what a scalar one
        // does in L2: tools/mb_red.cu, 126 vs 47 G updates/s)
        const T x1 = __shfl_down_sync(full, v[0], 1);
        const T x2 = __shfl_down_sync(full, v[0], 2);
        const T x3 = __shfl_down_sync(full, v[0], 3);
        if ((lane & 3) == 0) red_add_v4(Gp + corner_off(L, lane >> 2) * 4, v[0], x1, x2, x3);
      } else {
        const int j = ch * 32 + lane;
        if (j < V) atomicAdd(Gp + corner_off(L, j / C) * C + j % C, v[0]);
      }
    }
    return;
  }
  // end of my run (exclusive): next head after `lane`, or 32
  const unsigned after = lane == 31 ? 0u : (heads >> (lane + 1));
  const int run_end = after ? lane + __ffs(after) : 32;
  // scan steps bounded by the warp's longest run (fine levels: 1-2 lanes)
  const int maxrun = (int)__reduce_max_sync(full, head ? (unsigned)(run_end - lane) : 0u);
  // all 8 corners x C channels scan together (8C independent shuffle chains)
  T v[8][C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const T gc = active ? gl[c] : T(0);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k][c] = gc * coef[k];
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    if (o >= maxrun) break;
    const bool take = lane + o < run_end;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T y = __shfl_down_sync(full, v[k][c], o);
        if (take) v[k][c] += y;
      }
  }
  if (head && active) {
#pragma unroll
    for (int k = 0; k < 8; ++k) red_row<T, C>(Gp + corner_off(L, k) * C, v[k]);
  }
}

// corner weights w_k and their u-directional derivatives ju_k (world units),
// gs/diffcore.py:761-767, 874-890
template <typename T>
__device__ __forceinline__ void corner_w_ju(const LocT<T>& q, T iv, const T (&u)[3], T (&wk)[8],
                                            T (&ju)[8]) {
  const T x1 = q.fx, y1 = q.fy, z1 = q.fz;
  const T x0 = T(1) - x1, y0 = T(1) - y1, z0 = T(1) - z1;
  const T u0 = u[0] * iv, u1 = u[1] * iv, u2 = u[2] * iv;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int dx = (k >> 2) & 1, dy = (k >> 1) & 1, dz = k & 1;
    const T wx = dx ? x1 : x0, wy = dy ? y1 : y0, wz = dz ? z1 : z0;
    const T sx = dx ? T(1) : T(-1), sy = dy ? T(1) : T(-1), sz = dz ? T(1) : T(-1);
    wk[k] = (wx * wy) * wz;
    ju[k] = (sx * wy * wz) * u0 + (wx * sy * wz) * u1 + (wx * wy * sz) * u2;
  }
}

// warp outer products: acc0[i] += A0[r][i] B0[r][lane], acc1[i] += A1[r][i] B1[r][lane]
template <typename T, int NA0, int NA0P, int NA1, int NA1P>
__device__ __forceinline__ void warp_outer(const T* rows, int ROW, int oA0, int oB0, int oA1,
                                           int oB1, int lane, T (&acc0)[NA0], T (&acc1)[NA1]) {
#pragma unroll 1
  for (int r = 0; r < 32; ++r) {
    const T* rw = rows + (size_t)r * ROW;
    const T b0 = rw[oB0 + lane], b1 = rw[oB1 + lane];
#pragma unroll
    for (int i = 0; i < NA0P; i += 4) {
      T a0, a1, a2, a3;
      lds4(rw + oA0 + i, a0, a1, a2, a3);
      if (i < NA0) acc0[i] = fma(a0, b0, acc0[i]);
      if (i + 1 < NA0) acc0[i + 1] = fma(a1, b0, acc0[i + 1]);
      if (i + 2 < NA0) acc0[i + 2] = fma(a2, b0, acc0[i + 2]);
      if (i + 3 < NA0) acc0[i + 3] = fma(a3, b0, acc0[i + 3]);
    }
#pragma unroll
    for (int i = 0; i < NA1P; i += 4) {
      T a0, a1, a2, a3;
      lds4(rw + oA1 + i, a0, a1, a2, a3);
      if (i < NA1) acc1[i] = fma(a0, b1, acc1[i]);
      if (i + 1 < NA1) acc1[i + 1] = fma(a1, b1, acc1[i + 1]);
      if (i + 2 < NA1) acc1[i + 2] = fma(a2, b1, acc1[i + 2]);
      if (i + 3 < NA1) acc1[i + 3] = fma(a3, b1, acc1[i + 3]);
    }
  }
}

template <typename T, class S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_bwd_geom(Ws<T> w, Geo G, int M, int N,
                                                        const double* __restrict__ dep,
                                                        const T* __restrict__ spts, int nsp,
                                                        int agg_levels,
                                                        const T* __restrict__ mlp) {
  using R = GeoRow<T, S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sw = reinterpret_cast<T*>(smem_raw);                 // geometry weights
  T* sm = sw + ((S::NG + 3) / 4 * 4);                      // per-warp rows
  stage_weights<T, S>(sw, mlp, 0, S::NG);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T* rows = sm + (size_t)wid * 32 * R::ROW;
  T* myrow = rows + (size_t)lane * R::ROW;
  const int64_t MN = (int64_t)M * N, NS = MN + nsp;
  T acc0[R::A0], acc1[GSB_HID + 1], acc2 = T(0), accp = T(0);
#pragma unroll
  for (int i = 0; i < R::A0; ++i) acc0[i] = T(0);
#pragma unroll
  for (int i = 0; i <= GSB_HID; ++i) acc1[i] = T(0);
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  // per-sample inputs, prefetched one batch ahead
  auto fetch = [&](int64_t s, T& p, T (&u)[3], T (&pt)[3]) {
    if (s < NS) {
      p = w.pbar[s];
#pragma unroll
      for (int a = 0; a < 3; ++a) u[a] = w.ubar[s * 3 + a];
      if (s < MN) {
        const int ray = (int)((uint32_t)s / (uint32_t)N);
        taped_point<T>(w.o + ray * 3, w.r + ray * 3,
                       dep[(int64_t)ray * w.ld + (int)((uint32_t)s % (uint32_t)N)], G.lo, G.hi, pt);
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) pt[a] = spts[(s - MN) * 3 + a];
      }
    } else {  // inactive lanes evaluate a valid point and contribute zero
      p = T(0);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        u[a] = T(0);
        pt[a] = (T)G.lo[a];
      }
    }
  };
  int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * 32;
  T np, nu[3], npt[3];
  fetch(base + lane, np, nu, npt);
  for (; base < NS; base += nwarps * 32) {
    const int64_t s = base + lane;
    const bool active = s < NS;
    T p = np, u[3] = {nu[0], nu[1], nu[2]}, pt[3] = {npt[0], npt[1], npt[2]};
    fetch(base + nwarps * 32 + lane, np, nu, npt);
    // ---- one pass over the corners: z (-> row), v (-> row)
    LocT<T> loc[S::NL];
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      const LevelDev& L = G.lv[l];
      loc[l] = compact<T>(locate<false>(L, (double)pt[0], (double)pt[1], (double)pt[2], nullptr));
      T wk[8], ju[8];
      corner_w_ju(loc[l], (T)L.inv_vs, u, wk, ju);
      const T* F = reinterpret_cast<const T*>(L.feat) + (int64_t)loc[l].base * S::CG;
      T zl[S::CG], vl[S::CG];
#pragma unroll
      for (int c = 0; c < S::CG; ++c) zl[c] = vl[c] = T(0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        T row[S::CG];
        load_row<T, S::CG>(F + corner_off(L, k) * S::CG, row);
#pragma unroll
        for (int c = 0; c < S::CG; ++c) {
          zl[c] = fma(wk[k], row[c], zl[c]);
          vl[c] = fma(ju[k], row[c], vl[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < S::CG; ++c) {
        myrow[R::oA0 + l * S::CG + c] = zl[c];
        myrow[R::oQ + l * S::CG + c] = vl[c];
      }
    }
    // ---- forward, then delta0 and g = dphi/dz
    uint32_t m0, m1;
    {
      T h[GSB_HID];
      dense_f_row<T, S::IN_G>(sw + S::oGW0, myrow + R::oA0, h);
      add_bias(sw + S::oGb0, h);
      m0 = relu_mask(h);
      store32(myrow + R::oA1, h);                          // raw h0 (layer input)
      dense_f_row<T, GSB_HID>(sw + S::oGW1, myrow + R::oA1, h);
      add_bias(sw + S::oGb1, h);
      m1 = relu_mask(h);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) h[j] *= p;
      store32(myrow + R::oV2, h);                          // p h1
    }
    T gz[S::IN_G];
    {
      T d[GSB_HID];
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) d[j] = ((m1 >> j) & 1u) ? sw[S::oGW2 + j] : T(0);
      dense_d_row<T, GSB_HID>(sw + S::oGW1, d, m0, myrow + R::oB0);   // delta0
      load32(myrow + R::oB0, d);
      dense_d_reg<T, S::IN_G>(sw + S::oGW0, d, gz);        // g = dphi/dz
    }
    // ---- grid scatter: theta_l[idx_k] += g_l (p w_k + ju_k)
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      T wk[8], ju[8], coef[8];
      corner_w_ju(loc[l], (T)G.lv[l].inv_vs, u, wk, ju);
#pragma unroll
      for (int k = 0; k < 8; ++k) coef[k] = fma(p, wk[k], ju[k]);
      scatter_level<T, S::CG>(G.lv[l], loc[l], gz + l * S::CG, coef, active, false, w.det_keys,
                              w.det_vals, s * (S::NL + 1) + l);
    }
    // ---- A0 = [p z + v, p]; q0 = (v W0) (.) m0; A1 = [p h0 + q0, p]; V2 += dd1 (.) m1
    {
      T q0[GSB_HID];
      dense_f_row<T, S::IN_G>(sw + S::oGW0, myrow + R::oQ, q0);  // v W0
#pragma unroll
      for (int i = 0; i < S::IN_G; ++i)
        myrow[R::oA0 + i] = fma(p, myrow[R::oA0 + i], myrow[R::oQ + i]);
      myrow[R::oA0 + S::IN_G] = p;
      T a[GSB_HID];
      load32(myrow + R::oA1, a);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) {
        q0[j] = ((m0 >> j) & 1u) ? q0[j] : T(0);
        a[j] = fma(p, a[j], q0[j]);
      }
      store32(myrow + R::oA1, a);
      myrow[R::oA1 + GSB_HID] = p;
      store32(myrow + R::oQ, q0);
      dense_f_row<T, GSB_HID>(sw + S::oGW1, myrow + R::oQ, q0);  // q0 W1
      load32(myrow + R::oV2, a);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) a[j] += ((m1 >> j) & 1u) ? q0[j] : T(0);
      store32(myrow + R::oV2, a);
      reinterpret_cast<uint32_t*>(myrow + R::oM)[0] = active ? m1 : 0u;
    }
    if (!active) {
#pragma unroll 1
      for (int i = 0; i < R::oM; ++i) myrow[i] = T(0);
    }
    __syncwarp();
    // ---- outer products over the warp's 32 samples; lane owns column `lane`
    {
      const T w2l = sw[S::oGW2 + lane];
#pragma unroll 1
      for (int r = 0; r < 32; ++r) {
        const T* rw = rows + (size_t)r * R::ROW;
        const uint32_t mr = reinterpret_cast<const uint32_t*>(rw + R::oM)[0];
        const T b0 = rw[R::oB0 + lane];
        const T b1 = ((mr >> lane) & 1u) ? w2l : T(0);     // delta1 = W2 (.) m1
        acc2 += rw[R::oV2 + lane];
        accp += rw[R::oA0 + S::IN_G];                       // db2 = sum p
#pragma unroll
        for (int i = 0; i < R::A0P; i += 4) {
          T a0, a1, a2, a3;
          lds4(rw + R::oA0 + i, a0, a1, a2, a3);
          if (i < R::A0) acc0[i] = fma(a0, b0, acc0[i]);
          if (i + 1 < R::A0) acc0[i + 1] = fma(a1, b0, acc0[i + 1]);
          if (i + 2 < R::A0) acc0[i + 2] = fma(a2, b0, acc0[i + 2]);
          if (i + 3 < R::A0) acc0[i + 3] = fma(a3, b0, acc0[i + 3]);
        }
#pragma unroll
        for (int i = 0; i < R::A1P; i += 4) {
          T a0, a1, a2, a3;
          lds4(rw + R::oA1 + i, a0, a1, a2, a3);
          if (i <= GSB_HID) acc1[i] = fma(a0, b1, acc1[i]);
          if (i + 1 <= GSB_HID) acc1[i + 1] = fma(a1, b1, acc1[i + 1]);
          if (i + 2 <= GSB_HID) acc1[i + 2] = fma(a2, b1, acc1[i + 2]);
          if (i + 3 <= GSB_HID) acc1[i + 3] = fma(a3, b1, acc1[i + 3]);
        }
      }
    }
    __syncwarp();
  }
  // CTA reduction of the per-warp accumulators -> partial slot blockIdx.x
  __syncthreads();
  constexpr int NGP = S::NG;
  T* red = sm;  // [WARPS][NGP]
  {
    T* mine = red + (size_t)wid * NGP;
#pragma unroll
    for (int i = 0; i < S::IN_G; ++i) mine[S::oGW0 + i * GSB_HID + lane] = acc0[i];
    mine[S::oGb0 + lane] = acc0[S::IN_G];
#pragma unroll
    for (int i = 0; i < GSB_HID; ++i) mine[S::oGW1 + i * GSB_HID + lane] = acc1[i];
    mine[S::oGb1 + lane] = acc1[GSB_HID];
    mine[S::oGW2 + lane] = acc2;
    if (lane == 0) mine[S::oGb2] = accp;
  }
  __syncthreads();
  T* out = w.mlp_part + (size_t)blockIdx.x * S::NMLPP;
  for (int t = threadIdx.x; t < NGP; t += WARPS * 32) {
    T a = T(0);
#pragma unroll
    for (int k = 0; k < WARPS; ++k) a += red[(size_t)k * NGP + t];
    out[t] = a;
  }
}

// ---------------------------------------------------------------------------
// backward, colour: sigma(MLP_c([f_c, r])) with seed c_bar

template <typename T, class S>
struct ColRow {
  static constexpr int A0 = S::IN_C + 1;       // [inp, 1]
  static constexpr int A0P = (A0 + 3) / 4 * 4;
  static constexpr int oA0 = 0;
  static constexpr int oB0 = oA0 + A0P;        // a0_bar
  static constexpr int oA1 = oB0 + GSB_HID;    // [h0, 1]
  static constexpr int A1P = (GSB_HID + 1 + 3) / 4 * 4;
  static constexpr int oB1 = oA1 + A1P;        // a1_bar
  static constexpr int oH1 = oB1 + GSB_HID;    // h1
  static constexpr int oY = oH1 + GSB_HID;     // y_bar (3)
  static constexpr int ROW = oY + 4;
};

template <typename T, class S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_bwd_color(Ws<T> w, Geo G, int M, int N,
                                                         const double* __restrict__ dep,
                                                         const T* __restrict__ mlp) {
  using R = ColRow<T, S>;
  constexpr int CW = S::NMLP - S::oCW0;  // colour weights
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* swc = reinterpret_cast<T*>(smem_raw);   // colour block, offsets relative to oCW0
  T* sm = swc + ((CW + 3) / 4 * 4);
  for (int t = threadIdx.x; t < CW; t += blockDim.x) swc[t] = mlp[S::oCW0 + t];
  const T* sw = swc - S::oCW0;              // so that sw[S::oC*] addresses swc
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T* rows = sm + (size_t)wid * 32 * R::ROW;
  T* myrow = rows + (size_t)lane * R::ROW;
  const int64_t NS = (int64_t)M * N;
  T acc0[R::A0], acc1[GSB_HID + 1], acc2[3] = {T(0), T(0), T(0)}, accb2 = T(0);
#pragma unroll
  for (int i = 0; i < R::A0; ++i) acc0[i] = T(0);
#pragma unroll
  for (int i = 0; i <= GSB_HID; ++i) acc1[i] = T(0);
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  for (int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * 32; base < NS; base += nwarps * 32) {
    const int64_t s = base + lane;
    const bool active = s < NS;
    if (active) {
      const int ray = (int)((uint32_t)s / (uint32_t)N);
      T pt[3];
      taped_point<T>(w.o + ray * 3, w.r + ray * 3,
                     dep[(int64_t)ray * w.ld + (int)((uint32_t)s % (uint32_t)N)], G.lo, G.hi, pt);
      const LocT<T> q =
          compact<T>(locate<false>(G.col, (double)pt[0], (double)pt[1], (double)pt[2], nullptr));
      {
        T f[S::CC];
        gather_fast<T, S::CC>(G.col, q, f);
#pragma unroll
        for (int c = 0; c < S::CC; ++c) myrow[R::oA0 + c] = f[c];
#pragma unroll
        for (int a = 0; a < 3; ++a) myrow[R::oA0 + S::CC + a] = w.r[ray * 3 + a];
        myrow[R::oA0 + S::IN_C] = T(1);
#pragma unroll
        for (int i = S::IN_C + 1; i < R::A0P; ++i) myrow[R::oA0 + i] = T(0);
      }
      uint32_t m0, m1;
      T yb[3];
      {
        T h[GSB_HID];
        dense_f_row<T, S::IN_C>(sw + S::oCW0, myrow + R::oA0, h);
        add_bias(sw + S::oCb0, h);
        m0 = relu_mask(h);
        store32(myrow + R::oA1, h);
        myrow[R::oA1 + GSB_HID] = T(1);
#pragma unroll
        for (int i = GSB_HID + 1; i < R::A1P; ++i) myrow[R::oA1 + i] = T(0);
        dense_f_row<T, GSB_HID>(sw + S::oCW1, myrow + R::oA1, h);
        add_bias(sw + S::oCb1, h);
        m1 = relu_mask(h);
        store32(myrow + R::oH1, h);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          T a = T(0);
#pragma unroll
          for (int j = 0; j < GSB_HID; ++j) a = fma(h[j], sw[S::oCW2 + j * 3 + c], a);
          const T cc = sigmoid_fast(a + sw[S::oCb2 + c]);
          yb[c] = w.cbar[s * 3 + c] * (cc * (T(1) - cc));
          myrow[R::oY + c] = yb[c];
        }
        myrow[R::oY + 3] = T(0);
      }
      T a1b[GSB_HID];
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) {
        T a = T(0);
#pragma unroll
        for (int c = 0; c < 3; ++c) a = fma(sw[S::oCW2 + j * 3 + c], yb[c], a);
        a1b[j] = ((m1 >> j) & 1u) ? a : T(0);
      }
      store32(myrow + R::oB1, a1b);
      dense_d_row<T, GSB_HID>(sw + S::oCW1, a1b, m0, myrow + R::oB0);
      load32(myrow + R::oB0, a1b);  // a0_bar
      T fb[S::CC];
      dense_d_reg<T, S::CC>(sw + S::oCW0, a1b, fb);
      // colour grid scatter: theta_c[idx_k] += w_k f_bar
      T wk[8];
      corner_w(q, wk);
      if (w.det_keys) {
        det_put<T, S::CC>(w.det_keys, w.det_vals, s * (S::NL + 1) + S::NL, G.col, (int64_t)q.base, fb, wk,
                          true);
      } else {
        T* Gp = reinterpret_cast<T*>(G.col.grad) + (int64_t)q.base * S::CC;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          T vv[S::CC];
#pragma unroll
          for (int c = 0; c < S::CC; ++c) vv[c] = wk[k] * fb[c];
          red_row<T, S::CC>(Gp + corner_off(G.col, k) * S::CC, vv);
        }
      }
    } else {
#pragma unroll 1
      for (int i = 0; i < R::ROW; ++i) myrow[i] = T(0);
    }
    __syncwarp();
    warp_outer<T, R::A0, R::A0P, GSB_HID + 1, R::A1P>(rows, R::ROW, R::oA0, R::oB0, R::oA1, R::oB1,
                                                      lane, acc0, acc1);
#pragma unroll 1
    for (int r = 0; r < 32; ++r) {
      const T* rw = rows + (size_t)r * R::ROW;
      const T hj = rw[R::oH1 + lane];
      T y0, y1, y2, y3;
      lds4(rw + R::oY, y0, y1, y2, y3);
      acc2[0] = fma(hj, y0, acc2[0]);
      acc2[1] = fma(hj, y1, acc2[1]);
      acc2[2] = fma(hj, y2, acc2[2]);
      accb2 += lane == 0 ? y0 : (lane == 1 ? y1 : (lane == 2 ? y2 : T(0)));
    }
    __syncwarp();
  }
  __syncthreads();
  constexpr int NCP = S::NMLP - S::NG;
  T* red = sm;
  {
    T* mine = red + (size_t)wid * NCP;
    const int o = S::NG;
    if (lane < S::oCW0 - S::NG) mine[lane] = T(0);  // alignment padding
#pragma unroll
    for (int i = 0; i < S::IN_C; ++i) mine[S::oCW0 - o + i * GSB_HID + lane] = acc0[i];
    mine[S::oCb0 - o + lane] = acc0[S::IN_C];
#pragma unroll
    for (int i = 0; i < GSB_HID; ++i) mine[S::oCW1 - o + i * GSB_HID + lane] = acc1[i];
    mine[S::oCb1 - o + lane] = acc1[GSB_HID];
#pragma unroll
    for (int c = 0; c < 3; ++c) mine[S::oCW2 - o + lane * 3 + c] = acc2[c];
    if (lane < 3) mine[S::oCb2 - o + lane] = accb2;
  }
  __syncthreads();
  T* out = w.mlp_part + (size_t)blockIdx.x * S::NMLPP + S::NG;
  for (int t = threadIdx.x; t < NCP; t += WARPS * 32) {
    T a = T(0);
#pragma unroll
    for (int k = 0; k < WARPS; ++k) a += red[(size_t)k * NCP + t];
    out[t] = a;
  }
}

// ---------------------------------------------------------------------------
// deterministic finalization

// sum of the per-CTA partial weight gradients, fixed order (deterministic):
// block = 32 parameters x 8 warps; warp w sums slots w, w+8, ...; then the 8
// warp partials are added in warp order
template <typename T, class S>
__device__ __forceinline__ void finalize_mlp_block(const Ws<T>& w, T* grads, int64_t mlp_off, int nb_geo,
                                                   int nb_col, int bx) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int t = bx * 32 + lane;
  double a = 0.0;
  if (t < S::NMLP) {
    const int nb = t < S::NG ? nb_geo : nb_col;
    for (int b = wid; b < nb; b += 8) a += (double)w.mlp_part[(size_t)b * S::NMLPP + t];
  }
  red[wid][lane] = a;
  __syncthreads();
  if (wid == 0 && t < S::NMLP) {
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) tot += red[k][lane];
    grads[mlp_off + t] += (T)tot;
  }
}

// Deterministic reduction of the per-CTA MLP partials, split over (column
// group of 32 parameters) x (FIN_SPLIT chunks of the partial range): 4 loads
// in flight per warp, then the last chunk-block of a column group (atomic
// ticket) sums the chunk totals in chunk order.
constexpr int FIN_SPLIT = 16;

template <typename T, class S>
__device__ __forceinline__ void finalize_mlp2_block(const Ws<T>& w, T* grads, int64_t mlp_off, int nb_geo,
                                                    int nb_col, int bx, int y) {
  __shared__ double red[8][33];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int t = bx * 32 + lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (t < S::NMLP) {
    const int nb = t < S::NG ? nb_geo : nb_col;
    const int b0 = (int)((int64_t)nb * y / FIN_SPLIT), b1 = (int)((int64_t)nb * (y + 1) / FIN_SPLIT);
    const T* col = w.mlp_part + t;
    int b = b0 + wid;
    for (; b + 24 < b1; b += 32) {
      a0 += (double)col[(size_t)b * S::NMLPP];
      a1 += (double)col[(size_t)(b + 8) * S::NMLPP];
      a2 += (double)col[(size_t)(b + 16) * S::NMLPP];
      a3 += (double)col[(size_t)(b + 24) * S::NMLPP];
    }
    for (; b < b1; b += 8) a0 += (double)col[(size_t)b * S::NMLPP];
  }
  red[wid][lane] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (wid == 0) {
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) tot += red[k][lane];
    if (t < S::NMLP) w.fin_red[(size_t)y * S::NMLPP + t] = tot;
    __threadfence();
    __syncwarp();
    if (lane == 0) last = atomicAdd(&w.fin_cnt[bx], 1u) == FIN_SPLIT - 1;
  }
  __syncthreads();
  if (last && wid == 0) {
    __threadfence();
    if (t < S::NMLP) {
      double tot = 0.0;
      for (int k = 0; k < FIN_SPLIT; ++k) tot += __ldcg(&w.fin_red[(size_t)k * S::NMLPP + t]);
      grads[mlp_off + t] += (T)tot;
    }
    if (lane == 0) w.fin_cnt[bx] = 0u;  // ready for the next launch
  }
}
template <typename T, class S>
__global__ void __launch_bounds__(256) k_finalize_mlp2(Ws<T> w, T* grads, int64_t mlp_off,
                                                       int nb_geo, int nb_col) {
  finalize_mlp2_block<T, S>(w, grads, mlp_off, nb_geo, nb_col, blockIdx.x, blockIdx.y);
}

// Loss parts and the log_s gradient from the per-ray / per-smoothness-pair
// partials: one thread per item over many blocks, block partials in a
// scratch array, and the last block (atomic ticket) sums them in block order.
template <typename T>
__device__ __forceinline__ void finalize_loss_block(const Ws<T>& w, int M, int S, T* grads, const T* params,
                                                    int64_t log_s_off, const LossW& L, int blk, int nblk) {
  __shared__ double red[7][8];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int i = blk * 256 + tid;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  if (i < M) {
    const double* p = w.ray_part + (int64_t)i * 8;
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] = p[k];
  }
  if (i < S) acc[6] = w.smooth_part[i];
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const double v = warp_sum(acc[k]);
    if (lane == 0) red[k][wid] = v;
  }
  __syncthreads();
  if (tid < 7) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[tid][q];
    w.loss_red[blk * 8 + tid] = t;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(w.loss_cnt, 1u) == (unsigned)nblk - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // block partials summed by warp k (part k): lane-strided, then a fixed
  // butterfly -- deterministic, and 32-way parallel instead of one thread
  // walking every block
  if (wid < 7) {
    double a = 0.0;
    for (int b = lane; b < nblk; b += 32) a += __ldcg(&w.loss_red[b * 8 + wid]);
    a = warp_sum(a);
    if (lane == 0) red[wid][0] = a;
  }
  __syncthreads();
  if (tid != 0) return;
  double tot[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) tot[k] = red[k][0];
  *w.loss_cnt = 0u;  // ready for the next launch
  const T sT = exp(params[log_s_off]);
  const double s = (double)sT;
  long long nv = w.counts[GSB_C_VALID], ne = w.counts[GSB_C_EIK];
  double rgb = tot[0] / L.m_global;
  double dep = tot[1] / (double)(nv > 1 ? nv : 1);
  double sdf = tot[2] / L.m_global;
  double fs = tot[3] / L.m_global;
  double eik = tot[4] / (double)(ne > 1 ? ne : 1);
  double sm = L.smooth > 0.0 && S > 0 ? tot[6] / L.smooth_global : 0.0;
  w.parts[GSB_P_RGB] = rgb;
  w.parts[GSB_P_DEPTH] = dep;
  w.parts[GSB_P_SDF] = sdf;
  w.parts[GSB_P_FS] = fs;
  w.parts[GSB_P_EIK] = eik;
  w.parts[GSB_P_SMOOTH] = sm;
  w.parts[GSB_P_S] = s;
  w.parts[GSB_P_TOTAL] = L.rgb * rgb + L.depth * dep + L.sdf * sdf + L.fs * fs + L.eik * eik +
                         L.smooth * sm;
  // d total / d log_s = s * sum z_bar phi (exp vjp)
  grads[log_s_off] += (T)(tot[5] * s);
}
// the MLP reduction (blocks [0, ncol) one pass, or [0, ncol x FIN_SPLIT)
// split) and the loss reduction (the blocks after them) in one launch
template <typename T, class S, bool SPLIT>
__global__ void __launch_bounds__(256) k_finalize(Ws<T> w, T* grads, int64_t mlp_off, int nb_geo, int nb_col,
                                                  int M, int nsm, const T* params, int64_t log_s_off, LossW L,
                                                  int nloss) {
  constexpr int ncol = (S::NMLP + 31) / 32, nmlp = SPLIT ? ncol * FIN_SPLIT : ncol;
  const int b = blockIdx.x;
  if (b >= nmlp)
    finalize_loss_block<T>(w, M, nsm, grads, params, log_s_off, L, b - nmlp, nloss);
  else if constexpr (SPLIT)
    finalize_mlp2_block<T, S>(w, grads, mlp_off, nb_geo, nb_col, b % ncol, b / ncol);
  else
    finalize_mlp_block<T, S>(w, grads, mlp_off, nb_geo, nb_col, b);
}

// ---------------------------------------------------------------------------
// Adam over the arena (gs/optimizer.py:38-55): float64 math, storage dtype,
// non-finite gradients zeroed and counted, gradient cleared.

// learning-rate runs over the arena; lr < 0 marks a run this launch does not
// own (data-parallel ZeRO-1: another rank's shard): its gradients are only
// zeroed, p / m / v are neither read nor written
constexpr int GSB_ADAM_MAX_SEGS = 32;
struct AdamSegs {
  int64_t begin[GSB_ADAM_MAX_SEGS];
  double lr[GSB_ADAM_MAX_SEGS];
  int n;
};

struct AdamConst {
  double b1, b2, eps, c1, c2, ib1, ib2, inv_c1, inv_c2;  // ib = 1 - beta
};

// Exact form (float64 storage): every operation as numba performs it.
template <typename T>
__device__ __forceinline__ void adam_exact(T& p, T& g, T& m, T& v, double lr, const AdamConst& k,
                                           int& bad) {
  double gi = (double)g;
  if (!isfinite(gi)) {
    gi = 0.0;
    ++bad;
  }
  const double mi = k.b1 * (double)m + k.ib1 * gi;
  const double vi = k.b2 * (double)v + k.ib2 * gi * gi;
  m = (T)mi;
  v = (T)vi;
  p = (T)((double)p - lr * (mi / k.c1) / (sqrt(vi / k.c2) + k.eps));
  g = T(0);
}

// Fast form (float32 storage): m, v exactly as numba (float64 mul/add, no
// FMA); the update uses reciprocal multiplies and Newton-refined rsqrt/rcp
// in float64 (relative error ~1e-15), so the float32 rounding of p - update
// equals the reference's except when the exact value sits within ~1e-15 of
// a float32 rounding boundary.
__device__ __forceinline__ void adam_fast(float& p, float& g, float& m, float& v, double lr,
                                          const AdamConst& k, int& bad) {
  double gi = (double)g;
  if (!isfinite(gi)) {
    gi = 0.0;
    ++bad;
  }
  const double mi = k.b1 * (double)m + k.ib1 * gi;
  const double vi = k.b2 * (double)v + k.ib2 * gi * gi;
  m = (float)mi;
  v = (float)vi;
  const double q1 = mi * k.inv_c1, q2 = vi * k.inv_c2;
  double sq;
  if (q2 == 0.0) {  // never-touched parameter: sqrt(0) = 0 exactly
    sq = 0.0;
  } else if (q2 > 1e-30 && q2 < 1e30) {  // rsqrtf seed in float range
    double t = (double)rsqrtf((float)q2);
    t = t * fma(-0.5 * q2, t * t, 1.5);
    t = t * fma(-0.5 * q2, t * t, 1.5);
    sq = q2 * t;
    sq = fma(fma(-sq, sq, q2), 0.5 * t, sq);  // one Newton step on sqrt itself
  } else {
    sq = sqrt(q2);
  }
  const double den = sq + k.eps;
  double y = (double)__frcp_rn((float)den);
  y = fma(fma(-den, y, 1.0), y, y);
  y = fma(fma(-den, y, 1.0), y, y);
  const double num = lr * q1;
  double q = num * y;
  q = fma(fma(-q, den, num), y, q);
  p = (float)((double)p - q);
  g = 0.0f;
}

// kAdamU: vectors in flight per thread per trip
template <typename T, int kAdamU = 2>
__global__ void __launch_bounds__(256) k_adam(T* __restrict__ P, T* __restrict__ Gr, T* __restrict__ Mm,
                                              T* __restrict__ Vv, int64_t n, AdamSegs segs,
                                              AdamConst k, const double* guard, double thr,
                                              const int32_t* guard_status, int32_t* status) {
  // halt (this and every later update) where the reference raises before
  // its Adam step: a diverged total (gs/optimizer.py:368-371) or a step
  // error flag (GridBoundsError etc., raised inside train_objective)
  bool halt = guard && status[GSB_ST_DIVERGED];
  if (guard) {
    const double tot = guard[0];
    halt |= !(tot == tot) || isinf(tot) || tot > thr;
  }
  if (guard_status)
    halt |= guard_status[GSB_ST_BOUNDS] | guard_status[GSB_ST_OVERFLOW] |
            guard_status[GSB_ST_VIEWDIR];
  if (halt) {
    if (blockIdx.x == 0 && threadIdx.x == 0) status[GSB_ST_DIVERGED] = 1;
    return;
  }
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
  using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  int bad = 0;
  const int64_t nvec = n / V;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < nvec; i0 += kAdamU * stride) {
    // kAdamU independent vectors per iteration: more bytes in flight
    Vec p[kAdamU], g[kAdamU], m[kAdamU], v[kAdamU];
    double lr[kAdamU];
#pragma unroll
    for (int u = 0; u < kAdamU; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nvec) break;
      const int64_t e = i * V;
      int sidx = 0;
      for (int q = 1; q < segs.n; ++q)
        if (e >= segs.begin[q]) sidx = q;
      lr[u] = segs.lr[sidx];
      if (lr[u] < 0.0) continue;  // not owned: gradients zeroed below
      p[u] = __ldcs(reinterpret_cast<const Vec*>(P) + i);
      g[u] = __ldcs(reinterpret_cast<const Vec*>(Gr) + i);
      m[u] = __ldcs(reinterpret_cast<const Vec*>(Mm) + i);
      v[u] = __ldcs(reinterpret_cast<const Vec*>(Vv) + i);
    }
#pragma unroll
    for (int u = 0; u < kAdamU; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nvec) break;
      if (lr[u] < 0.0) {
        __stcs(reinterpret_cast<Vec*>(Gr) + i, Vec{});
        continue;
      }
      // a gradient vector that is already +0 (no sample touched these
      // parameters this step: ~3/4 of the rows at config 2) needs no zeroing
      // store; if m and v are +0 too (never touched), the update rewrites the
      // same bits everywhere and nothing is written back
      const uint4 gb = *reinterpret_cast<const uint4*>(&g[u]);
      const bool g_zero = (gb.x | gb.y | gb.z | gb.w) == 0u;
      {
        const uint4 mb = *reinterpret_cast<const uint4*>(&m[u]);
        const uint4 vb = *reinterpret_cast<const uint4*>(&v[u]);
        if (g_zero && ((mb.x | mb.y | mb.z | mb.w) | (vb.x | vb.y | vb.z | vb.w)) == 0u) continue;
      }
      T* pp = reinterpret_cast<T*>(&p[u]);
      T* gg = reinterpret_cast<T*>(&g[u]);
      T* mm = reinterpret_cast<T*>(&m[u]);
      T* vv = reinterpret_cast<T*>(&v[u]);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        if constexpr (sizeof(T) == 4)
          adam_fast(pp[q], gg[q], mm[q], vv[q], lr[u], k, bad);
        else
          adam_exact(pp[q], gg[q], mm[q], vv[q], lr[u], k, bad);
      }
      __stcs(reinterpret_cast<Vec*>(P) + i, p[u]);
      if (!g_zero) __stcs(reinterpret_cast<Vec*>(Gr) + i, g[u]);
      __stcs(reinterpret_cast<Vec*>(Mm) + i, m[u]);
      __stcs(reinterpret_cast<Vec*>(Vv) + i, v[u]);
    }
  }
  // tail
  for (int64_t e = nvec * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride) {
    int sidx = 0;
    for (int q = 1; q < segs.n; ++q)
      if (e >= segs.begin[q]) sidx = q;
    if (segs.lr[sidx] < 0.0)
      Gr[e] = T(0);
    else if constexpr (sizeof(T) == 4)
      adam_fast(P[e], Gr[e], Mm[e], Vv[e], segs.lr[sidx], k, bad);
    else
      adam_exact(P[e], Gr[e], Mm[e], Vv[e], segs.lr[sidx], k, bad);
  }
  bad = warp_sum(bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(status + GSB_ST_ADAM_BAD, bad);
}

// float32 storage with 256-bit (8-float) streaming accesses (sm_100's
// LDG/STG.256): half the memory instructions per byte of k_adam<float>.
// The learning-rate segment is looked up per 4-float half (segments are
// 16-byte aligned); a vector whose halves are both no-ops is not written.
// One vector per thread per trip, <= 64 registers (4 blocks of 256 per SM):
// 295 us per step at config 2 against 350 for k_adam<float>; two vectors per
// trip (106 registers, 2 blocks) measured 406, a 5-block cap (spills) 339.
__device__ __forceinline__ void ld8cs(const float* p, float (&r)[8]) {
  asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void st8cs(float* p, const float (&r)[8]) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]),
               "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
               : "memory");
}
__device__ __forceinline__ double adam_seg_lr(const AdamSegs& segs, int64_t e) {
  int sidx = 0;
  for (int q = 1; q < segs.n; ++q)
    if (e >= segs.begin[q]) sidx = q;
  return segs.lr[sidx];
}

template <int kU = 1>
__global__ void __launch_bounds__(256, 4) k_adam8(float* __restrict__ P, float* __restrict__ Gr,
                                               float* __restrict__ Mm, float* __restrict__ Vv, int64_t n,
                                               AdamSegs segs, AdamConst k, const double* guard, double thr,
                                               const int32_t* guard_status, int32_t* status) {
  bool halt = guard && status[GSB_ST_DIVERGED];
  if (guard) {
    const double tot = guard[0];
    halt |= !(tot == tot) || isinf(tot) || tot > thr;
  }
  if (guard_status)
    halt |= guard_status[GSB_ST_BOUNDS] | guard_status[GSB_ST_OVERFLOW] |
            guard_status[GSB_ST_VIEWDIR];
  if (halt) {
    if (blockIdx.x == 0 && threadIdx.x == 0) status[GSB_ST_DIVERGED] = 1;
    return;
  }
  int bad = 0;
  const int64_t nvec = n / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < nvec; i0 += kU * stride) {
    float p[kU][8], g[kU][8], m[kU][8], v[kU][8];
    double lr[kU][2];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nvec) break;
      lr[u][0] = adam_seg_lr(segs, i * 8);
      lr[u][1] = adam_seg_lr(segs, i * 8 + 4);
      ld8cs(Gr + i * 8, g[u]);
      if (lr[u][0] < 0.0 && lr[u][1] < 0.0) continue;  // not owned: gradients zeroed below
      ld8cs(P + i * 8, p[u]);
      ld8cs(Mm + i * 8, m[u]);
      ld8cs(Vv + i * 8, v[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nvec) break;
      uint32_t gor = 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q) gor |= __float_as_uint(g[u][q]);
      if (lr[u][0] < 0.0 && lr[u][1] < 0.0) {
        if (gor) {
          const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          st8cs(Gr + i * 8, z);
        }
        continue;
      }
      // g, m and v all +0: the update rewrites the same bits, nothing is written
      uint32_t mvor = 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q) mvor |= __float_as_uint(m[u][q]) | __float_as_uint(v[u][q]);
      if ((gor | mvor) == 0u) continue;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double l = lr[u][q >> 2];
        if (l < 0.0)
          g[u][q] = 0.f;  // a foreign half: parameters and moments written back unchanged
        else
          adam_fast(p[u][q], g[u][q], m[u][q], v[u][q], l, k, bad);
      }
      st8cs(P + i * 8, p[u]);
      if (gor) st8cs(Gr + i * 8, g[u]);
      st8cs(Mm + i * 8, m[u]);
      st8cs(Vv + i * 8, v[u]);
    }
  }
  for (int64_t e = nvec * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride) {
    const double l = adam_seg_lr(segs, e);
    if (l < 0.0)
      Gr[e] = 0.f;
    else
      adam_fast(P[e], Gr[e], Mm[e], Vv[e], l, k, bad);
  }
  bad = warp_sum(bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(status + GSB_ST_ADAM_BAD, bad);
}

// ---------------------------------------------------------------------------
// deterministic scatter mode: sum each grad row's entries in (sample, level,
// corner) order -- the entries were stably sorted by row address

static __global__ void k_det_iota(int32_t* idx, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) idx[i] = (int32_t)i;
}

template <typename T>
__global__ void k_det_reduce(const uint64_t* __restrict__ keys, const int32_t* __restrict__ order,
                             const T* __restrict__ vals, int64_t n, int C_geo, int C_col,
                             uintptr_t col_lo, uintptr_t col_hi) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t key = keys[i];
  if (key == ~0ull || (i > 0 && keys[i - 1] == key)) return;  // run heads only
  const int C = (key >= col_lo && key < col_hi) ? C_col : C_geo;
  T acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = T(0);
  for (int64_t j = i; j < n && keys[j] == key; ++j) {
    const T* v = vals + (int64_t)order[j] * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] += v[c];
  }
  T* row = reinterpret_cast<T*>((uintptr_t)key);
  for (int c = 0; c < C; ++c) row[c] += acc[c];
}

}  // namespace gsb
