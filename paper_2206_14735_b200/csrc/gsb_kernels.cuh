// gsb_kernels.cuh -- the GO-Surf training-step kernels (templated on the
// storage/compute type T and the grid shape S).
//
// Step data flow (all on one stream, no host round trips):
//   k_ray_setup      rays + stratified depths      gs/sampler.py:58-107, gs/renderer.py:302-321
//   k_sdf_eval       no-grad phi at listed samples gs/renderer.py:323-326, 236-240
//   k_importance     one importance round per ray  gs/renderer.py:329-342, gs/sampler.py:128-197
//   k_counts         tr/fs/eik partition counts    gs/renderer.py:384-412
//   k_fwd            phi, grad phi, colour          gs/renderer.py:348-365
//   k_smooth         smoothness loss + adjoints     gs/renderer.py:416-434
//   k_render         alphas/composite/losses/adjoints (warp-free, thread per ray)
//                                                  gs/renderer.py:112-159, 372-414
//   k_bwd_geom       grid scatter + geometry MLP grads
//   k_bwd_color      colour grid scatter + colour MLP grads
//   k_finalize_*     deterministic reductions of the per-CTA partials
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
  T* pbar;
  T* ubar;
  T* cbar;
  T* wts;
  double* ray_part;     // [M][8]
  double* smooth_part;  // [S]
  T* mlp_part;          // [nb_max][NMLP]
  int nb_max;
  long long* counts;
  double* parts;
  int32_t* status;
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

template <typename T>
__global__ void k_ray_setup(gsb_dataset_t D, const int64_t* __restrict__ ids, int M, int ray_base,
                            Ws<T> w, Geo G, int Nc, double nearv, double max_depth, int has_ff,
                            double ff, gsb_pcg64_t rng) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
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
  // stratified_coarse (gs/sampler.py:91-107) with uniform row (ray_base+i)
  Pcg g;
  g.init(rng);
  g.advance((uint64_t)(ray_base + i) * (uint64_t)Nc);
  double span = farv - nearv;
  double* dep = w.dep[0] + (int64_t)i * w.ld;
  for (int j = 0; j < Nc; ++j) {
    double u = g.next_double();
    dep[j] = nearv + span * (((double)j + u) / (double)Nc);
  }
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

static __device__ void importance_row(int K, int A, const double* d, const double* ph,
                                      const double* win, double s, double nearv, double farv,
                                      Pcg* g, const double* uni, double* out, int32_t* src,
                                      double* wout) {
  double cdf[GSB_KMAX];
  double c = 0.0;
  if (win) {  // weights given (importance_refine_with_sources signature)
    for (int i = 0; i < K - 1; ++i) {
      c = (i == 0) ? win[i] : c + win[i];
      cdf[i] = c;
    }
  } else {
    // render_weights_data (gs/renderer.py:162-173), sequential cumprod
    double sig_i = sigmoid_raw(s * ph[0]);
    double trans = 1.0;
    for (int i = 0; i < K - 1; ++i) {
      double sig_n = sigmoid_raw(s * ph[i + 1]);
      double den = sig_i >= 1e-12 ? sig_i : 1e-12;
      double ratio = sig_n / den;
      double om = ratio <= 1.0 ? ratio : 1.0;
      double wi = trans * (1.0 - om);
      if (wout) wout[i] = wi;
      c = (i == 0) ? wi : c + wi;
      cdf[i] = c;
      trans = trans * om;
      sig_i = sig_n;
    }
    if (wout) wout[K - 1] = trans * (1.0 - 1.0);
  }
  // importance_refine_with_sources (gs/sampler.py:128-169)
  bool dead = c <= 0.0;
  if (dead)
    for (int i = 0; i < K - 1; ++i) cdf[i] = (double)(i + 1);
  double last = cdf[K - 2];
  for (int i = 0; i < K - 1; ++i) cdf[i] = cdf[i] / last;
  double nw[GSB_AMAX];
  int ord[GSB_AMAX];
  for (int a = 0; a < A; ++a) {
    double u = uni ? uni[a] : g->next_double();
    // idx = #(cdf <= u), cdf non-decreasing -> upper bound
    int lo = 0, hi = K - 1;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
    }
    int idx = lo < K - 2 ? lo : K - 2;
    double clo = idx > 0 ? cdf[idx - 1] : 0.0, chi = cdf[idx];
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
    nw[a] = v;
    // stable insertion of a into ord by value
    int t = a;
    while (t > 0 && nw[ord[t - 1]] > v) {
      ord[t] = ord[t - 1];
      --t;
    }
    ord[t] = a;
  }
  // stable merge (np.argsort kind="stable": old columns precede new on ties)
  bool sorted = true;
  for (int i = 0; i + 1 < K; ++i)
    if (!(d[i] <= d[i + 1])) sorted = false;
  int n = K + A;
  if (sorted) {
    int i = 0, a = 0, o = 0;
    while (i < K || a < A) {
      if (a >= A || (i < K && !(nw[ord[a]] < d[i]))) {
        out[o] = d[i];
        src[o++] = i++;
      } else {
        out[o] = nw[ord[a]];
        src[o++] = -1;
        ++a;
      }
    }
  } else {  // general stable insertion sort over the concatenation
    for (int t = 0; t < n; ++t) {
      double v = t < K ? d[t] : nw[t - K];
      int sv = t < K ? t : -1;
      int q = t;
      while (q > 0 && out[q - 1] > v) {
        out[q] = out[q - 1];
        src[q] = src[q - 1];
        --q;
      }
      out[q] = v;
      src[q] = sv;
    }
  }
  bool bad = false;
  for (int i = 0; i + 1 < n; ++i)
    if (out[i + 1] - out[i] < 1e-9) bad = true;
  if (bad) separation_fallback(out, src, n);
}

template <typename T>
__global__ void k_importance_dev(Ws<T> w, int M, int K, int A, int ray_base,
                                 const double* __restrict__ dep, const double* __restrict__ phi,
                                 double* __restrict__ dep_out, double* __restrict__ phi_out,
                                 const T* __restrict__ log_s, gsb_pcg64_t rng,
                             int32_t* __restrict__ evl, int32_t* __restrict__ evl_count,
                             int64_t cap, int want_list) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  // ModelState.s_value() = float(np.exp(log_s)) in the model dtype
  const double s = (double)exp(log_s[0]);
  Pcg g;
  g.init(rng);
  g.advance((uint64_t)(ray_base + i) * (uint64_t)A);
  const double* d = dep + (int64_t)i * w.ld;
  const double* ph = phi + (int64_t)i * w.ld;
  double* out = dep_out + (int64_t)i * w.ld;
  int32_t src[GSB_KMAX];
  importance_row(K, A, d, ph, nullptr, s, w.nearv[i], w.farv[i], &g, nullptr, out, src, nullptr);
  double* po = phi_out + (int64_t)i * w.ld;
  int nnew = 0;
  for (int t = 0; t < K + A; ++t) {
    if (src[t] >= 0) po[t] = ph[src[t]];
    else ++nnew;
  }
  if (!want_list) return;
  int base = atomicAdd(evl_count, nnew);
  if (base + nnew > cap) {
    atomicOr(w.status + GSB_ST_OVERFLOW, 1);
    return;
  }
  for (int t = 0; t < K + A; ++t)
    if (src[t] < 0) evl[base++] = i * GSB_KMAX + t;
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
__global__ void k_smooth(Ws<T> w, int64_t MN, int S, T scale) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
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

template <typename T>
__global__ void __launch_bounds__(64) k_render(Ws<T> w, int M, int N, const double* __restrict__ dep,
                                               const T* __restrict__ params, int64_t log_s_off,
                                               LossW L) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const T s = exp(params[log_s_off]);  // ModelState.s_tensor (gs/renderer.py:83-84)
  const T SF = (T)1e-12, TF = (T)1e-15;
  T sig[GSB_KMAX], trn[GSB_KMAX];
  const int64_t s0 = (int64_t)i * N;
  const double* d = dep + (int64_t)i * w.ld;
  // ---- forward: alphas (:112-134) + composite (:137-159)
  for (int j = 0; j < N; ++j) sig[j] = sigmoid_raw(w.sphi[s0 + j] * s);
  T logt = T(0), ch[3] = {T(0), T(0), T(0)}, dh = T(0);
  for (int j = 0; j < N; ++j) {
    T al = T(0);
    if (j < N - 1) {
      T den = sig[j] >= SF ? sig[j] : SF;
      T ratio = sig[j + 1] / den;
      al = T(1) - (ratio <= T(1) ? ratio : T(1));
    }
    T om = T(1) - al;
    T Tj = j == 0 ? T(1) : exp(logt);
    trn[j] = Tj;
    logt += log(om >= TF ? om : TF);
    T wj = Tj * al;
    w.wts[s0 + j] = wj;
#pragma unroll
    for (int c = 0; c < 3; ++c) ch[c] += wj * w.scol[(s0 + j) * 3 + c];
    dh += wj * (T)d[j];
  }
  // ---- losses (:372-414)
  const int valid = w.valid[i];
  const double D = w.dray[i];
  T err[3], q = T(0);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    err[c] = ch[c] - w.col[i * 3 + c];
    q += err[c] * err[c];
  }
  T lrgb = sqrt(q + (T)1e-24);
  T dT = (T)D;
  T lde = valid ? fabs(dh - dT) : T(0);
  const long long nvalid = w.counts[GSB_C_VALID];
  const long long neik = w.counts[GSB_C_EIK];
  const T inv_nv = T(1) / (T)(nvalid > 1 ? nvalid : 1);
  const T inv_ne = T(1) / (T)(neik > 1 ? neik : 1);
  const T ntr = (T)max(w.cnt[i * 3 + 0], 1), nfs = (T)max(w.cnt[i * 3 + 1], 1);
  const T tr_t = (T)L.trunc;
  T sdf = T(0), fsv = T(0), eik = T(0);
  for (int j = 0; j < N; ++j) {
    double b = D - d[j];
    T bc = (T)b, ph = w.sphi[s0 + j];
    bool tr = valid && fabs(b) <= L.trunc;
    bool fs = valid && b > L.trunc;
    bool bh = valid && b < -L.trunc;
    if (tr) sdf += fabs(ph - bc);
    if (fs) {
      T e = exp(ph * (T)(-L.alpha));
      T inner = e - T(1);
      inner = T(0) >= inner ? T(0) : inner;
      T lin = ph - bc;
      fsv += inner >= lin ? inner : lin;
    }
    if (fs || bh || !valid) {
      const T* gp = w.sgphi + (s0 + j) * 3;
      T nn = sqrt((gp[0] * gp[0] + gp[1] * gp[1]) + gp[2] * gp[2] + (T)1e-20);
      T df = T(1) - nn;
      eik += df * df;
    }
  }
  (void)tr_t;
  double* part = w.ray_part + (int64_t)i * 8;
  part[0] = (double)lrgb;
  part[1] = (double)lde;
  part[2] = (double)(sdf / ntr);
  part[3] = (double)(fsv / nfs);
  part[4] = (double)eik;
  // ---- backward seeds
  const T Mg = (T)L.m_global;
  T chb[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) chb[c] = ((T)L.rgb / Mg) * err[c] / lrgb;
  const T dhb = valid ? (T)L.depth * sgn(dh - dT) * inv_nv : T(0);
  const T ksdf = ((T)L.sdf / Mg) / ntr, kfs = ((T)L.fs / Mg) / nfs;
  const T keik = (T)(-2.0 * L.eik) * inv_ne;
  T acc = T(0);      // L_bar suffix sum
  T carry = T(0);    // D-bar part of sigma_bar for sample j+1
  T logs = T(0);
  for (int j = N - 1; j >= 0; --j) {
    const int64_t sj = s0 + j;
    T al = T(0), ratio = T(0), den = T(1);
    if (j < N - 1) {
      den = sig[j] >= SF ? sig[j] : SF;
      ratio = sig[j + 1] / den;
      al = T(1) - (ratio <= T(1) ? ratio : T(1));
    }
    T om = T(1) - al;
    T Tj = trn[j];
    T wj = Tj * al;
    const T* cj = w.scol + sj * 3;
    T wbar = (chb[0] * cj[0] + chb[1] * cj[1]) + chb[2] * cj[2] + dhb * (T)d[j];
#pragma unroll
    for (int c = 0; c < 3; ++c) w.cbar[sj * 3 + c] = wj * chb[c];
    T Tbar = wbar * al;
    T Lbar = acc;
    acc += Tbar * Tj;
    T ombar = om >= TF ? Lbar / om : T(0);
    T abar = wbar * Tj - ombar;
    T sig_own = T(0);  // D-bar contribution to sigma_bar_j
    if (j < N - 1) {
      T rbar = ratio <= T(1) ? -abar : T(0);
      T sbn = carry + rbar / den;  // sigma_bar_{j+1}, now complete
      T sg = sig[j + 1];
      T zb = sbn * (sg * (T(1) - sg));
      // finalize sample j+1
      {
        const int64_t sn = sj + 1;
        T ph = w.sphi[sn];
        logs += zb * ph;
        double b = D - d[j + 1];
        T pb = zb * s;
        if (valid && fabs(b) <= L.trunc) pb += ksdf * sgn(ph - (T)b);
        if (valid && b > L.trunc) {
          T e = exp(ph * (T)(-L.alpha));
          T inner = e - T(1);
          T inner0 = T(0) >= inner ? T(0) : inner;
          T dfs = inner0 >= ph - (T)b ? (inner > T(0) ? e * (T)(-L.alpha) : T(0)) : T(1);
          pb += kfs * dfs;
        }
        w.pbar[sn] = pb;
      }
      sig_own = sig[j] >= SF ? -(rbar * sg) / (den * den) : T(0);
    }
    carry = sig_own;
    // eikonal adjoint for sample j
    {
      double b = D - d[j];
      bool fs = valid && b > L.trunc, bh = valid && b < -L.trunc;
      const T* gp = w.sgphi + sj * 3;
      if (fs || bh || !valid) {
        T nn = sqrt((gp[0] * gp[0] + gp[1] * gp[1]) + gp[2] * gp[2] + (T)1e-20);
        T k = keik * (T(1) - nn) / nn;
#pragma unroll
        for (int c = 0; c < 3; ++c) w.ubar[sj * 3 + c] = k * gp[c];
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) w.ubar[sj * 3 + c] = T(0);
      }
    }
  }
  {  // finalize sample 0
    T sg = sig[0];
    T zb = carry * (sg * (T(1) - sg));
    T ph = w.sphi[s0];
    logs += zb * ph;
    double b = D - d[0];
    T pb = zb * s;
    if (valid && fabs(b) <= L.trunc) pb += ksdf * sgn(ph - (T)b);
    if (valid && b > L.trunc) {
      T e = exp(ph * (T)(-L.alpha));
      T inner = e - T(1);
      T inner0 = T(0) >= inner ? T(0) : inner;
      T dfs = inner0 >= ph - (T)b ? (inner > T(0) ? e * (T)(-L.alpha) : T(0)) : T(1);
      pb += kfs * dfs;
    }
    w.pbar[s0] = pb;
  }
  part[5] = (double)logs;
}

// ---------------------------------------------------------------------------
// backward, geometry: grid scatter + geometry MLP weight gradients.
// Thread per sample.  Each thread's shared-memory row holds its activations
// and, at the end, its outer-product factors; every warp then accumulates
// the 32 samples' outer products with lane j owning output column j.

template <typename T, class S>
struct GeoRow {
  static constexpr int A0 = S::IN_G + 1;            // [p z + v, p]   (z staged here)
  static constexpr int A0P = (A0 + 3) / 4 * 4;
  static constexpr int oA0 = 0;
  static constexpr int oB0 = oA0 + A0P;             // delta0
  static constexpr int oA1 = oB0 + GSB_HID;         // [p h0 + q0, p] (h0 staged here)
  static constexpr int A1P = (GSB_HID + 1 + 3) / 4 * 4;
  static constexpr int oB1 = oA1 + A1P;             // delta1
  static constexpr int oV2 = oB1 + GSB_HID;         // p h1 + dd1 (.) m1
  static constexpr int oQ = oV2 + GSB_HID;          // q0 scratch
  static constexpr int ROW = oQ + GSB_HID;
};

template <typename T, int C>
__device__ __forceinline__ void scatter_level(const LevelDev& L, const LocT<T>& q, const T* gl,
                                              const T (&coef)[8], bool active, bool aggregate) {
  const unsigned full = 0xffffffffu;
  if (aggregate) {
    // every lane shares one cell (coarse levels): reduce across the warp first
    const int b0 = __shfl_sync(full, q.base, 0);
    if (__all_sync(full, !active || q.base == b0)) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        T v[C];
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = warp_sum(active ? gl[c] * coef[k] : T(0));
        if ((threadIdx.x & 31) == 0) {
          T* dst = reinterpret_cast<T*>(L.grad) + ((int64_t)b0 + corner_off(L, k)) * C;
          red_row<T, C>(dst, v);
        }
      }
      return;
    }
  }
  if (!active) return;
  T* Gp = reinterpret_cast<T*>(L.grad) + (int64_t)q.base * C;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    T v[C];
#pragma unroll
    for (int c = 0; c < C; ++c) v[c] = gl[c] * coef[k];
    red_row<T, C>(Gp + corner_off(L, k) * C, v);
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
  for (int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * 32; base < NS; base += nwarps * 32) {
    const int64_t s = base + lane;
    const bool active = s < NS;
    T p = T(0), u[3] = {T(0), T(0), T(0)}, pt[3];
    if (active) {
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
    } else {
      // inactive lanes evaluate a valid point and contribute zero
#pragma unroll
      for (int a = 0; a < 3; ++a) pt[a] = (T)G.lo[a];
    }
    LocT<T> loc[S::NL];
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      loc[l] = compact<T>(locate<false>(G.lv[l], (double)pt[0], (double)pt[1], (double)pt[2], nullptr));
      T f[S::CG];
      gather_fast<T, S::CG>(G.lv[l], loc[l], f);
#pragma unroll
      for (int c = 0; c < S::CG; ++c) myrow[R::oA0 + l * S::CG + c] = f[c];
    }
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
      load32(myrow + R::oA1, h);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) h[j] *= p;
      store32(myrow + R::oA1, h);                          // p h0
      myrow[R::oA1 + GSB_HID] = p;
    }
    T gz[S::IN_G];
    {
      T d[GSB_HID];
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) d[j] = ((m1 >> j) & 1u) ? sw[S::oGW2 + j] : T(0);
      store32(myrow + R::oB1, d);                          // delta1
      dense_d_row<T, GSB_HID>(sw + S::oGW1, d, m0, myrow + R::oB0);   // delta0
      load32(myrow + R::oB0, d);
      dense_d_reg<T, S::IN_G>(sw + S::oGW0, d, gz);        // g = dphi/dz
    }
    // per level: ju, v = theta . ju, scatter g_l (p w_k + ju_k)
    T v[S::IN_G];
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      const LevelDev& L = G.lv[l];
      const LocT<T>& q = loc[l];
      const T x1 = q.fx, y1 = q.fy, z1 = q.fz;
      const T x0 = T(1) - x1, y0 = T(1) - y1, z0 = T(1) - z1;
      const T iv = (T)L.inv_vs;
      const T u0 = u[0] * iv, u1 = u[1] * iv, u2 = u[2] * iv;
      T coef[8];
      T vl[S::CG];
#pragma unroll
      for (int c = 0; c < S::CG; ++c) vl[c] = T(0);
      const T* F = reinterpret_cast<const T*>(L.feat) + (int64_t)q.base * S::CG;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int dx = (k >> 2) & 1, dy = (k >> 1) & 1, dz = k & 1;
        const T wx = dx ? x1 : x0, wy = dy ? y1 : y0, wz = dz ? z1 : z0;
        const T sx = dx ? T(1) : T(-1), sy = dy ? T(1) : T(-1), sz = dz ? T(1) : T(-1);
        const T ju = (sx * wy * wz) * u0 + (wx * sy * wz) * u1 + (wx * wy * sz) * u2;
        coef[k] = p * ((wx * wy) * wz) + ju;
        T row[S::CG];
        load_row<T, S::CG>(F + corner_off(L, k) * S::CG, row);
#pragma unroll
        for (int c = 0; c < S::CG; ++c) vl[c] = fma(row[c], ju, vl[c]);
      }
#pragma unroll
      for (int c = 0; c < S::CG; ++c) v[l * S::CG + c] = vl[c];
      scatter_level<T, S::CG>(L, q, gz + l * S::CG, coef, active, l < agg_levels);
    }
    // A0 = [p z + v, p]
#pragma unroll
    for (int i = 0; i < S::IN_G; ++i) myrow[R::oA0 + i] = fma(p, myrow[R::oA0 + i], v[i]);
    myrow[R::oA0 + S::IN_G] = p;
    // q0 = (v W0) (.) m0 -> A1 += q0 ; dd1 = (q0 W1) (.) m1 -> V2 += dd1
    {
      T q0[GSB_HID];
      dense_f_reg<T, S::IN_G>(sw + S::oGW0, v, q0);
      T a[GSB_HID];
      load32(myrow + R::oA1, a);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) {
        q0[j] = ((m0 >> j) & 1u) ? q0[j] : T(0);
        a[j] += q0[j];
      }
      store32(myrow + R::oA1, a);
      store32(myrow + R::oQ, q0);
      dense_f_row<T, GSB_HID>(sw + S::oGW1, myrow + R::oQ, q0);
      load32(myrow + R::oV2, a);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) a[j] += ((m1 >> j) & 1u) ? q0[j] : T(0);
      store32(myrow + R::oV2, a);
    }
    if (!active) {
#pragma unroll 1
      for (int i = 0; i < R::ROW; ++i) myrow[i] = T(0);
    }
    __syncwarp();
    warp_outer<T, R::A0, R::A0P, GSB_HID + 1, R::A1P>(rows, R::ROW, R::oA0, R::oB0, R::oA1, R::oB1,
                                                      lane, acc0, acc1);
#pragma unroll 1
    for (int r = 0; r < 32; ++r) {
      acc2 += rows[(size_t)r * R::ROW + R::oV2 + lane];
      accp += rows[(size_t)r * R::ROW + R::oA0 + S::IN_G];  // db2 = sum p
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
  T* out = w.mlp_part + (size_t)blockIdx.x * S::NMLP;
  for (int t = threadIdx.x; t < NGP; t += blockDim.x) {
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
      T* Gp = reinterpret_cast<T*>(G.col.grad) + (int64_t)q.base * S::CC;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        T vv[S::CC];
#pragma unroll
        for (int c = 0; c < S::CC; ++c) vv[c] = wk[k] * fb[c];
        red_row<T, S::CC>(Gp + corner_off(G.col, k) * S::CC, vv);
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
  T* out = w.mlp_part + (size_t)blockIdx.x * S::NMLP + S::NG;
  for (int t = threadIdx.x; t < NCP; t += blockDim.x) {
    T a = T(0);
#pragma unroll
    for (int k = 0; k < WARPS; ++k) a += red[(size_t)k * NCP + t];
    out[t] = a;
  }
}

// ---------------------------------------------------------------------------
// deterministic finalization

template <typename T, class S>
__global__ void k_finalize_mlp(Ws<T> w, T* grads, int64_t mlp_off, int nb_geo, int nb_col) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S::NMLP) return;
  int nb = t < S::NG ? nb_geo : nb_col;
  double a = 0.0;
  for (int b = 0; b < nb; ++b) a += (double)w.mlp_part[(size_t)b * S::NMLP + t];
  grads[mlp_off + t] += (T)a;
}

template <typename T>
__global__ void k_finalize_loss(Ws<T> w, int M, int S, T* grads, const T* params, int64_t log_s_off,
                                LossW L) {
  __shared__ double red[7][32];
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    const double* p = w.ray_part + (int64_t)i * 8;
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] += p[k];
  }
  for (int j = threadIdx.x; j < S; j += blockDim.x) acc[6] += w.smooth_part[j];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    double v = warp_sum(acc[k]);
    if (lane == 0) red[k][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < 7; ++k)
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot[k] += red[k][q];
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
}

// ---------------------------------------------------------------------------
// Adam over the arena (gs/optimizer.py:38-55): float64 math, storage dtype,
// non-finite gradients zeroed and counted, gradient cleared.

struct AdamSegs {
  int64_t begin[16];
  double lr[16];
  int n;
};

template <typename T>
__device__ __forceinline__ void adam_one(T& p, T& g, T& m, T& v, double lr, double b1, double b2,
                                         double eps, double c1, double c2, int& bad) {
  double gi = (double)g;
  if (!isfinite(gi)) {
    gi = 0.0;
    ++bad;
  }
  double mi = b1 * (double)m + (1.0 - b1) * gi;
  double vi = b2 * (double)v + (1.0 - b2) * gi * gi;
  m = (T)mi;
  v = (T)vi;
  p = (T)((double)p - lr * (mi / c1) / (sqrt(vi / c2) + eps));
  g = T(0);
}

template <typename T>
__global__ void __launch_bounds__(256) k_adam(T* __restrict__ P, T* __restrict__ Gr, T* __restrict__ Mm,
                                              T* __restrict__ Vv, int64_t n, AdamSegs segs, double b1,
                                              double b2, double eps, double c1, double c2,
                                              const double* guard, double thr, int32_t* status) {
  if (guard) {
    double tot = guard[0];
    if (!(tot == tot) || isinf(tot) || tot > thr || status[GSB_ST_DIVERGED]) {
      if (blockIdx.x == 0 && threadIdx.x == 0) status[GSB_ST_DIVERGED] = 1;
      return;
    }
  }
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
  using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  int bad = 0;
  const int64_t nvec = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = i * V;
    int sidx = 0;
    for (int k = 1; k < segs.n; ++k)
      if (e >= segs.begin[k]) sidx = k;
    double lr = segs.lr[sidx];
    Vec p = reinterpret_cast<Vec*>(P)[i];
    Vec g = reinterpret_cast<Vec*>(Gr)[i];
    Vec m = reinterpret_cast<Vec*>(Mm)[i];
    Vec v = reinterpret_cast<Vec*>(Vv)[i];
    T* pp = reinterpret_cast<T*>(&p);
    T* gg = reinterpret_cast<T*>(&g);
    T* mm = reinterpret_cast<T*>(&m);
    T* vv = reinterpret_cast<T*>(&v);
#pragma unroll
    for (int k = 0; k < V; ++k) adam_one(pp[k], gg[k], mm[k], vv[k], lr, b1, b2, eps, c1, c2, bad);
    reinterpret_cast<Vec*>(P)[i] = p;
    reinterpret_cast<Vec*>(Gr)[i] = g;
    reinterpret_cast<Vec*>(Mm)[i] = m;
    reinterpret_cast<Vec*>(Vv)[i] = v;
  }
  // tail
  for (int64_t e = nvec * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int sidx = 0;
    for (int k = 1; k < segs.n; ++k)
      if (e >= segs.begin[k]) sidx = k;
    adam_one(P[e], Gr[e], Mm[e], Vv[e], segs.lr[sidx], b1, b2, eps, c1, c2, bad);
  }
  bad = warp_sum(bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(status + GSB_ST_ADAM_BAD, bad);
}

}  // namespace gsb
