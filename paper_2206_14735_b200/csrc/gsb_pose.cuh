// gsb_pose.cuh -- pose refinement: realised poses of the
// step and the gradients of the trainable (nu_f, t_f).
//
//   k_pose_table   R_f = R0_f exp_so3(nu_f) in the model dtype (the graph form,
//                  gs/camera.py:68-70, 96-122) -> ray table; and R0 exp_so3_data(nu)
//                  in f64 (PoseParam.matrix, gs/camera.py:75-80, 125-139) -> the
//                  smoothness-point table
//   k_pose_xbar    per taped sample: the cotangent of the tracked point
//                  (phi path J^T zbar, grad-phi path = in-cell Hessian block,
//                  colour path J_c^T fc_bar; gs/diffcore.py:893-991), zeroed
//                  where the clip is active, and the view-direction cotangent
//   k_pose_ray     per ray: o_bar = sum_n x_bar, r_bar = sum_n d x_bar + vdir_bar
//                  (gs/renderer.py:349-351, 361-364)
//   k_pose_frames  per frame: R_bar = sum r_bar dir_cam^T, t_bar = sum o_bar over the
//                  frame's rays (gs/renderer.py:304-309), then the exp_so3 adjoint;
//                  ACCUMULATED into the gradient arena
#pragma once

#include "gsb_kernels.cuh"

namespace gsb {

// --------------------------------------------------------------------------
// exp_so3 in the model dtype, as the graph evaluates it (gs/camera.py:96-122)

template <typename T>
struct So3 {
  T K[9], K2[9], th2, th, a, b;
  bool small;
};

template <typename T>
__device__ __forceinline__ So3<T> so3_graph(const T (&nu)[3], T (&E)[9]) {
  So3<T> q;
  const T z = T(0);
  const T K[9] = {z, -nu[2], nu[1], nu[2], z, -nu[0], -nu[1], nu[0], z};
#pragma unroll
  for (int i = 0; i < 9; ++i) q.K[i] = K[i];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      q.K2[i * 3 + j] = (K[i * 3] * K[j] + K[i * 3 + 1] * K[3 + j]) + K[i * 3 + 2] * K[6 + j];
  q.th2 = (nu[0] * nu[0] + nu[1] * nu[1]) + nu[2] * nu[2];
  q.small = sqrt((double)q.th2) < 1e-4;  // gs/camera.py:93, 110
  if (q.small) {
    q.a = (T(1) + q.th2 * T(-1.0 / 6.0)) + (q.th2 * q.th2) * T(1.0 / 120.0);
    q.b = (T(0.5) + q.th2 * T(-1.0 / 24.0)) + (q.th2 * q.th2) * T(1.0 / 720.0);
    q.th = T(0);
  } else {
    q.th = sqrt(q.th2);
    q.a = sin(q.th) / q.th;
    q.b = (T(1) - cos(q.th)) / q.th2;
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) E[i] = ((i % 4 == 0 ? T(1) : T(0)) + q.a * q.K[i]) + q.b * q.K2[i];
  return q;
}

// d/dnu <E(nu), Ebar> through the same graph
template <typename T>
__device__ __forceinline__ void so3_adjoint(const T (&nu)[3], const So3<T>& q, const T (&Eb)[9], T (&nub)[3]) {
  T ab = T(0), bb = T(0);
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    ab += Eb[i] * q.K[i];
    bb += Eb[i] * q.K2[i];
  }
  T Kb[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      // K2 = K K:  Kbar += K2bar K^T + K^T K2bar,  K2bar = b Ebar
      T s = T(0);
#pragma unroll
      for (int k = 0; k < 3; ++k) s += q.b * Eb[i * 3 + k] * q.K[j * 3 + k] + q.K[k * 3 + i] * q.b * Eb[k * 3 + j];
      Kb[i * 3 + j] = q.a * Eb[i * 3 + j] + s;
    }
  T th2b;
  if (q.small) {
    th2b = ab * (T(-1.0 / 6.0) + T(2.0 / 120.0) * q.th2) + bb * (T(-1.0 / 24.0) + T(2.0 / 720.0) * q.th2);
  } else {
    const T s = sin(q.th), c = cos(q.th);
    const T thb = ab * (c / q.th - s / (q.th * q.th)) + bb * (s / q.th2);
    th2b = thb / (T(2) * q.th) - bb * (T(1) - c) / (q.th2 * q.th2);
  }
  nub[0] = T(2) * nu[0] * th2b + (Kb[7] - Kb[5]);
  nub[1] = T(2) * nu[1] * th2b + (Kb[2] - Kb[6]);
  nub[2] = T(2) * nu[2] * th2b + (Kb[3] - Kb[1]);
}

// exp_so3_data (gs/camera.py:125-139), f64
__device__ __forceinline__ void so3_data(const double (&nu)[3], double (&E)[9]) {
  const double th2 = (nu[0] * nu[0] + nu[1] * nu[1]) + nu[2] * nu[2];
  const double K[9] = {0.0, -nu[2], nu[1], nu[2], 0.0, -nu[0], -nu[1], nu[0], 0.0};
  double a, b;
  if (sqrt(th2) < 1e-4) {
    a = (1.0 - th2 / 6.0) + th2 * th2 / 120.0;
    b = (0.5 - th2 / 24.0) + th2 * th2 / 720.0;
  } else {
    const double th = sqrt(th2);
    a = sin(th) / th;
    b = (1.0 - cos(th)) / th2;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double kk = (K[i * 3] * K[j] + K[i * 3 + 1] * K[3 + j]) + K[i * 3 + 2] * K[6 + j];
      E[i * 3 + j] = ((i == j ? 1.0 : 0.0) + a * K[i * 3 + j]) + b * kk;
    }
}

// one thread per frame: table (F,12) model-dtype values, table64 (F,12) f64
template <typename T>
__global__ void k_pose_table(gsb_pose_t P, const T* __restrict__ params, double* __restrict__ tab,
                             double* __restrict__ tab64) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= P.n_frames) return;
  const int64_t no = P.nu_offset[f], to = P.t_offset[f];
  T nu[3], t[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    nu[a] = no >= 0 ? params[no + a] : T(0);
    t[a] = to >= 0 ? params[to + a] : (T)P.t_fixed[f * 3 + a];
  }
  T E[9];
  so3_graph<T>(nu, E);
  T R0c[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R0c[i] = (T)P.R0[f * 9 + i];
  double nud[3] = {(double)nu[0], (double)nu[1], (double)nu[2]}, Ed[9];
  so3_data(nud, Ed);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const T r = (R0c[i * 3] * E[j] + R0c[i * 3 + 1] * E[3 + j]) + R0c[i * 3 + 2] * E[6 + j];
      tab[f * 12 + i * 3 + j] = (double)r;
      const double* R0 = P.R0 + f * 9;
      tab64[f * 12 + i * 3 + j] = (R0[i * 3] * Ed[j] + R0[i * 3 + 1] * Ed[3 + j]) + R0[i * 3 + 2] * Ed[6 + j];
    }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    tab[f * 12 + 9 + a] = (double)t[a];
    tab64[f * 12 + 9 + a] = (double)t[a];
  }
}

// --------------------------------------------------------------------------
// per-sample point cotangent

// sum_k e_k dw_k/dx (cell units) and the off-diagonal Hessian of
// sum_k e_k w_k (gs/diffcore.py:783-804)
__device__ __forceinline__ void corner_grad_hess(const double (&e)[8], double fx, double fy, double fz,
                                                 double (&gr)[3], double (&h)[3]) {
  const double x0 = 1.0 - fx, y0 = 1.0 - fy, z0 = 1.0 - fz;
  gr[0] = (e[4] - e[0]) * (y0 * z0) + (e[5] - e[1]) * (y0 * fz) + (e[6] - e[2]) * (fy * z0) +
          (e[7] - e[3]) * (fy * fz);
  gr[1] = (e[2] - e[0]) * (x0 * z0) + (e[3] - e[1]) * (x0 * fz) + (e[6] - e[4]) * (fx * z0) +
          (e[7] - e[5]) * (fx * fz);
  gr[2] = (e[1] - e[0]) * (x0 * y0) + (e[3] - e[2]) * (x0 * fy) + (e[5] - e[4]) * (fx * y0) +
          (e[7] - e[6]) * (fx * fy);
  h[0] = z0 * (e[0] + e[6] - e[2] - e[4]) + fz * (e[1] + e[7] - e[3] - e[5]);  // h12
  h[1] = y0 * (e[0] + e[5] - e[1] - e[4]) + fy * (e[2] + e[7] - e[3] - e[6]);  // h13
  h[2] = x0 * (e[0] + e[3] - e[1] - e[2]) + fx * (e[4] + e[7] - e[5] - e[6]);  // h23
}

// e_k = sum_c theta[idx_k, c] g_c (storage-dtype products, f64 accumulator,
// as _nb_dx_forward's per-corner contraction)
template <typename T, int C>
__device__ __forceinline__ void corner_contract(const LevelDev& L, int64_t base, const T* g, double (&e)[8]) {
  const T* F = reinterpret_cast<const T*>(L.feat) + base * C;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    T row[C];
    load_row<T, C>(F + corner_off(L, k) * C, row);
    double a = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) a += (double)(row[c] * g[c]);
    e[k] = a;
  }
}

template <typename T, class S>
__global__ void __launch_bounds__(128) k_pose_xbar(Ws<T> w, Geo G, int M, int N,
                                                   const double* __restrict__ dep,
                                                   const T* __restrict__ mlp, T* __restrict__ xbar) {
  using R = FwdRow<T, S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sw = reinterpret_cast<T*>(smem_raw);
  T* myrow = sw + (S::NMLP + 3) / 4 * 4 + (size_t)threadIdx.x * R::ROW;
  stage_weights<T, S>(sw, mlp, 0, S::NMLP);
  __syncthreads();
  const int64_t MN = (int64_t)M * N;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= MN) return;
  const int ray = (int)(s / N), j = (int)(s % N);
  // x = o + d r in the dtype, clip (gs/renderer.py:349-355); the clip passes
  // the cotangent where lo <= x <= hi (maximum / minimum ties, gs/diffcore.py:506-529)
  T p[3];
  bool inside[3];
  {
    const T d = (T)dep[(int64_t)ray * w.ld + j];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      T x = w.o[ray * 3 + a] + d * w.r[ray * 3 + a];
      const T l = (T)G.lo[a], h = (T)G.hi[a];
      inside[a] = x >= l && x <= h;
      x = x >= l ? x : l;
      x = x <= h ? x : h;
      p[a] = x;
    }
  }
  // geometry forward: masks, then g = dphi/dz
  LocT<T> loc[S::NL];
#pragma unroll
  for (int l = 0; l < S::NL; ++l) {
    loc[l] = compact<T>(locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2], nullptr));
    T f[S::CG];
    gather_fast<T, S::CG>(G.lv[l], loc[l], f);
#pragma unroll
    for (int c = 0; c < S::CG; ++c) myrow[R::oZ + l * S::CG + c] = f[c];
  }
  T gz[S::IN_G];
  {
    T h[GSB_HID];
    dense_f_row<T, S::IN_G>(sw + S::oGW0, myrow + R::oZ, h);
    add_bias(sw + S::oGb0, h);
    const uint32_t m0 = relu_mask(h);
    store32(myrow + R::oH, h);
    dense_f_row<T, GSB_HID>(sw + S::oGW1, myrow + R::oH, h);
    add_bias(sw + S::oGb1, h);
    const uint32_t m1 = relu_mask(h);
    T d[GSB_HID];
#pragma unroll
    for (int jj = 0; jj < GSB_HID; ++jj) d[jj] = ((m1 >> jj) & 1u) ? sw[S::oGW2 + jj] : T(0);
    dense_d_row<T, GSB_HID>(sw + S::oGW1, d, m0, myrow + R::oD);
    load32(myrow + R::oD, d);
    dense_d_reg<T, S::IN_G>(sw + S::oGW0, d, gz);
  }
  const double pb = (double)w.pbar[s];
  const double u[3] = {(double)w.ubar[s * 3], (double)w.ubar[s * 3 + 1], (double)w.ubar[s * 3 + 2]};
  double xb[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int l = 0; l < S::NL; ++l) {
    const LevelDev& L = G.lv[l];
    double e[8], gr[3], h[3];
    corner_contract<T, S::CG>(L, loc[l].base, gz + l * S::CG, e);
    corner_grad_hess(e, (double)loc[l].fx, (double)loc[l].fy, (double)loc[l].fz, gr, h);
    const double iv = L.inv_vs, iv2 = 1.0 / (L.vs * L.vs);
    // phi path: J^T (p g); grad-phi path: Hessian block against u
    xb[0] += gr[0] * iv * pb + (h[0] * u[1] + h[1] * u[2]) * iv2;
    xb[1] += gr[1] * iv * pb + (h[0] * u[0] + h[2] * u[2]) * iv2;
    xb[2] += gr[2] * iv * pb + (h[1] * u[0] + h[2] * u[1]) * iv2;
  }
  // colour: sigma(MLP_c([f_c, r])) backprop to the input (gs/decoders.py:86-99)
  const Loc qc = locate<false>(G.col, (double)p[0], (double)p[1], (double)p[2], nullptr);
  {
    T f[S::CC];
    gather_fast<T, S::CC>(G.col, compact<T>(qc), f);
#pragma unroll
    for (int c = 0; c < S::CC; ++c) myrow[R::oZ + c] = f[c];
#pragma unroll
    for (int a = 0; a < 3; ++a) myrow[R::oZ + S::CC + a] = w.r[ray * 3 + a];
  }
  T inb[S::IN_C];
  {
    T h[GSB_HID];
    dense_f_row<T, S::IN_C>(sw + S::oCW0, myrow + R::oZ, h);
    add_bias(sw + S::oCb0, h);
    const uint32_t m0 = relu_mask(h);
    store32(myrow + R::oH, h);
    dense_f_row<T, GSB_HID>(sw + S::oCW1, myrow + R::oH, h);
    add_bias(sw + S::oCb1, h);
    const uint32_t m1 = relu_mask(h);
    T yb[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T cc = w.scol[s * 3 + c];
      yb[c] = w.cbar[s * 3 + c] * (cc * (T(1) - cc));
    }
    T d[GSB_HID];
#pragma unroll
    for (int jj = 0; jj < GSB_HID; ++jj) {
      const T a = (sw[S::oCW2 + jj * 3] * yb[0] + sw[S::oCW2 + jj * 3 + 1] * yb[1]) +
                  sw[S::oCW2 + jj * 3 + 2] * yb[2];
      d[jj] = ((m1 >> jj) & 1u) ? a : T(0);
    }
    dense_d_row<T, GSB_HID>(sw + S::oCW1, d, m0, myrow + R::oD);
    load32(myrow + R::oD, d);
    dense_d_reg<T, S::IN_C>(sw + S::oCW0, d, inb);
  }
  {
    double e[8], gr[3], h[3];
    corner_contract<T, S::CC>(G.col, qc.base, inb, e);
    corner_grad_hess(e, qc.fx, qc.fy, qc.fz, gr, h);
#pragma unroll
    for (int a = 0; a < 3; ++a) xb[a] += gr[a] * G.col.inv_vs;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    xbar[s * 6 + a] = inside[a] ? (T)xb[a] : T(0);
    xbar[s * 6 + 3 + a] = inb[S::CC + a];
  }
}

// float32 form: the step's k_fwd_tc left dphi/dz (w.pose_g) and k_bwd_color_tc
// the colour-input cotangent (w.pose_fb: f_bar, then the view-direction
// part); only the per-corner contractions remain (no MLP recomputation)
template <class S>
__global__ void __launch_bounds__(128) k_pose_fast(Ws<float> w, Geo G, int M, int N,
                                                   const double* __restrict__ dep, float* __restrict__ xbar) {
  const int64_t MN = (int64_t)M * N;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= MN) return;
  const int ray = (int)(s / N), j = (int)(s % N);
  float p[3];
  bool inside[3];
  {
    const float d = (float)dep[(int64_t)ray * w.ld + j];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float x = w.o[ray * 3 + a] + d * w.r[ray * 3 + a];
      const float l = (float)G.lo[a], h = (float)G.hi[a];
      inside[a] = x >= l && x <= h;
      x = x >= l ? x : l;
      x = x <= h ? x : h;
      p[a] = x;
    }
  }
  const double pb = (double)w.pbar[s];
  const double u[3] = {(double)w.ubar[s * 3], (double)w.ubar[s * 3 + 1], (double)w.ubar[s * 3 + 2]};
  double xb[3] = {0.0, 0.0, 0.0};
  const float* gz = w.pose_g + s * S::IN_G;
#pragma unroll
  for (int l = 0; l < S::NL; ++l) {
    const LevelDev& L = G.lv[l];
    const Loc q = locate<false>(L, (double)p[0], (double)p[1], (double)p[2], nullptr);
    float g[S::CG];
#pragma unroll
    for (int c = 0; c < S::CG; ++c) g[c] = gz[l * S::CG + c];
    double e[8], gr[3], h[3];
    corner_contract<float, S::CG>(L, q.base, g, e);
    corner_grad_hess(e, q.fx, q.fy, q.fz, gr, h);
    const double iv = L.inv_vs, iv2 = 1.0 / (L.vs * L.vs);
    xb[0] += gr[0] * iv * pb + (h[0] * u[1] + h[1] * u[2]) * iv2;
    xb[1] += gr[1] * iv * pb + (h[0] * u[0] + h[2] * u[2]) * iv2;
    xb[2] += gr[2] * iv * pb + (h[1] * u[0] + h[2] * u[1]) * iv2;
  }
  const float* fb = w.pose_fb + s * 12;
  {
    const Loc qc = locate<false>(G.col, (double)p[0], (double)p[1], (double)p[2], nullptr);
    float f[S::CC];
#pragma unroll
    for (int c = 0; c < S::CC; ++c) f[c] = fb[c];
    double e[8], gr[3], h[3];
    corner_contract<float, S::CC>(G.col, qc.base, f, e);
    corner_grad_hess(e, qc.fx, qc.fy, qc.fz, gr, h);
#pragma unroll
    for (int a = 0; a < 3; ++a) xb[a] += gr[a] * G.col.inv_vs;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    xbar[s * 6 + a] = inside[a] ? (float)xb[a] : 0.f;
    xbar[s * 6 + 3 + a] = fb[S::CC + a];
  }
}

// warp per ray: o_bar = sum x_bar, r_bar = sum d x_bar + vdir_bar, then (lane 0)
// R_bar = r_bar dir_cam^T (gs/renderer.py:307-309): rbar[ray] = (R_bar[9],
// o_bar[3], frame) in f64, stride kRbar
constexpr int kRbar = 16;

template <typename T>
__global__ void __launch_bounds__(128) k_pose_ray(Ws<T> w, gsb_dataset_t D, const int64_t* __restrict__ ids,
                                                  int M, int N, const double* __restrict__ dep,
                                                  const T* __restrict__ xbar, double* __restrict__ rbar) {
  const int lane = threadIdx.x & 31;
  const int ray = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (ray >= M) return;
  double v[6] = {0, 0, 0, 0, 0, 0};
  for (int jj = lane; jj < N; jj += 32) {
    const int64_t s = (int64_t)ray * N + jj;
    const T d = (T)dep[(int64_t)ray * w.ld + jj];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T x = xbar[s * 6 + a];
      v[a] += (double)x;
      v[3 + a] += (double)(d * x) + (double)xbar[s * 6 + 3 + a];
    }
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  if (lane != 0) return;
  const int64_t hw = (int64_t)D.height * D.width;
  const int64_t flat = ids[ray];
  const int64_t rem = flat % hw;
  const int pv = (int)(rem / D.width), pu = (int)(rem % D.width);
  // dir_cam (gs/camera.py:142-157) cast to the dtype (gs/renderer.py:308)
  const double dx = ((double)pu - D.cx) / D.fx, dy = ((double)pv - D.cy) / D.fy;
  const double nrm = sqrt((dx * dx + dy * dy) + 1.0);
  const T dc[3] = {(T)(dx / nrm), (T)(dy / nrm), (T)(1.0 / nrm)};
  double* o = rbar + (int64_t)ray * kRbar;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = 0; b < 3; ++b) o[a * 3 + b] = v[3 + a] * (double)dc[b];
    o[9 + a] = v[a];
  }
  o[12] = (double)(flat / hw);
}

// block per frame: R_bar, t_bar over the frame's rays, exp_so3 adjoint
template <typename T>
__global__ void __launch_bounds__(1024) k_pose_frames(int M, gsb_pose_t P, const T* __restrict__ params,
                                                     const double* __restrict__ rbar, T* __restrict__ grads) {
  const int f = blockIdx.x;
  const int64_t no = P.nu_offset[f], to = P.t_offset[f];
  if (no < 0 && to < 0) return;
  double acc[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) acc[i] = 0.0;
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    const double* r = rbar + (int64_t)i * kRbar;
    if ((int)r[12] != f) continue;
#pragma unroll
    for (int k = 0; k < 12; ++k) acc[k] += r[k];
  }
  __shared__ double red[32][12];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    if (lane == 0) red[wid][i] = acc[i];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 12; ++i) {
    double a = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) a += red[k][i];
    acc[i] = a;
  }
  if (to >= 0)
#pragma unroll
    for (int a = 0; a < 3; ++a) grads[to + a] += (T)acc[9 + a];
  if (no < 0) return;
  // R = R0c E:  Ebar = R0c^T R_bar
  T nu[3], E[9], Eb[9];
#pragma unroll
  for (int a = 0; a < 3; ++a) nu[a] = params[no + a];
  const So3<T> q = so3_graph<T>(nu, E);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T s = T(0);
#pragma unroll
      for (int k = 0; k < 3; ++k) s += (T)P.R0[f * 9 + k * 3 + i] * (T)acc[k * 3 + j];
      Eb[i * 3 + j] = s;
    }
  T nub[3];
  so3_adjoint<T>(nu, q, Eb, nub);
#pragma unroll
  for (int a = 0; a < 3; ++a) grads[no + a] += nub[a];
}

namespace host {

// pose scratch: [xbar MN x 6 T][rbar M x kRbar f64] and, float32, the step's
// per-sample [dphi/dz MN x IN_G][colour-input cotangent MN x 12]
struct PoseLayout {
  size_t xbar, rbar, g, fb, total;
};
template <typename T>
inline PoseLayout pose_layout(const Sizes& z, int in_g) {
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  PoseLayout L;
  L.xbar = 0;
  L.rbar = up((size_t)z.MN * 6 * sizeof(T));
  size_t o = up(L.rbar + (size_t)z.M * kRbar * sizeof(double));
  L.g = L.fb = 0;
  if (sizeof(T) == 4) {
    L.g = o;
    o = up(o + (size_t)z.MN * in_g * 4);
    L.fb = o;
    o = up(o + (size_t)z.MN * 12 * 4);
  }
  L.total = o;
  return L;
}
template <typename T>
inline size_t pose_scratch_bytes(const Sizes& z, int in_g) {
  return pose_layout<T>(z, in_g).total;
}

}  // namespace host
}  // namespace gsb
