// gsb_mlp.cuh -- decoder MLP building blocks (gs/decoders.py:55-99) for
// thread-per-sample kernels.
//
// The weights of the 16->32->32->1 geometry and (C+3)->32->32->3 colour MLPs
// are staged once per CTA in shared memory (arena layout, see Shape).  All
// lanes of a warp read the same weights at the same time, so every 16-byte
// shared load is a broadcast that feeds four FMAs; loops are ordered so the
// contiguous weight index is innermost.
#pragma once

#include "gsb_common.cuh"

namespace gsb {

template <typename T>
__device__ __forceinline__ void lds4(const T* p, T& a, T& b, T& c, T& d) {
  if constexpr (sizeof(T) == 4) {
    float4 v = *reinterpret_cast<const float4*>(p);
    a = v.x; b = v.y; c = v.z; d = v.w;
  } else {
    double2 u = *reinterpret_cast<const double2*>(p);
    double2 v = *reinterpret_cast<const double2*>(p + 2);
    a = u.x; b = u.y; c = v.x; d = v.y;
  }
}

// out[j] = sum_i x[i] W[i][j] + b[j]   (W stored (in, 32) row-major)
template <typename T, int IN>
__device__ __forceinline__ void dense_fwd(const T* __restrict__ W, const T* __restrict__ b,
                                          const T* x, T (&out)[GSB_HID]) {
#pragma unroll
  for (int j = 0; j < GSB_HID; ++j) out[j] = T(0);
#pragma unroll
  for (int i = 0; i < IN; ++i) {
    const T xi = x[i];
#pragma unroll
    for (int j = 0; j < GSB_HID; j += 4) {
      T w0, w1, w2, w3;
      lds4(W + i * GSB_HID + j, w0, w1, w2, w3);
      out[j] = fma(xi, w0, out[j]);
      out[j + 1] = fma(xi, w1, out[j + 1]);
      out[j + 2] = fma(xi, w2, out[j + 2]);
      out[j + 3] = fma(xi, w3, out[j + 3]);
    }
  }
#pragma unroll
  for (int j = 0; j < GSB_HID; j += 4) {
    T b0, b1, b2, b3;
    lds4(b + j, b0, b1, b2, b3);
    out[j] += b0;
    out[j + 1] += b1;
    out[j + 2] += b2;
    out[j + 3] += b3;
  }
}

// y[i] = sum_j W[i][j] x[j]   (rows of W contiguous; the transposed product
// of the backward pass)
template <typename T, int OUT>
__device__ __forceinline__ void dense_bwd(const T* __restrict__ W, const T (&x)[GSB_HID], T* y) {
#pragma unroll
  for (int i = 0; i < OUT; ++i) {
    T a0 = T(0), a1 = T(0);
#pragma unroll
    for (int j = 0; j < GSB_HID; j += 4) {
      T w0, w1, w2, w3;
      lds4(W + i * GSB_HID + j, w0, w1, w2, w3);
      a0 = fma(w0, x[j], a0);
      a1 = fma(w1, x[j + 1], a1);
      a0 = fma(w2, x[j + 2], a0);
      a1 = fma(w3, x[j + 3], a1);
    }
    y[i] = a0 + a1;
  }
}

template <typename T>
__device__ __forceinline__ uint32_t relu_mask(T (&h)[GSB_HID]) {
  uint32_t m = 0u;
#pragma unroll
  for (int j = 0; j < GSB_HID; ++j) {
    const bool pos = h[j] > T(0);  // gs/diffcore.py:483-492 (mask a > 0)
    h[j] = pos ? h[j] : T(0);
    m |= (uint32_t)pos << j;
  }
  return m;
}

template <typename T>
__device__ __forceinline__ T dot32(const T* __restrict__ w, const T (&x)[GSB_HID]) {
  T a0 = T(0), a1 = T(0);
#pragma unroll
  for (int j = 0; j < GSB_HID; j += 4) {
    T w0, w1, w2, w3;
    lds4(w + j, w0, w1, w2, w3);
    a0 = fma(x[j], w0, a0);
    a1 = fma(x[j + 1], w1, a1);
    a0 = fma(x[j + 2], w2, a0);
    a1 = fma(x[j + 3], w3, a1);
  }
  return a0 + a1;
}

// stage the MLP block (arena layout) into shared memory
template <typename T, class S>
__device__ __forceinline__ void stage_weights(T* sw, const T* __restrict__ mlp, int first, int count) {
  for (int t = threadIdx.x; t < count; t += blockDim.x) sw[first + t] = mlp[first + t];
}

// ---------------------------------------------------------------------------
// per-level location kept across the MLP (compact: vertex index + fractions)

template <typename T>
struct LocT {
  int32_t base;
  T fx, fy, fz;
};

template <typename T>
__device__ __forceinline__ LocT<T> compact(const Loc& q) {
  LocT<T> r;
  r.base = (int32_t)q.base;
  r.fx = (T)q.fx;
  r.fy = (T)q.fy;
  r.fz = (T)q.fz;
  return r;
}

template <typename T>
__device__ __forceinline__ void corner_w(const LocT<T>& q, T (&w)[8]) {
  const T x1 = q.fx, y1 = q.fy, z1 = q.fz;
  const T x0 = T(1) - x1, y0 = T(1) - y1, z0 = T(1) - z1;
  const T a00 = x0 * y0, a01 = x0 * y1, a10 = x1 * y0, a11 = x1 * y1;
  w[0] = a00 * z0; w[1] = a00 * z1; w[2] = a01 * z0; w[3] = a01 * z1;
  w[4] = a10 * z0; w[5] = a10 * z1; w[6] = a11 * z0; w[7] = a11 * z1;
}

template <typename T, int C>
__device__ __forceinline__ void gather_fast(const LevelDev& L, const LocT<T>& q, T* out) {
  const T* F = reinterpret_cast<const T*>(L.feat) + (int64_t)q.base * C;
  T w[8];
  corner_w(q, w);
#pragma unroll
  for (int c = 0; c < C; ++c) out[c] = T(0);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    T row[C];
    load_row<T, C>(F + corner_off(L, k) * C, row);
#pragma unroll
    for (int c = 0; c < C; ++c) out[c] = fma(w[k], row[c], out[c]);
  }
}

// gather_fast plus the level's spatial Jacobian of the features,
// J[c][a] = d/dfrac_a sum_k w_k theta_k[c] (grid units; gs/diffcore.py:844-871
// before the 1/vs), from the same corner rows: grad phi then needs
// g . J instead of a second read of the corners
template <typename T, int C>
__device__ __forceinline__ void jac_from_rows(const LocT<T>& q, const T (&r)[8][C], T* out, T (&J)[3 * C]) {
  T w[8];
  corner_w(q, w);
  const T x1 = q.fx, y1 = q.fy, z1 = q.fz;
  const T x0 = T(1) - x1, y0 = T(1) - y1, z0 = T(1) - z1;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = fma(w[k], r[k][c], acc);
    out[c] = acc;
    J[3 * c + 0] = (r[4][c] - r[0][c]) * (y0 * z0) + (r[5][c] - r[1][c]) * (y0 * z1) +
                   (r[6][c] - r[2][c]) * (y1 * z0) + (r[7][c] - r[3][c]) * (y1 * z1);
    J[3 * c + 1] = (r[2][c] - r[0][c]) * (x0 * z0) + (r[3][c] - r[1][c]) * (x0 * z1) +
                   (r[6][c] - r[4][c]) * (x1 * z0) + (r[7][c] - r[5][c]) * (x1 * z1);
    J[3 * c + 2] = (r[1][c] - r[0][c]) * (x0 * y0) + (r[3][c] - r[2][c]) * (x0 * y1) +
                   (r[5][c] - r[4][c]) * (x1 * y0) + (r[7][c] - r[6][c]) * (x1 * y1);
  }
}
template <typename T, int C>
__device__ __forceinline__ void gather_jac(const LevelDev& L, const LocT<T>& q, T* out, T (&J)[3 * C]) {
  const T* F = reinterpret_cast<const T*>(L.feat) + (int64_t)q.base * C;
  T r[8][C];
#pragma unroll
  for (int k = 0; k < 8; ++k) load_row<T, C>(F + corner_off(L, k) * C, r[k]);
  jac_from_rows<T, C>(q, r, out, J);
}

// grad phi contribution g . J / vs of a level whose Jacobian was kept
template <typename T, int C>
__device__ __forceinline__ void level_dx_jac(const LevelDev& L, const T (&J)[3 * C], const T* gl,
                                             T (&gr)[3]) {
  const T iv = (T)L.inv_vs;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    T acc = T(0);
#pragma unroll
    for (int c = 0; c < C; ++c) acc = fma(gl[c], J[3 * c + a], acc);
    gr[a] += acc * iv;
  }
}

// d/dx <interp(theta, x), g>  (gs/diffcore.py:844-871)
template <typename T, int C>
__device__ __forceinline__ void level_dx_fast(const LevelDev& L, const LocT<T>& q, const T* gl,
                                              T (&gr)[3]) {
  const T* F = reinterpret_cast<const T*>(L.feat) + (int64_t)q.base * C;
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
  const T x1 = q.fx, y1 = q.fy, z1 = q.fz;
  const T x0 = T(1) - x1, y0 = T(1) - y1, z0 = T(1) - z1;
  const T iv = (T)L.inv_vs;
  gr[0] += ((e[4] - e[0]) * (y0 * z0) + (e[5] - e[1]) * (y0 * z1) + (e[6] - e[2]) * (y1 * z0) +
            (e[7] - e[3]) * (y1 * z1)) * iv;
  gr[1] += ((e[2] - e[0]) * (x0 * z0) + (e[3] - e[1]) * (x0 * z1) + (e[6] - e[4]) * (x1 * z0) +
            (e[7] - e[5]) * (x1 * z1)) * iv;
  gr[2] += ((e[1] - e[0]) * (x0 * y0) + (e[3] - e[2]) * (x0 * y1) + (e[5] - e[4]) * (x1 * y0) +
            (e[7] - e[6]) * (x1 * y1)) * iv;
}

// sample point of (ray, slot) in the model dtype: x = o + d r, clipped
// (gs/renderer.py:349-355; d cast to the dtype, mul then add)
template <typename T>
__device__ __forceinline__ void taped_point(const T* __restrict__ o, const T* __restrict__ r,
                                            double dep, const double* lo, const double* hi,
                                            T (&p)[3]) {
  const T d = (T)dep;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    T x = o[a] + d * r[a];
    const T l = (T)lo[a], h = (T)hi[a];
    x = x >= l ? x : l;
    x = x <= h ? x : h;
    p[a] = x;
  }
}

}  // namespace gsb

namespace gsb {

// ---------------------------------------------------------------------------
// Row-staged layer products.  Each thread owns one shared-memory row of its
// sample's activations (16-byte aligned); outer loops stay rolled so live
// ranges are bounded, the 32-wide inner loop is unrolled.

template <typename T>
__device__ __forceinline__ void sts4(T* p, T a, T b, T c, T d) {
  if constexpr (sizeof(T) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
  } else {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
    *reinterpret_cast<double2*>(p + 2) = make_double2(c, d);
  }
}

// acc[j] += x * W[j], j < 32 (W contiguous, broadcast reads)
template <typename T>
__device__ __forceinline__ void axpy32(const T* __restrict__ W, T x, T (&acc)[GSB_HID]) {
#pragma unroll
  for (int j = 0; j < GSB_HID; j += 4) {
    T w0, w1, w2, w3;
    lds4(W + j, w0, w1, w2, w3);
    acc[j] = fma(x, w0, acc[j]);
    acc[j + 1] = fma(x, w1, acc[j + 1]);
    acc[j + 2] = fma(x, w2, acc[j + 2]);
    acc[j + 3] = fma(x, w3, acc[j + 3]);
  }
}

// acc[j] = sum_{i<IN} xr[i] W[i][j]   (inputs from the thread's own row)
template <typename T, int IN>
__device__ __forceinline__ void dense_f_row(const T* __restrict__ W, const T* xr,
                                            T (&acc)[GSB_HID]) {
#pragma unroll
  for (int j = 0; j < GSB_HID; ++j) acc[j] = T(0);
  constexpr int IN4 = IN / 4;
#pragma unroll 1
  for (int i4 = 0; i4 < IN4; ++i4) {
    T x0, x1, x2, x3;
    lds4(xr + 4 * i4, x0, x1, x2, x3);
    const T* w = W + 4 * i4 * GSB_HID;
    axpy32(w, x0, acc);
    axpy32(w + GSB_HID, x1, acc);
    axpy32(w + 2 * GSB_HID, x2, acc);
    axpy32(w + 3 * GSB_HID, x3, acc);
  }
#pragma unroll
  for (int i = IN4 * 4; i < IN; ++i) axpy32(W + i * GSB_HID, xr[i], acc);
}

// acc[j] = sum_{i<IN} x[i] W[i][j]   (inputs in registers)
template <typename T, int IN>
__device__ __forceinline__ void dense_f_reg(const T* __restrict__ W, const T* x,
                                            T (&acc)[GSB_HID]) {
#pragma unroll
  for (int j = 0; j < GSB_HID; ++j) acc[j] = T(0);
#pragma unroll
  for (int i = 0; i < IN; ++i) axpy32(W + i * GSB_HID, x[i], acc);
}

template <typename T>
__device__ __forceinline__ void add_bias(const T* __restrict__ b, T (&acc)[GSB_HID]) {
#pragma unroll
  for (int j = 0; j < GSB_HID; j += 4) {
    T b0, b1, b2, b3;
    lds4(b + j, b0, b1, b2, b3);
    acc[j] += b0;
    acc[j + 1] += b1;
    acc[j + 2] += b2;
    acc[j + 3] += b3;
  }
}

// yr[o] = mask_o ? sum_j W[o][j] x[j] : 0, o < OUT (OUT % 4 == 0), to own row
template <typename T, int OUT>
__device__ __forceinline__ void dense_d_row(const T* __restrict__ W, const T (&x)[GSB_HID],
                                            uint32_t mask, T* yr) {
  static_assert(OUT % 4 == 0, "row outputs in groups of 4");
#pragma unroll 1
  for (int o4 = 0; o4 < OUT / 4; ++o4) {
    const T* w = W + 4 * o4 * GSB_HID;
    T y0 = dot32(w, x), y1 = dot32(w + GSB_HID, x), y2 = dot32(w + 2 * GSB_HID, x),
      y3 = dot32(w + 3 * GSB_HID, x);
    const uint32_t m = mask >> (4 * o4);
    sts4(yr + 4 * o4, (m & 1u) ? y0 : T(0), (m & 2u) ? y1 : T(0), (m & 4u) ? y2 : T(0),
         (m & 8u) ? y3 : T(0));
  }
}

// y[o] = sum_j W[o][j] x[j], o < OUT, to registers
template <typename T, int OUT>
__device__ __forceinline__ void dense_d_reg(const T* __restrict__ W, const T (&x)[GSB_HID],
                                            T* y) {
#pragma unroll
  for (int o = 0; o < OUT; ++o) y[o] = dot32(W + o * GSB_HID, x);
}

template <typename T>
__device__ __forceinline__ void load32(const T* r, T (&x)[GSB_HID]) {
#pragma unroll
  for (int j = 0; j < GSB_HID; j += 4) lds4(r + j, x[j], x[j + 1], x[j + 2], x[j + 3]);
}

template <typename T>
__device__ __forceinline__ void store32(T* r, const T (&x)[GSB_HID]) {
#pragma unroll
  for (int j = 0; j < GSB_HID; j += 4) sts4(r + j, x[j], x[j + 1], x[j + 2], x[j + 3]);
}

}  // namespace gsb
