// gsb_fast.cuh -- float32 production kernels for the taped pass.
//
// Weight feed: the MLP block lives in __constant__ memory (copied from the
// arena each step) and is read as float4 with compile-time offsets, which
// sm_100a serves through the uniform datapath (LDCU.128): four FFMAs per
// uniform load and no MIO traffic (tools/mb_weights.cu measured 63-71% of
// the FFMA peak this way vs ~8% for shared-memory broadcast).  Activations
// stay in registers (thread per sample).
//
// Weight gradients: the per-sample outer products
// dW0 += (p z + v) x delta0, dW1 += (p h0 + q0) x delta1, colour analogues,
// run on the tensor cores with mma.sync m16n8k8 TF32 in 3xTF32 split
// precision (hi*hi + hi*lo + lo*hi, ~fp32 accuracy), K = the warp's 32
// samples, operands read from per-sample shared-memory rows.
#pragma once

#include "gsb_mlp.cuh"

namespace gsb {

namespace {
__constant__ float4 c_w4[GSB_MLP_MAX / 4];  // one copy per translation unit
}

__device__ __forceinline__ float4 cw4(int i4) { return c_w4[i4]; }
__device__ __forceinline__ float cws(int i) {
  const float4 v = c_w4[i >> 2];
  switch (i & 3) {
    case 0: return v.x;
    case 1: return v.y;
    case 2: return v.z;
    default: return v.w;
  }
}

// acc[j] = sum_{i<IN} x[i] W[i][j] + b[j]; W at constant offset oW, b at oB
template <int IN, int oW, int oB>
__device__ __forceinline__ void cdense(const float* x, float (&acc)[GSB_HID]) {
#pragma unroll
  for (int j = 0; j < GSB_HID; ++j) acc[j] = 0.f;
#pragma unroll
  for (int i = 0; i < IN; ++i) {
#pragma unroll
    for (int j4 = 0; j4 < GSB_HID / 4; ++j4) {
      const float4 w = cw4((oW + i * GSB_HID) / 4 + j4);
      acc[4 * j4] = fmaf(x[i], w.x, acc[4 * j4]);
      acc[4 * j4 + 1] = fmaf(x[i], w.y, acc[4 * j4 + 1]);
      acc[4 * j4 + 2] = fmaf(x[i], w.z, acc[4 * j4 + 2]);
      acc[4 * j4 + 3] = fmaf(x[i], w.w, acc[4 * j4 + 3]);
    }
  }
  if (oB >= 0) {
#pragma unroll
    for (int j4 = 0; j4 < GSB_HID / 4; ++j4) {
      const float4 b = cw4(oB / 4 + j4);
      acc[4 * j4] += b.x;
      acc[4 * j4 + 1] += b.y;
      acc[4 * j4 + 2] += b.z;
      acc[4 * j4 + 3] += b.w;
    }
  }
}

// y[o] = sum_j W[o][j] x[j], o < OUT   (rows of W contiguous)
template <int OUT, int oW>
__device__ __forceinline__ void cdense_t(const float (&x)[GSB_HID], float* y) {
#pragma unroll
  for (int o = 0; o < OUT; ++o) {
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int j4 = 0; j4 < GSB_HID / 4; ++j4) {
      const float4 w = cw4((oW + o * GSB_HID) / 4 + j4);
      a0 = fmaf(w.x, x[4 * j4], a0);
      a1 = fmaf(w.y, x[4 * j4 + 1], a1);
      a0 = fmaf(w.z, x[4 * j4 + 2], a0);
      a1 = fmaf(w.w, x[4 * j4 + 3], a1);
    }
    y[o] = a0 + a1;
  }
}

template <int oW>
__device__ __forceinline__ float cdot32(const float (&x)[GSB_HID]) {
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int j4 = 0; j4 < GSB_HID / 4; ++j4) {
    const float4 w = cw4(oW / 4 + j4);
    a0 = fmaf(x[4 * j4], w.x, a0);
    a1 = fmaf(x[4 * j4 + 1], w.y, a1);
    a0 = fmaf(x[4 * j4 + 2], w.z, a0);
    a1 = fmaf(x[4 * j4 + 3], w.w, a1);
  }
  return a0 + a1;
}

__device__ __forceinline__ uint32_t relu_m(float (&h)[GSB_HID]) {
  uint32_t m = 0u;
#pragma unroll
  for (int j = 0; j < GSB_HID; ++j) {
    const bool pos = h[j] > 0.f;
    h[j] = pos ? h[j] : 0.f;
    m |= (uint32_t)pos << j;
  }
  return m;
}

// ---------------------------------------------------------------------------
// 3xTF32 mma.sync helpers (m16n8k8, row.col, fp32 accumulate)

__device__ __forceinline__ uint32_t tf32_of(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32_of(x);
  lo = tf32_of(x - __uint_as_float(hi));
}
// per-use split (3 integer/FP ops instead of two emulated cvt.rna): hi rounds
// the mantissa half-away at bit 13, lo = x - hi is exact and goes to the MMA
// raw (the tensor core ignores its low 13 bits): |x - hi - lo_tf32| <= 2^-21 |x|
__device__ __forceinline__ void split_fast(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// d += A B with A, B each split hi/lo (3 products)
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4],
                                     const uint32_t (&al)[4], uint32_t bh0, uint32_t bh1,
                                     uint32_t bl0, uint32_t bl1) {
  mma_tf32(d, al, bh0, bh1);
  mma_tf32(d, ah, bl0, bl1);
  mma_tf32(d, ah, bh0, bh1);
}

// A fragment of A^T (features x samples) from sample-major rows:
// a0 = row[k0+t][m0+g], a1 = row[k0+t][m0+g+8], a2 = row[k0+t+4][m0+g], a3 = row[k0+t+4][m0+g+8]
__device__ __forceinline__ void frag_a(const float* rows, int ROW, int off, int k0, int m0,
                                       uint32_t (&ah)[4], uint32_t (&al)[4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float* r0 = rows + (k0 + t) * ROW + off + m0 + g;
  const float* r1 = rows + (k0 + t + 4) * ROW + off + m0 + g;
  split_fast(r0[0], ah[0], al[0]);
  split_fast(r0[8], ah[1], al[1]);
  split_fast(r1[0], ah[2], al[2]);
  split_fast(r1[8], ah[3], al[3]);
}
// B fragment (samples x outputs) from rows: b0 = row[k0+t][n0+g], b1 = row[k0+t+4][n0+g]
__device__ __forceinline__ void frag_b(const float* rows, int ROW, int off, int k0, int n0,
                                       uint32_t& bh0, uint32_t& bh1, uint32_t& bl0,
                                       uint32_t& bl1) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  split_fast(rows[(k0 + t) * ROW + off + n0 + g], bh0, bl0);
  split_fast(rows[(k0 + t + 4) * ROW + off + n0 + g], bh1, bl1);
}

// scatter D fragments of an (m-tile, n-tile) into a row-major [rows][32] block
__device__ __forceinline__ void frag_d_store(const float (&d)[4], float* out, int m0, int n0,
                                             int mrows) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int r0 = m0 + g, r1 = m0 + g + 8, c = n0 + 2 * t;
  if (r0 < mrows) {
    out[r0 * GSB_HID + c] = d[0];
    out[r0 * GSB_HID + c + 1] = d[1];
  }
  if (r1 < mrows) {
    out[r1 * GSB_HID + c] = d[2];
    out[r1 * GSB_HID + c + 1] = d[3];
  }
}

// ---------------------------------------------------------------------------
// no-grad SDF at listed samples (importance passes)

template <class S>
__global__ void __launch_bounds__(128) k_sdf_eval_f(Ws<float> w, Geo G, int M, int Nc,
                                                    const double* __restrict__ dep,
                                                    double* __restrict__ phi,
                                                    const int32_t* __restrict__ list,
                                                    const int32_t* __restrict__ list_count) {
  const int64_t total = list ? (int64_t)(*list_count) : (int64_t)M * Nc;
  if (blockIdx.x * (int64_t)128 >= total) return;  // block-uniform
  {  // one point per thread (no loop: no hoisting of constant-bank loads)
    const int64_t t = blockIdx.x * (int64_t)128 + threadIdx.x;
    const bool act = t < total;
    int ray = 0, slot = 0;
    if (act) {
      if (list) {
        const int32_t e = list[t];
        ray = e / GSB_KMAX;
        slot = e % GSB_KMAX;
      } else {
        ray = (int)((uint32_t)t / (uint32_t)Nc);
        slot = (int)((uint32_t)t % (uint32_t)Nc);
      }
    }
    const double d = act ? dep[(int64_t)ray * w.ld + slot] : 0.0;
    float p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double x = w.od[ray * 3 + a] + d * w.rd[ray * 3 + a];
      x = x >= G.lo[a] ? x : G.lo[a];
      x = x <= G.hi[a] ? x : G.hi[a];
      p[a] = (float)x;
    }
    float z[S::IN_G];
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      const Loc q = locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2],
                                  act ? w.status : nullptr);
      gather_fast<float, S::CG>(G.lv[l], compact<float>(q), z + l * S::CG);
    }
    float h0[GSB_HID], h1[GSB_HID];
    cdense<S::IN_G, S::oGW0, S::oGb0>(z, h0);
    relu_m(h0);
    cdense<GSB_HID, S::oGW1, S::oGb1>(h0, h1);
    relu_m(h1);
    const float f = cdot32<S::oGW2>(h1) + cws(S::oGb2);
    if (act) phi[(int64_t)ray * w.ld + slot] = (double)f;
  }
}

// ---------------------------------------------------------------------------
// taped forward: phi, grad phi (gs/renderer.py:356-358), colour (:360-365)

template <class S>
__global__ void __launch_bounds__(128) k_fwd_f(Ws<float> w, Geo G, int M, int N,
                                               const double* __restrict__ dep,
                                               const float* __restrict__ spts, int nsp) {
  const int64_t MN = (int64_t)M * N;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool act = s < MN + nsp;
  float p[3];
  int ray = -1;
  if (act && s < MN) {
    ray = (int)((uint32_t)s / (uint32_t)N);
    taped_point<float>(w.o + ray * 3, w.r + ray * 3,
                       dep[(int64_t)ray * w.ld + (int)((uint32_t)s % (uint32_t)N)], G.lo, G.hi, p);
  } else if (act) {
#pragma unroll
    for (int a = 0; a < 3; ++a) p[a] = spts[(s - MN) * 3 + a];
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) p[a] = (float)G.lo[a];
  }
  LocT<float> loc[S::NL];
  float z[S::IN_G];
#pragma unroll
  for (int l = 0; l < S::NL; ++l) {
    loc[l] = compact<float>(locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2],
                                          act ? w.status : nullptr));
    gather_fast<float, S::CG>(G.lv[l], loc[l], z + l * S::CG);
  }
  uint32_t m0, m1;
  float phi;
  {
    float h0[GSB_HID], h1[GSB_HID];
    cdense<S::IN_G, S::oGW0, S::oGb0>(z, h0);
    m0 = relu_m(h0);
    cdense<GSB_HID, S::oGW1, S::oGb1>(h0, h1);
    m1 = relu_m(h1);
    phi = cdot32<S::oGW2>(h1) + cws(S::oGb2);
  }
  // grad phi: g = W0 ((W1 (W2 . m1)) . m0), then sum_l J_l^T g_l
  float gz[S::IN_G];
  {
    float d1[GSB_HID], d0[GSB_HID];
#pragma unroll
    for (int j = 0; j < GSB_HID; ++j) d1[j] = ((m1 >> j) & 1u) ? cws(S::oGW2 + j) : 0.f;
    cdense_t<GSB_HID, S::oGW1>(d1, d0);
#pragma unroll
    for (int i = 0; i < GSB_HID; ++i) d0[i] = ((m0 >> i) & 1u) ? d0[i] : 0.f;
    cdense_t<S::IN_G, S::oGW0>(d0, gz);
  }
  float gr[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int l = 0; l < S::NL; ++l) level_dx_fast<float, S::CG>(G.lv[l], loc[l], gz + l * S::CG, gr);
  if (act) {
    w.sphi[s] = phi;
#pragma unroll
    for (int a = 0; a < 3; ++a) w.sgphi[s * 3 + a] = gr[a];
  }
  // colour: sigmoid(MLP_c([f_c, r]))  (gs/decoders.py:86-99); smoothness
  // points (ray < 0) evaluate a harmless colour and do not store it
  const int cr = ray < 0 ? 0 : ray;
  const Loc qc = locate<false>(G.col, (double)p[0], (double)p[1], (double)p[2], nullptr);
  float inp[S::IN_C];
  gather_fast<float, S::CC>(G.col, compact<float>(qc), inp);
#pragma unroll
  for (int a = 0; a < 3; ++a) inp[S::CC + a] = w.r[cr * 3 + a];
  float h0[GSB_HID], h1[GSB_HID];
  cdense<S::IN_C, S::oCW0, S::oCb0>(inp, h0);
  relu_m(h0);
  cdense<GSB_HID, S::oCW1, S::oCb1>(h0, h1);
  relu_m(h1);
  float y[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < GSB_HID; ++j) a = fmaf(h1[j], cws(S::oCW2 + j * 3 + c), a);
    y[c] = sigmoid_fast(a + cws(S::oCb2 + c));
  }
  if (act && ray >= 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) w.scol[s * 3 + c] = y[c];
  }
}

// ---------------------------------------------------------------------------
// backward, geometry (float32): scatter + MLP weight gradients

template <class S>
struct GeoRowF {
  // per-sample outer-product factors; ROW = 8 (mod 32) keeps the mma fragment
  // reads (8 rows x 4 columns per access) free of bank conflicts
  static constexpr int oA0 = 0;                 // p z + v      (IN_G)
  static constexpr int oP = S::IN_G;            // p
  static constexpr int oB0 = 20;                // delta0       (32)
  static constexpr int oA1 = oB0 + GSB_HID;     // p h0 + q0    (32)
  static constexpr int oV2 = oA1 + GSB_HID;     // p h1 + dd1 (.) m1 (32)
  static constexpr int oM = oV2 + GSB_HID;      // m1 bits
  static constexpr int ROW = 136;
  static_assert(oM < ROW && ROW % 32 == 8 && S::IN_G <= 16, "row layout");
};

template <class S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_bwd_geom_f(Ws<float> w, Geo G, int M, int N,
                                                          const double* __restrict__ dep,
                                                          const float* __restrict__ spts, int nsp,
                                                          int agg_levels) {
  using R = GeoRowF<S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sm = reinterpret_cast<float*>(smem_raw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* rows = sm + (size_t)wid * 32 * R::ROW;
  float* myrow = rows + (size_t)lane * R::ROW;
  const int64_t MN = (int64_t)M * N, NS = MN + nsp;
  // tensor-core accumulators: dW0 (16 x 32) and dW1 (32 x 32) as m16n8 tiles
  float d0[4][4], d1[2][4][4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      d0[nt][c] = 0.f;
      d1[0][nt][c] = 0.f;
      d1[1][nt][c] = 0.f;
    }
  float acc_b0 = 0.f, acc_b1 = 0.f, acc_w2 = 0.f, acc_p = 0.f;
  const float w2l = cws(S::oGW2 + lane);
  // one 32-sample batch per warp (no loop: keeps the constant-bank weight
  // loads next to their FMAs instead of hoisted into registers)
  {
    const int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * 32;
    const int64_t s = base + lane;
    const bool active = s < NS;
    float p = 0.f, u[3] = {0.f, 0.f, 0.f}, pt[3];
    if (active) {
      p = w.pbar[s];
#pragma unroll
      for (int a = 0; a < 3; ++a) u[a] = w.ubar[s * 3 + a];
      if (s < MN) {
        const int ray = (int)((uint32_t)s / (uint32_t)N);
        taped_point<float>(w.o + ray * 3, w.r + ray * 3,
                           dep[(int64_t)ray * w.ld + (int)((uint32_t)s % (uint32_t)N)], G.lo,
                           G.hi, pt);
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) pt[a] = spts[(s - MN) * 3 + a];
      }
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) pt[a] = (float)G.lo[a];
    }
    // one pass over the corners: z and v = sum_k ju_k theta_k
    LocT<float> loc[S::NL];
    float z[S::IN_G], v[S::IN_G];
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      const LevelDev& L = G.lv[l];
      loc[l] = compact<float>(locate<false>(L, (double)pt[0], (double)pt[1], (double)pt[2], nullptr));
      float wk[8], ju[8];
      corner_w_ju(loc[l], (float)L.inv_vs, u, wk, ju);
      const float* F = reinterpret_cast<const float*>(L.feat) + (int64_t)loc[l].base * S::CG;
#pragma unroll
      for (int c = 0; c < S::CG; ++c) z[l * S::CG + c] = v[l * S::CG + c] = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float row[S::CG];
        load_row<float, S::CG>(F + corner_off(L, k) * S::CG, row);
#pragma unroll
        for (int c = 0; c < S::CG; ++c) {
          z[l * S::CG + c] = fmaf(wk[k], row[c], z[l * S::CG + c]);
          v[l * S::CG + c] = fmaf(ju[k], row[c], v[l * S::CG + c]);
        }
      }
    }
    // forward (masks), p h0 -> A1, p h1 -> V2
    uint32_t m0, m1;
    {
      float h0[GSB_HID], h1[GSB_HID];
      cdense<S::IN_G, S::oGW0, S::oGb0>(z, h0);
      m0 = relu_m(h0);
      cdense<GSB_HID, S::oGW1, S::oGb1>(h0, h1);
      m1 = relu_m(h1);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) {
        h0[j] *= p;
        h1[j] *= p;
      }
      store32(myrow + R::oA1, h0);
      store32(myrow + R::oV2, h1);
    }
    // delta0 -> B0, g = dphi/dz
    float gz[S::IN_G];
    {
      float d1v[GSB_HID], d0v[GSB_HID];
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) d1v[j] = ((m1 >> j) & 1u) ? cws(S::oGW2 + j) : 0.f;
      cdense_t<GSB_HID, S::oGW1>(d1v, d0v);
#pragma unroll
      for (int i = 0; i < GSB_HID; ++i) d0v[i] = ((m0 >> i) & 1u) ? d0v[i] : 0.f;
      store32(myrow + R::oB0, d0v);
      cdense_t<S::IN_G, S::oGW0>(d0v, gz);
    }
    // grid scatter: theta_l[idx_k] += g_l (p w_k + ju_k)
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      float wk[8], ju[8], coef[8];
      corner_w_ju(loc[l], (float)G.lv[l].inv_vs, u, wk, ju);
#pragma unroll
      for (int k = 0; k < 8; ++k) coef[k] = fmaf(p, wk[k], ju[k]);
      scatter_level<float, S::CG>(G.lv[l], loc[l], gz + l * S::CG, coef, active, l < agg_levels);
    }
    // A0 = p z + v ; q0 = (v W0) (.) m0 -> A1 ; dd1 = (q0 W1) (.) m1 -> V2
    {
#pragma unroll
      for (int i = 0; i < S::IN_G; ++i) myrow[R::oA0 + i] = fmaf(p, z[i], v[i]);
      myrow[R::oP] = p;
      float q0[GSB_HID], dd[GSB_HID];
      cdense<S::IN_G, S::oGW0, -1>(v, q0);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) q0[j] = ((m0 >> j) & 1u) ? q0[j] : 0.f;
      float a[GSB_HID];
      load32(myrow + R::oA1, a);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) a[j] += q0[j];
      store32(myrow + R::oA1, a);
      cdense<GSB_HID, S::oGW1, -1>(q0, dd);
      load32(myrow + R::oV2, a);
#pragma unroll
      for (int j = 0; j < GSB_HID; ++j) a[j] += ((m1 >> j) & 1u) ? dd[j] : 0.f;
      store32(myrow + R::oV2, a);
      reinterpret_cast<uint32_t*>(myrow + R::oM)[0] = active ? m1 : 0u;
    }
    if (!active) {
#pragma unroll 1
      for (int i = 0; i < R::oM; ++i) myrow[i] = 0.f;
    }
    __syncwarp();
    // ---- outer products on the tensor cores: K = the warp's 32 samples
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int k0 = ks * 8;
      const int g = lane >> 2, t = lane & 3;
      const uint32_t mk0 = reinterpret_cast<const uint32_t*>(rows + (k0 + t) * R::ROW + R::oM)[0];
      const uint32_t mk1 = reinterpret_cast<const uint32_t*>(rows + (k0 + t + 4) * R::ROW + R::oM)[0];
      uint32_t ah[4], al[4];
      frag_a(rows, R::ROW, R::oA0, k0, 0, ah, al);      // A0^T rows 0..15
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t bh0, bh1, bl0, bl1;
        frag_b(rows, R::ROW, R::oB0, k0, nt * 8, bh0, bh1, bl0, bl1);
        mma3(d0[nt], ah, al, bh0, bh1, bl0, bl1);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        frag_a(rows, R::ROW, R::oA1, k0, mt * 16, ah, al);  // A1^T rows
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          // delta1[k][n] = m1_k(n) ? W2[n] : 0
          const int n = nt * 8 + g;
          const float w2n = __shfl_sync(0xffffffffu, w2l, n);
          const float b0v = ((mk0 >> n) & 1u) ? w2n : 0.f;
          const float b1v = ((mk1 >> n) & 1u) ? w2n : 0.f;
          uint32_t bh0, bh1, bl0, bl1;
          split_tf32(b0v, bh0, bl0);
          split_tf32(b1v, bh1, bl1);
          mma3(d1[mt][nt], ah, al, bh0, bh1, bl0, bl1);
        }
      }
    }
    // bias gradients and dW2 (column sums) on the FMA pipe; lane owns column
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      const float* rw = rows + (size_t)r * R::ROW;
      const float pr = rw[R::oP];
      const uint32_t mr = reinterpret_cast<const uint32_t*>(rw + R::oM)[0];
      acc_b0 = fmaf(pr, rw[R::oB0 + lane], acc_b0);                 // db0 = sum p delta0
      acc_b1 = fmaf(pr, ((mr >> lane) & 1u) ? w2l : 0.f, acc_b1);   // db1 = sum p delta1
      acc_w2 += rw[R::oV2 + lane];                                   // dW2 = sum V2
      acc_p += pr;                                                   // db2 = sum p
    }
    __syncwarp();
  }
  // CTA reduction -> partial slot blockIdx.x (geometry block of the MLP)
  __syncthreads();
  constexpr int NGP = S::NG;
  float* red = sm;  // [WARPS][NGP]
  {
    float* mine = red + (size_t)wid * NGP;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) frag_d_store(d0[nt], mine + S::oGW0, 0, nt * 8, S::IN_G);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) frag_d_store(d1[mt][nt], mine + S::oGW1, mt * 16, nt * 8, GSB_HID);
    mine[S::oGb0 + lane] = acc_b0;
    mine[S::oGb1 + lane] = acc_b1;
    mine[S::oGW2 + lane] = acc_w2;
    if (lane == 0) mine[S::oGb2] = acc_p;
  }
  __syncthreads();
  float* out = w.mlp_part + (size_t)blockIdx.x * S::NMLP;
  for (int t = threadIdx.x; t < NGP; t += WARPS * 32) {
    float a = 0.f;
#pragma unroll
    for (int k = 0; k < WARPS; ++k) a += red[(size_t)k * NGP + t];
    out[t] = a;
  }
}

// ---------------------------------------------------------------------------
// backward, colour (float32)

template <class S>
struct ColRowF {
  static constexpr int oA0 = 0;               // [inp (IN_C), 1]
  static constexpr int oB0 = 16;              // a0_bar (32)
  static constexpr int oA1 = oB0 + GSB_HID;   // h0 (32)
  static constexpr int oB1 = oA1 + GSB_HID;   // a1_bar (32)
  static constexpr int oH1 = oB1 + GSB_HID;   // h1 (32)
  static constexpr int oY = oH1 + GSB_HID;    // y_bar (3), zero-padded to 8
  static constexpr int ROW = 168;
  static_assert(oY + 8 <= ROW && ROW % 32 == 8 && S::IN_C + 1 <= 16, "row layout");
};

template <class S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_bwd_color_f(Ws<float> w, Geo G, int M, int N,
                                                           const double* __restrict__ dep) {
  using R = ColRowF<S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sm = reinterpret_cast<float*>(smem_raw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* rows = sm + (size_t)wid * 32 * R::ROW;
  float* myrow = rows + (size_t)lane * R::ROW;
  const int64_t NS = (int64_t)M * N;
  float e0[4][4], e1[2][4][4], e2[2][4];  // dW0c (16 x 32), dW1c (32 x 32), dW2c (32 x 8)
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      e0[nt][c] = 0.f;
      e1[0][nt][c] = 0.f;
      e1[1][nt][c] = 0.f;
    }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int c = 0; c < 4; ++c) e2[mt][c] = 0.f;
  float acc_b1 = 0.f, acc_b2 = 0.f;
  {
    const int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * 32;
    const int64_t s = base + lane;
    const bool active = s < NS;
    const int ray = active ? (int)((uint32_t)s / (uint32_t)N) : 0;
    float pt[3];
    taped_point<float>(w.o + ray * 3, w.r + ray * 3,
                       active ? dep[(int64_t)ray * w.ld + (int)((uint32_t)s % (uint32_t)N)] : 0.0,
                       G.lo, G.hi, pt);
    const LocT<float> q =
        compact<float>(locate<false>(G.col, (double)pt[0], (double)pt[1], (double)pt[2], nullptr));
    float inp[S::IN_C];
    gather_fast<float, S::CC>(G.col, q, inp);
#pragma unroll
    for (int a = 0; a < 3; ++a) inp[S::CC + a] = w.r[ray * 3 + a];
#pragma unroll
    for (int i = 0; i < S::IN_C; ++i) myrow[R::oA0 + i] = inp[i];
    myrow[R::oA0 + S::IN_C] = 1.f;
#pragma unroll
    for (int i = S::IN_C + 1; i < 16; ++i) myrow[R::oA0 + i] = 0.f;
    uint32_t m0, m1;
    float yb[3];
    {
      float h0[GSB_HID], h1[GSB_HID];
      cdense<S::IN_C, S::oCW0, S::oCb0>(inp, h0);
      m0 = relu_m(h0);
      store32(myrow + R::oA1, h0);
      cdense<GSB_HID, S::oCW1, S::oCb1>(h0, h1);
      m1 = relu_m(h1);
      store32(myrow + R::oH1, h1);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < GSB_HID; ++j) a = fmaf(h1[j], cws(S::oCW2 + j * 3 + c), a);
        const float cc = sigmoid_fast(a + cws(S::oCb2 + c));
        yb[c] = active ? w.cbar[s * 3 + c] * (cc * (1.f - cc)) : 0.f;
      }
    }
    sts4(myrow + R::oY, yb[0], yb[1], yb[2], 0.f);
    sts4(myrow + R::oY + 4, 0.f, 0.f, 0.f, 0.f);
    float a1b[GSB_HID], a0b[GSB_HID];
#pragma unroll
    for (int j = 0; j < GSB_HID; ++j) {
      float a = 0.f;
#pragma unroll
      for (int c = 0; c < 3; ++c) a = fmaf(cws(S::oCW2 + j * 3 + c), yb[c], a);
      a1b[j] = ((m1 >> j) & 1u) ? a : 0.f;
    }
    store32(myrow + R::oB1, a1b);
    cdense_t<GSB_HID, S::oCW1>(a1b, a0b);
#pragma unroll
    for (int i = 0; i < GSB_HID; ++i) a0b[i] = ((m0 >> i) & 1u) ? a0b[i] : 0.f;
    store32(myrow + R::oB0, a0b);
    float fb[S::CC];
    cdense_t<S::CC, S::oCW0>(a0b, fb);
    {  // colour grid scatter: theta_c[idx_k] += w_k f_bar (warp-segmented)
      float wk[8];
      corner_w(q, wk);
      scatter_level<float, S::CC>(G.col, q, fb, wk, active, false);
    }
    if (!active) {
#pragma unroll 1
      for (int i = 0; i < R::ROW; ++i) myrow[i] = 0.f;
    }
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int k0 = ks * 8;
      uint32_t ah[4], al[4];
      frag_a(rows, R::ROW, R::oA0, k0, 0, ah, al);      // [inp, 1]^T
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t bh0, bh1, bl0, bl1;
        frag_b(rows, R::ROW, R::oB0, k0, nt * 8, bh0, bh1, bl0, bl1);
        mma3(e0[nt], ah, al, bh0, bh1, bl0, bl1);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        frag_a(rows, R::ROW, R::oA1, k0, mt * 16, ah, al);  // h0^T
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          uint32_t bh0, bh1, bl0, bl1;
          frag_b(rows, R::ROW, R::oB1, k0, nt * 8, bh0, bh1, bl0, bl1);
          mma3(e1[mt][nt], ah, al, bh0, bh1, bl0, bl1);
        }
        frag_a(rows, R::ROW, R::oH1, k0, mt * 16, ah, al);  // h1^T x y_bar
        uint32_t bh0, bh1, bl0, bl1;
        frag_b(rows, R::ROW, R::oY, k0, 0, bh0, bh1, bl0, bl1);
        mma3(e2[mt], ah, al, bh0, bh1, bl0, bl1);
      }
    }
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      const float* rw = rows + (size_t)r * R::ROW;
      acc_b1 += rw[R::oB1 + lane];                           // db1 = sum a1_bar
      acc_b2 += lane < 3 ? rw[R::oY + lane] : 0.f;            // db2 = sum y_bar
    }
    __syncwarp();
  }
  __syncthreads();
  constexpr int NCP = S::NMLP - S::NG;
  float* red = sm;
  {
    float* mine = red + (size_t)wid * NCP;
    const int o = S::NG;
    if (lane < S::oCW0 - S::NG) mine[lane] = 0.f;  // alignment padding
    // dW0c rows 0..IN_C-1, db0c = row IN_C (the ones column)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) frag_d_store(e0[nt], mine + (S::oCW0 - o), 0, nt * 8, S::IN_C + 1);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) frag_d_store(e1[mt][nt], mine + (S::oCW1 - o), mt * 16, nt * 8, GSB_HID);
    mine[S::oCb1 - o + lane] = acc_b1;
    if (lane < 3) mine[S::oCb2 - o + lane] = acc_b2;
  }
  __syncwarp();
  {
    // dW2c (32 x 3): fragments hold [32 x 8]; keep columns 0..2
    float* mine = red + (size_t)wid * NCP;
    const int o = S::NG;
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r0 = mt * 16 + g, r1 = r0 + 8, c = 2 * t;
      if (c < 3) {
        mine[S::oCW2 - o + r0 * 3 + c] = e2[mt][0];
        mine[S::oCW2 - o + r1 * 3 + c] = e2[mt][2];
      }
      if (c + 1 < 3) {
        mine[S::oCW2 - o + r0 * 3 + c + 1] = e2[mt][1];
        mine[S::oCW2 - o + r1 * 3 + c + 1] = e2[mt][3];
      }
    }
  }
  __syncthreads();
  float* out = w.mlp_part + (size_t)blockIdx.x * S::NMLP + S::NG;
  for (int t = threadIdx.x; t < NCP; t += WARPS * 32) {
    float a = 0.f;
#pragma unroll
    for (int k = 0; k < WARPS; ++k) a += red[(size_t)k * NCP + t];
    out[t] = a;
  }
}

}  // namespace gsb
