// gsb_tc.cuh -- float32 taped pass with the decoders on the tensor cores.
//
// Work split: a warp owns 32 samples.  Per-sample
// scalar work -- point, grid location, trilinear gather, grad-phi assembly,
// grid scatter -- runs lane-per-sample.  The MLP layers run as chains of
// mma.sync m16n8k8 TF32 in 3xTF32 split precision (hi*hi + hi*lo + lo*hi,
// ~fp32 accuracy), activations resident in registers as accumulator ("D")
// fragments: lane (g = lane/4, t = lane%4) of m-tile mt holds samples
// 16mt+g (r = 0,1) and 16mt+g+8 (r = 2,3) at features 8nn+2t+(r&1).
//
// Chaining without shuffles: the A operand of k-step kk wants features
// {slot t, slot t+4} of block kk; we *define* slot t <-> feature 2t and slot
// t+4 <-> feature 2t+1, so the D fragment of feature block kk is the A
// fragment {d0, d2, d1, d3}, and the weight (B) fragments are built with the
// same permutation of their contraction index once per step (k_wfrag), split
// into tf32 hi/lo, and staged in shared memory per CTA.
//
// tools/mb_layers.cu measured this form at 84-101% of the fp32 FFMA peak
// (effective) already at 1-2 CTAs/SM with ~10x fewer issued instructions
// and ~10x less code than the unrolled-FFMA kernels (round-1 history), whose
// 100-190 KB of SASS thrashed the instruction cache.
#pragma once

#include "gsb_mma.cuh"

namespace gsb {
namespace tc {

constexpr int kFragMax = 128;  // B fragments per model (446 shape: 100)
constexpr int kVecBase = kFragMax * 32;  // uint4 index of the vector block in the buffer

// vector block (floats; segments padded to 8): geometry b0, b1, W2, b2 then
// colour b0c, b1c, b2c
struct GVec {
  static constexpr int b0 = 0, b1 = 32, w2 = 64, b2 = 96, N = 104;
};
struct CVec {
  static constexpr int b0 = 0, b1 = 32, b2 = 64, w2 = 72, N = 168;  // w2: W2c (32 x 3)
};
// tcgen05 operand block (gsb_t5.cuh): geometry W0 / W1 as B operands (out x in,
// canonical K-major, no swizzle), tf32 hi and lo tiles; float offsets
struct UmmaW {
  // geometry W0^T, W1^T (forward), W1, W0 (delta chain: B[n][k] = W[n][k]),
  // colour W0c^T, W1c^T; hi then lo tile each
  static constexpr int W0H = 0, W0L = 512, W1H = 1024, W1L = 2048;
  static constexpr int W1NH = 3072, W1NL = 4096, W0NH = 5120, W0NL = 5632;
  static constexpr int C0H = 6144, C0L = 6656, C1H = 7168, C1L = 8192;
  // colour backward chain: W1c (a1b -> a0b), W0c rows (a0b -> [f_bar, r_bar])
  static constexpr int C1NH = 9216, C1NL = 10240, C0NH = 11264, C0NL = 11776;
  static constexpr int N = 12288;
  static constexpr int NFWD = 9216;  // geometry + colour forward tiles (k_fwd_t5)
  static constexpr int kTiles = 16;
};
constexpr int kUmmaBaseU4 = kVecBase + (GVec::N + CVec::N) / 4;
constexpr int kFragBufU4 = kUmmaBaseU4 + UmmaW::N / 4;

// element (r, k) of an [R x K] fp32 operand tile: core matrices of 8 rows x
// 4 k (16-byte rows, 128 B), K-adjacent core matrices 128 B apart (LBO), 8-row
// groups K/4 core matrices apart (SBO = 32 K bytes)
__host__ __device__ __forceinline__ int kmaj(int r, int k, int K) {
  return (r >> 3) * (K / 4) * 32 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

// ---- one-shot TMA bulk staging (cp.async.bulk + mbarrier transaction count)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// thread 0: stage fragments [first, first + count) to sfr and `nvec` floats of
// the vector block (from float offset voff) to svec; all threads later mbar_wait
__device__ __forceinline__ void stage_async(uint64_t* bar, uint4* sfr, const uint4* gbuf, int first,
                                            int count, float* svec, int voff, int nvec) {
  if (threadIdx.x == 0) {
    const uint32_t fb = (uint32_t)count * 32u * 16u, vb = (uint32_t)nvec * 4u;
    mbar_expect(bar, fb + vb);
    bulk_g2s(sfr, gbuf + first * 32, fb, bar);
    bulk_g2s(svec, reinterpret_cast<const float*>(gbuf + kVecBase) + voff, vb, bar);
  }
}

// B-fragment ids (each = 32 lanes x uint4 {hi0, hi1, lo0, lo1})
template <class S>
struct Fr {
  static constexpr int KG = (S::IN_G + 7) / 8;  // geometry input k-steps
  static constexpr int KC = (S::IN_C + 7) / 8;  // colour input k-steps
  static constexpr int NCC = (S::CC + 7) / 8;   // colour-feature gradient n-tiles
  static constexpr int G_W0 = 0;                // z W0        KG x 4
  static constexpr int G_W1 = G_W0 + KG * 4;    // h0 W1       4 x 4
  static constexpr int G_W1T = G_W1 + 16;       // d1 W1^T     4 x 4
  static constexpr int G_W0T = G_W1T + 16;      // d0 W0^T     4 x KG
  static constexpr int NGEO = G_W0T + 4 * KG;
  static constexpr int C_W0 = NGEO;             // inp W0c     KC x 4
  static constexpr int C_W1 = C_W0 + KC * 4;    // h0c W1c     4 x 4
  static constexpr int C_W2 = C_W1 + 16;        // h1c W2c     4 x 1
  static constexpr int C_W2T = C_W2 + 4;        // ybar W2c^T  1 x 4
  static constexpr int C_W1T = C_W2T + 4;       // a1b W1c^T   4 x 4
  static constexpr int C_W0T = C_W1T + 16;      // a0b W0c^T   4 x NCC
  static constexpr int NALL = C_W0T + 4 * NCC;
  static_assert(NALL <= kFragMax, "fragment buffer");
};

// One block per fragment id, one thread per lane.  Contraction index k of
// fragment (kk, nn): b0 <-> k = 8kk+2t, b1 <-> k = 8kk+2t+1; output n = 8nn+g.
template <class S>
__device__ __forceinline__ void wfrag_block(const float* __restrict__ mlp, uint4* __restrict__ out, int id) {
  using F = Fr<S>;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (id > F::NALL) {  // tcgen05 B tiles (UmmaW), hi / lo per matrix
    const int tile = id - F::NALL - 1, lo = tile & 1, mat = tile >> 1;
    // mat: 0 W0^T, 1 W1^T, 2 W1, 3 W0, 4 W0c^T, 5 W1c^T, 6 W1c, 7 W0c.  B[n][k], K contiguous
    int oW, K, Nn, rows, off;
    bool tr;  // true: B[n][k] = W[k][n] (W stored (in, out) row-major, 32 columns)
    switch (mat) {
      case 0: oW = S::oGW0; K = 8 * F::KG; Nn = GSB_HID; rows = S::IN_G; tr = true; off = lo ? UmmaW::W0L : UmmaW::W0H; break;
      case 1: oW = S::oGW1; K = GSB_HID; Nn = GSB_HID; rows = GSB_HID; tr = true; off = lo ? UmmaW::W1L : UmmaW::W1H; break;
      case 2: oW = S::oGW1; K = GSB_HID; Nn = GSB_HID; rows = GSB_HID; tr = false; off = lo ? UmmaW::W1NL : UmmaW::W1NH; break;
      case 3: oW = S::oGW0; K = GSB_HID; Nn = 16; rows = S::IN_G; tr = false; off = lo ? UmmaW::W0NL : UmmaW::W0NH; break;
      case 4: oW = S::oCW0; K = 8 * F::KC; Nn = GSB_HID; rows = S::IN_C; tr = true; off = lo ? UmmaW::C0L : UmmaW::C0H; break;
      case 5: oW = S::oCW1; K = GSB_HID; Nn = GSB_HID; rows = GSB_HID; tr = true; off = lo ? UmmaW::C1L : UmmaW::C1H; break;
      case 6: oW = S::oCW1; K = GSB_HID; Nn = GSB_HID; rows = GSB_HID; tr = false; off = lo ? UmmaW::C1NL : UmmaW::C1NH; break;
      default: oW = S::oCW0; K = GSB_HID; Nn = 16; rows = S::IN_C; tr = false; off = lo ? UmmaW::C0NL : UmmaW::C0NH; break;
    }
    float* o = reinterpret_cast<float*>(out + kUmmaBaseU4) + off;
    for (int i = threadIdx.x; i < Nn * K; i += blockDim.x) {
      const int n = i / K, k = i % K;
      float v = 0.f;
      if (tr) {
        if (k < rows) v = mlp[oW + k * GSB_HID + n];
      } else {
        if (n < rows) v = mlp[oW + n * GSB_HID + k];  // W rows are the outputs here
      }
      uint32_t h, l;
      split_tf32(v, h, l);
      o[kmaj(n, k, K)] = __uint_as_float(lo ? l : h);
    }
    return;
  }
  if (threadIdx.x >= 32) return;  // fragments and vectors: one warp per block
  if (id == F::NALL) {  // bias / W2 vectors: geometry block then colour block
    float* v = reinterpret_cast<float*>(out + kVecBase);
    for (int i = lane; i < GVec::N + CVec::N; i += 32) {
      float x = 0.f;
      if (i < GVec::N) {
        if (i < 32) x = mlp[S::oGb0 + i];
        else if (i < 64) x = mlp[S::oGb1 + i - 32];
        else if (i < 96) x = mlp[S::oGW2 + i - 64];
        else if (i == 96) x = mlp[S::oGb2];
      } else {
        const int j = i - GVec::N;
        if (j < 32) x = mlp[S::oCb0 + j];
        else if (j < 64) x = mlp[S::oCb1 + j - 32];
        else if (j < 67) x = mlp[S::oCb2 + j - 64];
        else if (j >= CVec::w2 && j < CVec::w2 + 96) x = mlp[S::oCW2 + j - CVec::w2];
      }
      v[i] = x;
    }
    return;
  }
  int oW, rows, cols, NN, li, lim;
  bool tr;
  if (id < F::G_W1) {
    oW = S::oGW0; rows = S::IN_G; cols = GSB_HID; tr = false; NN = 4; li = id - F::G_W0; lim = 0;
  } else if (id < F::G_W1T) {
    oW = S::oGW1; rows = GSB_HID; cols = GSB_HID; tr = false; NN = 4; li = id - F::G_W1; lim = 0;
  } else if (id < F::G_W0T) {
    oW = S::oGW1; rows = GSB_HID; cols = GSB_HID; tr = true; NN = 4; li = id - F::G_W1T; lim = GSB_HID;
  } else if (id < F::C_W0) {
    oW = S::oGW0; rows = S::IN_G; cols = GSB_HID; tr = true; NN = F::KG; li = id - F::G_W0T; lim = S::IN_G;
  } else if (id < F::C_W1) {
    oW = S::oCW0; rows = S::IN_C; cols = GSB_HID; tr = false; NN = 4; li = id - F::C_W0; lim = 0;
  } else if (id < F::C_W2) {
    oW = S::oCW1; rows = GSB_HID; cols = GSB_HID; tr = false; NN = 4; li = id - F::C_W1; lim = 0;
  } else if (id < F::C_W2T) {
    oW = S::oCW2; rows = GSB_HID; cols = 3; tr = false; NN = 1; li = id - F::C_W2; lim = 0;
  } else if (id < F::C_W1T) {
    oW = S::oCW2; rows = GSB_HID; cols = 3; tr = true; NN = 4; li = id - F::C_W2T; lim = GSB_HID;
  } else if (id < F::C_W0T) {
    oW = S::oCW1; rows = GSB_HID; cols = GSB_HID; tr = true; NN = 4; li = id - F::C_W1T; lim = GSB_HID;
  } else {
    oW = S::oCW0; rows = S::IN_C; cols = GSB_HID; tr = true; NN = F::NCC; li = id - F::C_W0T; lim = S::CC;
  }
  const int kk = li / NN, nn = li % NN;
  const int n = 8 * nn + g;
  float b[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int k = 8 * kk + 2 * t + h;
    float v = 0.f;
    if (!tr) {
      if (k < rows && n < cols) v = mlp[oW + k * cols + n];  // W[k][n]
    } else {
      if (n < lim && k < cols) v = mlp[oW + n * cols + k];   // W^T[k][n] = W[n][k]
    }
    b[h] = v;
  }
  uint32_t h0, l0, h1, l1;
  split_tf32(b[0], h0, l0);
  split_tf32(b[1], h1, l1);
  out[id * 32 + lane] = make_uint4(h0, h1, l0, l1);
}
template <class S>
__global__ void __launch_bounds__(128) k_wfrag(const float* __restrict__ mlp, uint4* __restrict__ out) {
  wfrag_block<S>(mlp, out, blockIdx.x);
}
// blocks of k_wfrag
template <class S>
constexpr int wfrag_blocks() { return Fr<S>::NALL + 1 + UmmaW::kTiles; }

// ---------------------------------------------------------------------------
// fragment helpers

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// value barrier: the compiler cannot see through it, so work that depends on
// it is recomputed instead of kept live (and spilled) across the MLP phase
__device__ __forceinline__ float opaque(float x) {
  float y;
  asm volatile("mov.b32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <typename T>
__device__ __forceinline__ LocT<T> opaque(const LocT<T>& q) {
  LocT<T> r;
  r.base = __float_as_int(opaque(__int_as_float(q.base)));
  r.fx = opaque(q.fx);
  r.fy = opaque(q.fy);
  r.fz = opaque(q.fz);
  return r;
}

// A operand from the D fragment of feature block kk
__device__ __forceinline__ void a_from_d(const float (&x)[4], uint32_t (&ah)[4], uint32_t (&al)[4]) {
  split_fast(x[0], ah[0], al[0]);
  split_fast(x[2], ah[1], al[1]);
  split_fast(x[1], ah[2], al[2]);
  split_fast(x[3], ah[3], al[3]);
}

// A operand from sample-major shared rows (features at off + 8kk + {2t, 2t+1})
template <int ROW>
__device__ __forceinline__ void a_from_rows(const float* rows, int off, int m0, int kk,
                                            uint32_t (&ah)[4], uint32_t (&al)[4]) {
  const int lane = lane_id(), g = lane >> 2, t = lane & 3;
  const float2 u = *reinterpret_cast<const float2*>(rows + (m0 + g) * ROW + off + 8 * kk + 2 * t);
  const float2 v = *reinterpret_cast<const float2*>(rows + (m0 + g + 8) * ROW + off + 8 * kk + 2 * t);
  split_fast(u.x, ah[0], al[0]);
  split_fast(v.x, ah[1], al[1]);
  split_fast(u.y, ah[2], al[2]);
  split_fast(v.y, ah[3], al[3]);
}

// Y[mt][nn] += A(mt, kk) B(kk, nn); B fragments at fr[(kk*NN + nn)*32 + lane]
template <int MT, int KK, int NN, class AF>
__device__ __forceinline__ void mma_layer(const AF& afrag, const uint4* fr, float (&Y)[MT][NN][4]) {
  const int lane = lane_id();
#pragma unroll
  for (int kk = 0; kk < KK; ++kk) {
    uint32_t ah[MT][4], al[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) afrag(mt, kk, ah[mt], al[mt]);
    uint4 b[NN];
#pragma unroll
    for (int nn = 0; nn < NN; ++nn) b[nn] = fr[(kk * NN + nn) * 32 + lane];
    // three passes (lo*hi, hi*lo, hi*hi), each sweeping the MT x NN independent
    // accumulators, so consecutive MMAs never wait on each other
#pragma unroll
    for (int nn = 0; nn < NN; ++nn)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) mma_tf32(Y[mt][nn], al[mt], b[nn].x, b[nn].y);
#pragma unroll
    for (int nn = 0; nn < NN; ++nn)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) mma_tf32(Y[mt][nn], ah[mt], b[nn].z, b[nn].w);
#pragma unroll
    for (int nn = 0; nn < NN; ++nn)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) mma_tf32(Y[mt][nn], ah[mt], b[nn].x, b[nn].y);
  }
}

// D[mt][nt] += A[mt] B[nt] in 3xTF32, pass-interleaved over the MT x NT tiles
template <int MT, int NT>
__device__ __forceinline__ void mma3_sweep(float (&D)[MT][NT][4], const uint32_t (&ah)[MT][4],
                                           const uint32_t (&al)[MT][4], const uint32_t (&bh0)[NT],
                                           const uint32_t (&bh1)[NT], const uint32_t (&bl0)[NT],
                                           const uint32_t (&bl1)[NT]) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) mma_tf32(D[mt][nt], al[mt], bh0[nt], bh1[nt]);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) mma_tf32(D[mt][nt], ah[mt], bl0[nt], bl1[nt]);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) mma_tf32(D[mt][nt], ah[mt], bh0[nt], bh1[nt]);
}

template <int MT, int NN>
__device__ __forceinline__ void fill_cols(float (&Y)[MT][NN][4], const float* v) {
  const int t = lane_id() & 3;
#pragma unroll
  for (int nn = 0; nn < NN; ++nn) {
    const float2 b = *reinterpret_cast<const float2*>(v + 8 * nn + 2 * t);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      Y[mt][nn][0] = b.x;
      Y[mt][nn][1] = b.y;
      Y[mt][nn][2] = b.x;
      Y[mt][nn][3] = b.y;
    }
  }
}

template <int MT, int NN>
__device__ __forceinline__ void zero_d(float (&Y)[MT][NN][4]) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nn = 0; nn < NN; ++nn)
#pragma unroll
      for (int r = 0; r < 4; ++r) Y[mt][nn][r] = 0.f;
}

// ReLU in place (relu_m semantics: pos ? h : 0), returns the mask bits
// (bit mt*16 + nn*4 + r)
template <int MT>
__device__ __forceinline__ uint32_t relu_d(float (&Y)[MT][4][4]) {
  uint32_t m = 0u;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const bool pos = Y[mt][nn][r] > 0.f;
        Y[mt][nn][r] = pos ? Y[mt][nn][r] : 0.f;
        m |= (uint32_t)pos << (mt * 16 + nn * 4 + r);
      }
  return m;
}

template <int MT>
__device__ __forceinline__ void mask_d(float (&Y)[MT][4][4], uint32_t m) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int r = 0; r < 4; ++r)
        Y[mt][nn][r] = ((m >> (mt * 16 + nn * 4 + r)) & 1u) ? Y[mt][nn][r] : 0.f;
}

// delta1 = m1 ? W2[col] : 0 (D form)
template <int MT>
__device__ __forceinline__ void delta1_d(float (&Y)[MT][4][4], uint32_t m1, const float* w2) {
  const int t = lane_id() & 3;
#pragma unroll
  for (int nn = 0; nn < 4; ++nn) {
    const float2 w = *reinterpret_cast<const float2*>(w2 + 8 * nn + 2 * t);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int r = 0; r < 4; ++r)
        Y[mt][nn][r] = ((m1 >> (mt * 16 + nn * 4 + r)) & 1u) ? ((r & 1) ? w.y : w.x) : 0.f;
  }
}

// D fragments -> sample-major rows (features at off + 8nn + {2t, 2t+1})
template <int ROW, int MT, int NN>
__device__ __forceinline__ void store_d(const float (&Y)[MT][NN][4], float* rows, int off) {
  const int lane = lane_id(), g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nn = 0; nn < NN; ++nn) {
      *reinterpret_cast<float2*>(rows + (16 * mt + g) * ROW + off + 8 * nn + 2 * t) =
          make_float2(Y[mt][nn][0], Y[mt][nn][1]);
      *reinterpret_cast<float2*>(rows + (16 * mt + g + 8) * ROW + off + 8 * nn + 2 * t) =
          make_float2(Y[mt][nn][2], Y[mt][nn][3]);
    }
}

// sample-major rows -> D fragments (inverse of store_d)
template <int ROW, int MT, int NN>
__device__ __forceinline__ void load_d(float (&Y)[MT][NN][4], const float* rows, int off) {
  const int lane = lane_id(), g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nn = 0; nn < NN; ++nn) {
      const float2 a = *reinterpret_cast<const float2*>(rows + (16 * mt + g) * ROW + off + 8 * nn + 2 * t);
      const float2 b = *reinterpret_cast<const float2*>(rows + (16 * mt + g + 8) * ROW + off + 8 * nn + 2 * t);
      Y[mt][nn][0] = a.x;
      Y[mt][nn][1] = a.y;
      Y[mt][nn][2] = b.x;
      Y[mt][nn][3] = b.y;
    }
}

// per-sample 32-bit feature mask of a D-form layer for rows g / g+8 of m-tile mt
// (OR over the quad); valid in every lane of the quad
__device__ __forceinline__ uint32_t row_mask(uint32_t m, int mt, int half) {
  const int t = lane_id() & 3;
  uint32_t r = 0u;
#pragma unroll
  for (int nn = 0; nn < 4; ++nn)
#pragma unroll
    for (int c = 0; c < 2; ++c)
      r |= ((m >> (mt * 16 + nn * 4 + 2 * half + c)) & 1u) << (8 * nn + 2 * t + c);
  r |= __shfl_xor_sync(0xffffffffu, r, 1);
  r |= __shfl_xor_sync(0xffffffffu, r, 2);
  return r;
}

// Sum v over the 8 lanes that share t (lane bits 2..4) as a butterfly
// reduce-scatter: N/2 + N/4 + N/8 shuffles instead of 3N for an all-reduce.
// The lane keeps chunk q = 4 b4 + 2 b3 + b2 (its lane bits) of N/8 values.
template <int N>
__device__ __forceinline__ void reduce_scatter_g(const float (&v)[N], float (&out)[N / 8]) {
  static_assert(N % 8 == 0, "N");
  const int lane = lane_id();
  const bool h4 = (lane >> 4) & 1, h3 = (lane >> 3) & 1, h2 = (lane >> 2) & 1;
  float a[N / 2], b[N / 4];
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const float send = h4 ? v[i] : v[N / 2 + i];
    a[i] = (h4 ? v[N / 2 + i] : v[i]) + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < N / 4; ++i) {
    const float send = h3 ? a[i] : a[N / 4 + i];
    b[i] = (h3 ? a[N / 4 + i] : a[i]) + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int i = 0; i < N / 8; ++i) {
    const float send = h2 ? b[i] : b[N / 8 + i];
    out[i] = (h2 ? b[N / 8 + i] : b[i]) + __shfl_xor_sync(0xffffffffu, send, 4);
  }
}
__device__ __forceinline__ int rs_chunk() {
  const int lane = lane_id();
  return 4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1);
}

// phi = h1 . W2 + b2 for rows g, g+8 of each m-tile (quad reduction)
template <int MT>
__device__ __forceinline__ void phi_d(const float (&h1)[MT][4][4], const float* w2, float b2,
                                      float (&phi)[MT][2]) {
  const int t = lane_id() & 3;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) {
      const float2 w = *reinterpret_cast<const float2*>(w2 + 8 * nn + 2 * t);
      s0 = fmaf(h1[mt][nn][0], w.x, s0);
      s0 = fmaf(h1[mt][nn][1], w.y, s0);
      s1 = fmaf(h1[mt][nn][2], w.x, s1);
      s1 = fmaf(h1[mt][nn][3], w.y, s1);
    }
    s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    phi[mt][0] = s0 + b2;
    phi[mt][1] = s1 + b2;
  }
}

// ---------------------------------------------------------------------------
// no-grad SDF at listed samples (importance passes, gs/renderer.py:330-340)

template <class S, int WARPS>
struct SdfTc {
  using F = Fr<S>;
  static constexpr int ROW = 24;  // z (8 KG) ; phi at 16
  static constexpr int NFR = F::G_W1T;  // G_W0, G_W1
  static constexpr size_t smem() {
    return (size_t)NFR * 32 * 16 + GVec::N * 4 + (size_t)WARPS * 32 * ROW * 4;
  }
  static_assert(8 * F::KG <= 16, "row layout");
};

template <class S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_sdf_eval_tc(Ws<float> w, Geo G, int M, int Nc,
                                                            const float* __restrict__ mlp,
                                                            const double* __restrict__ dep,
                                                            double* __restrict__ phi,
                                                            const int32_t* __restrict__ list,
                                                            const int32_t* __restrict__ list_count) {
  using K = SdfTc<S, WARPS>;
  using F = Fr<S>;
  constexpr int ROW = K::ROW;
  extern __shared__ uint4 smem4[];
  uint4* sfr = smem4;
  float* svec = reinterpret_cast<float*>(sfr + K::NFR * 32);
  float* rows_all = svec + GVec::N;
  const int lane = lane_id(), wid = threadIdx.x >> 5, g = lane >> 2;
  const int64_t total = list ? (int64_t)(*list_count) : (int64_t)M * Nc;
  if ((int64_t)blockIdx.x * WARPS * 32 >= total) return;  // block-uniform
  __shared__ __align__(8) uint64_t s_bar;
  if (threadIdx.x == 0) mbar_init(&s_bar);
  __syncthreads();
  stage_async(&s_bar, sfr, w.wfrag, F::G_W0, K::NFR, svec, 0, GVec::N);
  float* rows = rows_all + wid * 32 * ROW;
  const int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * 32;
  if (base >= total) return;  // warp-uniform; no block barrier below
  const int64_t s = base + lane;
  const bool act = s < total;
  int ray = 0, slot = 0;
  if (act) {
    if (list) {
      const int32_t e = list[s];
      ray = e / GSB_KMAX;
      slot = e % GSB_KMAX;
    } else {
      ray = (int)((uint32_t)s / (uint32_t)Nc);
      slot = (int)((uint32_t)s % (uint32_t)Nc);
    }
  }
  {
    const double d = act ? dep[(int64_t)ray * w.ld + slot] : 0.0;
    float p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double x = w.od[ray * 3 + a] + d * w.rd[ray * 3 + a];
      x = x >= G.lo[a] ? x : G.lo[a];
      x = x <= G.hi[a] ? x : G.hi[a];
      p[a] = (float)x;
    }
    float z[8 * F::KG];
#pragma unroll
    for (int i = S::IN_G; i < 8 * F::KG; ++i) z[i] = 0.f;
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      const Loc q = locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2],
                                  (act && l == S::NL - 1) ? w.status : nullptr);  // as t5::k_sdf_eval_t5
      gather_fast<float, S::CG>(G.lv[l], compact<float>(q), z + l * S::CG);
    }
    float* my = rows + lane * ROW;
#pragma unroll
    for (int i = 0; i < 8 * F::KG; i += 2) *reinterpret_cast<float2*>(my + i) = make_float2(z[i], z[i + 1]);
  }
  mbar_wait(&s_bar, 0);
  __syncwarp();
  float h0[2][4][4], h1[2][4][4];
  fill_cols(h0, svec + GVec::b0);
  mma_layer<2, F::KG, 4>(
      [&](int mt, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_rows<ROW>(rows, 0, 16 * mt, kk, ah, al); },
      sfr + (F::G_W0 - F::G_W0) * 32, h0);
  relu_d(h0);
  fill_cols(h1, svec + GVec::b1);
  mma_layer<2, 4, 4>([&](int mt, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(h0[mt][kk], ah, al); },
                     sfr + (F::G_W1 - F::G_W0) * 32, h1);
  relu_d(h1);
  float ph[2][2];
  phi_d(h1, svec + GVec::w2, svec[GVec::b2], ph);
  __syncwarp();
  if ((lane & 3) == 0) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      rows[(16 * mt + g) * ROW + 16] = ph[mt][0];
      rows[(16 * mt + g + 8) * ROW + 16] = ph[mt][1];
    }
  }
  __syncwarp();
  if (act) phi[(int64_t)ray * w.ld + slot] = (double)rows[lane * ROW + 16];
}

// ---------------------------------------------------------------------------
// taped forward: phi, grad phi (gs/renderer.py:356-358), colour (:360-365)

template <class S, int WARPS>
struct FwdTc {
  using F = Fr<S>;
  static constexpr int ROW = 40;
  static constexpr int oZ = 0;    // z, later dphi/dz (16)
  static constexpr int oC = 16;   // colour input [f_c, r] (16), later phi at oC
  static constexpr int oY = 32;   // colour (8 columns)
  static constexpr int NFR = F::C_W2T;  // geometry (all) + colour forward
  static constexpr int VEC = GVec::N + CVec::N;
  static constexpr size_t smem() {
    return (size_t)NFR * 32 * 16 + VEC * 4 + (size_t)WARPS * 32 * ROW * 4;
  }
  static_assert(8 * F::KG <= 16 && 8 * F::KC <= 16 && ROW % 32 == 8, "row layout");
};

template <class S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_fwd_tc(Ws<float> w, Geo G, int M, int N,
                                                       const float* __restrict__ mlp,
                                                       const double* __restrict__ dep,
                                                       const float* __restrict__ spts, int nsp) {
  using K = FwdTc<S, WARPS>;
  using F = Fr<S>;
  constexpr int ROW = K::ROW;
  extern __shared__ uint4 smem4[];
  uint4* sfr = smem4;
  float* gvec = reinterpret_cast<float*>(sfr + K::NFR * 32);
  float* cvec = gvec + GVec::N;
  float* rows_all = cvec + CVec::N;
  const int lane = lane_id(), wid = threadIdx.x >> 5, g = lane >> 2;
  const int64_t MN = (int64_t)M * N, NS = MN + nsp;
  if ((int64_t)blockIdx.x * WARPS * 32 >= NS) return;
  __shared__ __align__(8) uint64_t s_bar;
  if (threadIdx.x == 0) mbar_init(&s_bar);
  __syncthreads();
  stage_async(&s_bar, sfr, w.wfrag, 0, K::NFR, gvec, 0, GVec::N + CVec::N);
  float* rows = rows_all + wid * 32 * ROW;
  const int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * 32;
  if (base >= NS) return;
  const int64_t s = base + lane;
  const bool act = s < NS;
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
  {
    float* my = rows + lane * ROW;
    float z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0.f;
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      loc[l] = compact<float>(locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2],
                                            (act && l == S::NL - 1) ? w.status : nullptr));
      gather_fast<float, S::CG>(G.lv[l], loc[l], z + l * S::CG);
    }
#pragma unroll
    for (int i = 0; i < 16; i += 2) *reinterpret_cast<float2*>(my + K::oZ + i) = make_float2(z[i], z[i + 1]);
    // colour input: grid features + view direction; smoothness points
    // (ray < 0) evaluate a harmless colour that is not stored
    const int cr = ray < 0 ? 0 : ray;
    const Loc qc = locate<false>(G.col, (double)p[0], (double)p[1], (double)p[2], nullptr);
    float inp[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) inp[i] = 0.f;
    gather_fast<float, S::CC>(G.col, compact<float>(qc), inp);
#pragma unroll
    for (int a = 0; a < 3; ++a) inp[S::CC + a] = w.r[cr * 3 + a];
#pragma unroll
    for (int i = 0; i < 16; i += 2) *reinterpret_cast<float2*>(my + K::oC + i) = make_float2(inp[i], inp[i + 1]);
  }
  mbar_wait(&s_bar, 0);
  __syncwarp();
  // MLP phases one m-tile (16 samples) at a time: half the live fragments
  // (occupancy), B fragments re-read from shared memory per m-tile
#pragma unroll 1
  for (int mt = 0; mt < 2; ++mt) {
    float* rm = rows + 16 * mt * ROW;
    // ---- colour: sigmoid(MLP_c([f_c, r]))  (gs/decoders.py:86-99)
    {
      float c0[1][4][4], c1[1][4][4], y[1][1][4];
      fill_cols(c0, cvec + CVec::b0);
      mma_layer<1, F::KC, 4>(
          [&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_rows<ROW>(rm, K::oC, 0, kk, ah, al); },
          sfr + F::C_W0 * 32, c0);
      relu_d(c0);
      fill_cols(c1, cvec + CVec::b1);
      mma_layer<1, 4, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(c0[0][kk], ah, al); },
                         sfr + F::C_W1 * 32, c1);
      relu_d(c1);
      fill_cols(y, cvec + CVec::b2);
      mma_layer<1, 4, 1>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(c1[0][kk], ah, al); },
                         sfr + F::C_W2 * 32, y);
#pragma unroll
      for (int r = 0; r < 4; ++r) y[0][0][r] = sigmoid_fast(y[0][0][r]);
      store_d<ROW>(y, rm, K::oY);
    }
    // ---- geometry: phi and dphi/dz = W0 ((W1 (W2 . m1)) . m0)
    {
      float h0[1][4][4], h1[1][4][4];
      fill_cols(h0, gvec + GVec::b0);
      mma_layer<1, F::KG, 4>(
          [&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_rows<ROW>(rm, K::oZ, 0, kk, ah, al); },
          sfr + F::G_W0 * 32, h0);
      const uint32_t m0 = relu_d(h0);
      fill_cols(h1, gvec + GVec::b1);
      mma_layer<1, 4, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(h0[0][kk], ah, al); },
                         sfr + F::G_W1 * 32, h1);
      const uint32_t m1 = relu_d(h1);
      float ph[1][2];
      phi_d(h1, gvec + GVec::w2, gvec[GVec::b2], ph);
      // delta chain (h0 and h1 registers reused)
      delta1_d(h1, m1, gvec + GVec::w2);
      zero_d(h0);
      mma_layer<1, 4, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(h1[0][kk], ah, al); },
                         sfr + F::G_W1T * 32, h0);
      mask_d(h0, m0);
      float gz[1][F::KG][4];
      zero_d(gz);
      mma_layer<1, 4, F::KG>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(h0[0][kk], ah, al); },
                             sfr + F::G_W0T * 32, gz);
      __syncwarp();  // every lane's z / colour-input reads of this m-tile are done
      store_d<ROW>(gz, rm, K::oZ);
      if ((lane & 3) == 0) {
        rm[g * ROW + K::oC] = ph[0][0];
        rm[(g + 8) * ROW + K::oC] = ph[0][1];
      }
    }
  }
  __syncwarp();
  if (!act) return;
  const float* my = rows + lane * ROW;
  float gr[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int l = 0; l < S::NL; ++l) level_dx_fast<float, S::CG>(G.lv[l], loc[l], my + K::oZ + l * S::CG, gr);
  w.sphi[s] = my[K::oC];
#pragma unroll
  for (int a = 0; a < 3; ++a) w.sgphi[s * 3 + a] = gr[a];
  if (ray >= 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) w.scol[s * 3 + c] = my[K::oY + c];
    if (w.pose_g) {  // pose refinement: keep dphi/dz for gsb_pose_grad (gsb_pose.cuh)
#pragma unroll
      for (int i = 0; i < S::IN_G; ++i) w.pose_g[s * S::IN_G + i] = my[K::oZ + i];
    }
  }
}

// ---------------------------------------------------------------------------
// backward, geometry: grid scatter + MLP weight grads

template <class S, int WARPS>
struct GeoTc {
  using F = Fr<S>;
  static constexpr int ROW = 104;  // 6 warps x 13 KB + 25 KB weights: 2 CTAs = 12 warps / SM
  static constexpr int oZ = 0;     // z, later dphi/dz (16)
  static constexpr int oA0 = 16;   // p z + v (16)
  static constexpr int oP = 32;    // p
  static constexpr int oM = 33;    // m1 bits
  static constexpr int oB0 = 40;   // delta0 (32)
  static constexpr int oV = oB0;   // v = sum_k ju_k theta_k (16): consumed before delta0 lands
  static constexpr int oA1 = 72;   // p h0 + q0 (32)
  static constexpr int NFR = F::NGEO;
  static constexpr size_t smem_rows() { return (size_t)WARPS * 32 * ROW * 4; }
  static constexpr size_t smem() { return (size_t)NFR * 32 * 16 + GVec::N * 4 + smem_rows(); }
  static_assert(oA1 + GSB_HID <= ROW && ROW % 32 == 8 && S::IN_G <= 16, "row layout");
};

template <class S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_bwd_geom_tc(Ws<float> w, Geo G, int M, int N,
                                                            const float* __restrict__ mlp,
                                                            const double* __restrict__ dep,
                                                            const float* __restrict__ spts, int nsp,
                                                            int agg_levels) {
  using K = GeoTc<S, WARPS>;
  using F = Fr<S>;
  constexpr int ROW = K::ROW;
  extern __shared__ uint4 smem4[];
  uint4* sfr = smem4;
  float* gvec = reinterpret_cast<float*>(sfr + K::NFR * 32);
  float* rows_all = gvec + GVec::N;
  const int lane = lane_id(), wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  __shared__ __align__(8) uint64_t s_bar;
  if (threadIdx.x == 0) mbar_init(&s_bar);
  __syncthreads();
  stage_async(&s_bar, sfr, w.wfrag, F::G_W0, K::NFR, gvec, 0, GVec::N);
  float* rows = rows_all + wid * 32 * ROW;
  float* myrow = rows + lane * ROW;
  const int64_t MN = (int64_t)M * N, NS = MN + nsp;
  const int64_t s = ((int64_t)blockIdx.x * WARPS + wid) * 32 + lane;
  const bool active = s < NS;
  // ---- per sample: point, z and v in one pass over the corners
  LocT<float> loc[S::NL];
  {
    float p = 0.f, u[3] = {0.f, 0.f, 0.f};
    float pt[3];
    if (active) {
      p = w.pbar[s];
#pragma unroll
      for (int a = 0; a < 3; ++a) u[a] = w.ubar[s * 3 + a];
      if (s < MN) {
        const int ray = (int)((uint32_t)s / (uint32_t)N);
        taped_point<float>(w.o + ray * 3, w.r + ray * 3,
                           dep[(int64_t)ray * w.ld + (int)((uint32_t)s % (uint32_t)N)], G.lo, G.hi, pt);
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) pt[a] = spts[(s - MN) * 3 + a];
      }
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) pt[a] = (float)G.lo[a];
    }
    float z[16], v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = v[i] = 0.f;
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      const LevelDev& L = G.lv[l];
      const LocT<float> lq = compact<float>(locate<false>(L, (double)pt[0], (double)pt[1], (double)pt[2], nullptr));
      loc[l] = lq;
      float wk[8], ju[8];
      corner_w_ju(lq, (float)L.inv_vs, u, wk, ju);
      const float* Fp = reinterpret_cast<const float*>(L.feat) + (int64_t)lq.base * S::CG;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float row[S::CG];
        load_row<float, S::CG>(Fp + corner_off(L, k) * S::CG, row);
#pragma unroll
        for (int c = 0; c < S::CG; ++c) {
          z[l * S::CG + c] = fmaf(wk[k], row[c], z[l * S::CG + c]);
          v[l * S::CG + c] = fmaf(ju[k], row[c], v[l * S::CG + c]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      *reinterpret_cast<float2*>(myrow + K::oZ + i) = make_float2(z[i], z[i + 1]);
      *reinterpret_cast<float2*>(myrow + K::oV + i) = make_float2(v[i], v[i + 1]);
      *reinterpret_cast<float2*>(myrow + K::oA0 + i) =
          make_float2(fmaf(p, z[i], v[i]), fmaf(p, z[i + 1], v[i + 1]));
    }
    myrow[K::oP] = p;
  }
  mbar_wait(&s_bar, 0);
  __syncwarp();
  // ---- MLP on the tensor cores, one m-tile (16 samples) at a time
  float accb0[4][2], accb1[4][2], accw2[4][2];  // column partial sums (cols 8nn+2t+c)
#pragma unroll
  for (int nn = 0; nn < 4; ++nn)
#pragma unroll
    for (int c = 0; c < 2; ++c) accb0[nn][c] = accb1[nn][c] = accw2[nn][c] = 0.f;
#pragma unroll 1
  for (int mt = 0; mt < 2; ++mt) {
    float* rm = rows + 16 * mt * ROW;
    const float pg[2] = {rm[g * ROW + K::oP], rm[(g + 8) * ROW + K::oP]};  // p of rows g, g+8
    float h0[1][4][4], h1[1][4][4];
    fill_cols(h0, gvec + GVec::b0);
    mma_layer<1, F::KG, 4>(
        [&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_rows<ROW>(rm, K::oZ, 0, kk, ah, al); },
        sfr + F::G_W0 * 32, h0);
    const uint32_t m0 = relu_d(h0);
    fill_cols(h1, gvec + GVec::b1);
    mma_layer<1, 4, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(h0[0][kk], ah, al); },
                       sfr + F::G_W1 * 32, h1);
    // A1 = p h0 (+ q0 below) parked in the row so h0 dies here
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int r = 0; r < 4; ++r) h0[0][nn][r] *= pg[r >> 1];
    store_d<ROW>(h0, rm, K::oA1);
    const uint32_t m1 = relu_d(h1);
    // dW2 += p h1 (column sums); per-sample m1 masks for the dW1 outer product
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int c = 0; c < 2; ++c) accw2[nn][c] += pg[0] * h1[0][nn][c] + pg[1] * h1[0][nn][2 + c];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const uint32_t msk = row_mask(m1, 0, hf);
      if (t == 0) reinterpret_cast<uint32_t*>(rm + (g + 8 * hf) * ROW + K::oM)[0] = msk;
    }
    // q0 = (v W0) . m0 ; A1 = p h0 + q0 ; dd1 = (q0 W1) . m1 -> dW2
    {
      float q0[1][4][4];
      zero_d(q0);
      mma_layer<1, F::KG, 4>(
          [&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_rows<ROW>(rm, K::oV, 0, kk, ah, al); },
          sfr + F::G_W0 * 32, q0);
      mask_d(q0, m0);
      load_d<ROW>(h0, rm, K::oA1);
#pragma unroll
      for (int nn = 0; nn < 4; ++nn)
#pragma unroll
        for (int r = 0; r < 4; ++r) h0[0][nn][r] += q0[0][nn][r];
      store_d<ROW>(h0, rm, K::oA1);
      zero_d(h1);
      mma_layer<1, 4, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(q0[0][kk], ah, al); },
                         sfr + F::G_W1 * 32, h1);
      mask_d(h1, m1);
#pragma unroll
      for (int nn = 0; nn < 4; ++nn)
#pragma unroll
        for (int c = 0; c < 2; ++c) accw2[nn][c] += h1[0][nn][c] + h1[0][nn][2 + c];
    }
    // delta1 = m1 . W2 -> db1 = sum p delta1 ; delta0 = (delta1 W1^T) . m0 -> rows, db0 ;
    // dphi/dz = delta0 W0^T -> rows (scatter)
    delta1_d(h1, m1, gvec + GVec::w2);
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int c = 0; c < 2; ++c) accb1[nn][c] += pg[0] * h1[0][nn][c] + pg[1] * h1[0][nn][2 + c];
    zero_d(h0);
    mma_layer<1, 4, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(h1[0][kk], ah, al); },
                       sfr + F::G_W1T * 32, h0);
    mask_d(h0, m0);
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int c = 0; c < 2; ++c) accb0[nn][c] += pg[0] * h0[0][nn][c] + pg[1] * h0[0][nn][2 + c];
    __syncwarp();  // v reads of this m-tile are done: delta0 takes its slot
    store_d<ROW>(h0, rm, K::oB0);
    float gz[1][F::KG][4];
    zero_d(gz);
    mma_layer<1, 4, F::KG>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(h0[0][kk], ah, al); },
                           sfr + F::G_W0T * 32, gz);
    __syncwarp();  // z reads of this m-tile are done
    store_d<ROW>(gz, rm, K::oZ);
  }
  __syncwarp();
  // ---- grid scatter: theta_l[idx_k] += g_l (p w_k + ju_k)
  const float p = myrow[K::oP];
  float u[3] = {0.f, 0.f, 0.f};
  if (active) {
#pragma unroll
    for (int a = 0; a < 3; ++a) u[a] = opaque(w.ubar[s * 3 + a]);
  }
#pragma unroll
  for (int l = 0; l < S::NL; ++l) {
    const LocT<float> lq = opaque(loc[l]);
    float wk[8], ju[8], coef[8];
    corner_w_ju(lq, (float)G.lv[l].inv_vs, u, wk, ju);
#pragma unroll
    for (int k = 0; k < 8; ++k) coef[k] = fmaf(p, wk[k], ju[k]);
    scatter_level<float, S::CG>(G.lv[l], lq, myrow + K::oZ + l * S::CG, coef, active, false,
                                w.det_keys, w.det_vals, s * (S::NL + 1) + l);
  }
  // ---- outer products over the warp's samples: dW0 += A0^T delta0, dW1 += A1^T delta1
  float d0[1][4][4], d1[2][4][4];
  zero_d(d0);
  zero_d(d1);
  const float w2l = gvec[GVec::w2 + lane];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int k0 = ks * 8;
    const uint32_t mk0 = reinterpret_cast<const uint32_t*>(rows + (k0 + t) * ROW + K::oM)[0];
    const uint32_t mk1 = reinterpret_cast<const uint32_t*>(rows + (k0 + t + 4) * ROW + K::oM)[0];
    uint32_t ah[2][4], al[2][4], bh0[4], bh1[4], bl0[4], bl1[4];
    {  // dW0 += A0^T delta0
      uint32_t a1h[1][4], a1l[1][4];
      frag_a(rows, ROW, K::oA0, k0, 0, a1h[0], a1l[0]);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) frag_b(rows, ROW, K::oB0, k0, nt * 8, bh0[nt], bh1[nt], bl0[nt], bl1[nt]);
      mma3_sweep(d0, a1h, a1l, bh0, bh1, bl0, bl1);
    }
    // dW1 += A1^T delta1, delta1[k][n] = m1_k(n) ? W2[n] : 0
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int n = nt * 8 + g;
      const float w2n = __shfl_sync(0xffffffffu, w2l, n);
      split_fast(((mk0 >> n) & 1u) ? w2n : 0.f, bh0[nt], bl0[nt]);
      split_fast(((mk1 >> n) & 1u) ? w2n : 0.f, bh1[nt], bl1[nt]);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) frag_a(rows, ROW, K::oA1, k0, mt * 16, ah[mt], al[mt]);
    mma3_sweep(d1, ah, al, bh0, bh1, bl0, bl1);
  }
  // column sums over the warp: reduce the 8 lanes sharing t
#pragma unroll
  for (int nn = 0; nn < 4; ++nn)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        accb0[nn][c] += __shfl_xor_sync(0xffffffffu, accb0[nn][c], o);
        accb1[nn][c] += __shfl_xor_sync(0xffffffffu, accb1[nn][c], o);
        accw2[nn][c] += __shfl_xor_sync(0xffffffffu, accw2[nn][c], o);
      }
  float accp = p;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) accp += __shfl_xor_sync(0xffffffffu, accp, o);
  // ---- CTA reduction -> partial slot blockIdx.x (geometry block of the MLP)
  __syncthreads();
  constexpr int NGP = S::NG;
  float* red = rows_all;  // [WARPS][NGP] over the (now free) rows
  {
    float* mine = red + (size_t)wid * NGP;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) frag_d_store(d0[0][nt], mine + S::oGW0, 0, nt * 8, S::IN_G);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) frag_d_store(d1[mt][nt], mine + S::oGW1, mt * 16, nt * 8, GSB_HID);
    if (g == 0) {
#pragma unroll
      for (int nn = 0; nn < 4; ++nn)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          mine[S::oGb0 + 8 * nn + 2 * t + c] = accb0[nn][c];
          mine[S::oGb1 + 8 * nn + 2 * t + c] = accb1[nn][c];
          mine[S::oGW2 + 8 * nn + 2 * t + c] = accw2[nn][c];
        }
    }
    if (lane == 0) mine[S::oGb2] = accp;
  }
  __syncthreads();
  const int slot = w.mlp_slots > 0 ? (int)(blockIdx.x % (unsigned)w.mlp_slots) : (int)blockIdx.x;
  float* out = w.mlp_part + (size_t)slot * S::NMLPP;
  for (int i = threadIdx.x; i < NGP; i += WARPS * 32) {
    float a = 0.f;
#pragma unroll
    for (int k = 0; k < WARPS; ++k) a += red[(size_t)k * NGP + i];
    if (w.mlp_slots > 0)
      atomicAdd(out + i, a);  // few L2-resident slots instead of one partial row per CTA
    else
      out[i] = a;
  }
}

// ---------------------------------------------------------------------------
// backward, colour

template <class S, int WARPS>
struct ColTc {
  using F = Fr<S>;
  static constexpr int ROW = 104;  // 4 warps x 13 KB + 27 KB weights: 2 CTAs = 8 warps / SM (measured best: the
                                   // smaller shared-memory carve-out leaves L1 for the colour-corner gathers)
  static constexpr int oA0 = 0;    // [inp (IN_C), 1, 0...] (16)
  static constexpr int oB0 = 16;   // a0_bar (32)
  static constexpr int oA1 = 48;   // h0c (32)
  static constexpr int oY = 80;    // y_bar (8 columns, 3 used)
  static constexpr int oM = 88;    // m1 bits (colour layer 1)
  static constexpr int oFB = 90;   // f_bar (8 columns, CC used)
  static constexpr int oCB = 98;   // cbar prefetch (3)
  static constexpr int NFR = F::NALL - F::NGEO;
  static constexpr size_t smem_rows() { return (size_t)WARPS * 32 * ROW * 4; }
  static constexpr size_t smem() { return (size_t)NFR * 32 * 16 + CVec::N * 4 + smem_rows(); }
  static_assert(oCB + 3 <= ROW && ROW % 32 == 8 && S::IN_C + 1 <= 16 && S::CC <= 8 && GSB_HID == 32,
                "row layout");
};

// Colour backward.  Sample-major rows hold only the outer-product factors
// [inp, 1] and a0_bar (dW0c, db0c) and h0c (dW1c); the dW1c partner a1_bar
// is rebuilt per fragment from y_bar, the layer-1 mask and W2c; dW2c, db1c
// and db2c are column sums of D fragments.
template <class S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, WARPS <= 6 ? 2 : 1) k_bwd_color_tc(Ws<float> w, Geo G, int M, int N,
                                                             const float* __restrict__ mlp,
                                                             const double* __restrict__ dep) {
  using K = ColTc<S, WARPS>;
  using F = Fr<S>;
  constexpr int ROW = K::ROW;
  extern __shared__ uint4 smem4[];
  uint4* sfr = smem4;  // fragment ids F::C_W0.. at index (id - NGEO)
  float* cvec = reinterpret_cast<float*>(sfr + K::NFR * 32);
  float* rows_all = cvec + CVec::N;
  const int lane = lane_id(), wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  __shared__ __align__(8) uint64_t s_bar;
  if (threadIdx.x == 0) mbar_init(&s_bar);
  __syncthreads();
  stage_async(&s_bar, sfr, w.wfrag, F::NGEO, K::NFR, cvec, GVec::N, CVec::N);
  const uint4* fr = sfr - F::NGEO * 32;  // index by global fragment id
  float* rows = rows_all + wid * 32 * ROW;
  float* myrow = rows + lane * ROW;
  const int64_t NS = (int64_t)M * N;
  const int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * 32;
  const int64_t s = base + lane;
  const bool active = s < NS;
  const int ray = active ? (int)((uint32_t)s / (uint32_t)N) : 0;
  LocT<float> q;
  {
    float pt[3];
    taped_point<float>(w.o + ray * 3, w.r + ray * 3,
                       active ? dep[(int64_t)ray * w.ld + (int)((uint32_t)s % (uint32_t)N)] : 0.0,
                       G.lo, G.hi, pt);
#pragma unroll
    for (int c = 0; c < 3; ++c) myrow[K::oCB + c] = active ? w.cbar[s * 3 + c] : 0.f;
    q = compact<float>(locate<false>(G.col, (double)pt[0], (double)pt[1], (double)pt[2], nullptr));
    float inp[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) inp[i] = 0.f;
    gather_fast<float, S::CC>(G.col, q, inp);
#pragma unroll
    for (int a = 0; a < 3; ++a) inp[S::CC + a] = w.r[ray * 3 + a];
    inp[S::IN_C] = 1.f;  // ones column: db0c rides on the dW0c outer product
#pragma unroll
    for (int i = 0; i < 16; i += 2) *reinterpret_cast<float2*>(myrow + K::oA0 + i) = make_float2(inp[i], inp[i + 1]);
  }
  mbar_wait(&s_bar, 0);
  __syncwarp();
  // ---- per m-tile: forward (masks, h0c), y_bar, a1_bar, a0_bar, f_bar
  // column sums, reduced over the warp per m-tile (reduce_scatter_g): this lane
  // owns column j = 8 (q >> 1) + 2t + (q & 1) of db1c and dW2c, q = rs_chunk()
  float sb1 = 0.f, sw2[3] = {0.f, 0.f, 0.f}, accb2[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) accb2[c] = 0.f;
#pragma unroll 1
  for (int mt = 0; mt < 2; ++mt) {
    float* rm = rows + 16 * mt * ROW;
    float c0[1][4][4], c1[1][4][4];
    fill_cols(c0, cvec + CVec::b0);
    mma_layer<1, F::KC, 4>(
        [&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_rows<ROW>(rm, K::oA0, 0, kk, ah, al); },
        fr + F::C_W0 * 32, c0);
    const uint32_t m0 = relu_d(c0);
    store_d<ROW>(c0, rm, K::oA1);
    fill_cols(c1, cvec + CVec::b1);
    mma_layer<1, 4, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(c0[0][kk], ah, al); },
                       fr + F::C_W1 * 32, c1);
    const uint32_t m1 = relu_d(c1);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const uint32_t msk = row_mask(m1, 0, hf);
      if (t == 0) reinterpret_cast<uint32_t*>(rm + (g + 8 * hf) * ROW + K::oM)[0] = msk;
    }
    float yb[1][1][4];
    fill_cols(yb, cvec + CVec::b2);
    mma_layer<1, 4, 1>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(c1[0][kk], ah, al); },
                       fr + F::C_W2 * 32, yb);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int col = 2 * t + (r & 1);
      const float cc = sigmoid_fast(yb[0][0][r]);
      yb[0][0][r] = col < 3 ? rm[(g + 8 * (r >> 1)) * ROW + K::oCB + col] * (cc * (1.f - cc)) : 0.f;
    }
    store_d<ROW>(yb, rm, K::oY);
    // y_bar of rows g, g+8 in every lane of the quad (cols 0,1 live in t=0, col 2 in t=1)
    float yv[2][3];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const int src = lane & ~3;
      yv[hf][0] = __shfl_sync(0xffffffffu, yb[0][0][2 * hf], src);
      yv[hf][1] = __shfl_sync(0xffffffffu, yb[0][0][2 * hf + 1], src);
      yv[hf][2] = __shfl_sync(0xffffffffu, yb[0][0][2 * hf], src + 1);
    }
    // dW2c += h1c^T y_bar: this m-tile's column sums, reduced over the warp and
    // accumulated (m-tile order) in the rows' spare columns; db2c += y_bar
    {
      float pw[24], r3[3];
#pragma unroll
      for (int nn = 0; nn < 4; ++nn)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            pw[(nn * 2 + cc) * 3 + c] = fmaf(c1[0][nn][cc], yv[0][c], c1[0][nn][2 + cc] * yv[1][c]);
      reduce_scatter_g(pw, r3);
#pragma unroll
      for (int c = 0; c < 3; ++c) sw2[c] += r3[c];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) accb2[c] += yv[0][c] + yv[1][c];
    // a1_bar = (y_bar W2c^T) . m1 -> db1c ; a0_bar = (a1_bar W1c^T) . m0 -> rows ; f_bar
    zero_d(c1);
    mma_layer<1, 1, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(yb[0][kk], ah, al); },
                       fr + F::C_W2T * 32, c1);
    mask_d(c1, m1);
    {
      float pb[8], r1[1];
#pragma unroll
      for (int nn = 0; nn < 4; ++nn)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) pb[nn * 2 + cc] = c1[0][nn][cc] + c1[0][nn][2 + cc];
      reduce_scatter_g(pb, r1);
      sb1 += r1[0];
    }
    zero_d(c0);
    mma_layer<1, 4, 4>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(c1[0][kk], ah, al); },
                       fr + F::C_W1T * 32, c0);
    mask_d(c0, m0);
    store_d<ROW>(c0, rm, K::oB0);
    float fb[1][F::NCC][4];
    zero_d(fb);
    mma_layer<1, 4, F::NCC>([&](int, int kk, uint32_t (&ah)[4], uint32_t (&al)[4]) { a_from_d(c0[0][kk], ah, al); },
                            fr + F::C_W0T * 32, fb);
    store_d<ROW>(fb, rm, K::oFB);
  }
  __syncwarp();
  {  // colour grid scatter: theta_c[idx_k] += w_k f_bar (warp-segmented)
    float wk[8];
    corner_w(q, wk);
    scatter_level<float, S::CC>(G.col, q, myrow + K::oFB, wk, active, false, w.det_keys, w.det_vals,
                                s * (S::NL + 1) + S::NL);
  }
  if (w.pose_fb && active) {  // pose refinement: f_bar and the view-direction cotangent
    float* o = w.pose_fb + s * 12;
#pragma unroll
    for (int c = 0; c < S::CC; ++c) o[c] = myrow[K::oFB + c];
#pragma unroll
    for (int a = 0; a < 3; ++a) {  // (a0_bar W0c^T) at the view-direction inputs
      const float* wr = mlp + S::oCW0 + (S::CC + a) * GSB_HID;
      float acc = 0.f;
#pragma unroll
      for (int jj = 0; jj < GSB_HID; ++jj) acc = fmaf(myrow[K::oB0 + jj], __ldg(wr + jj), acc);
      o[S::CC + a] = acc;
    }
  }
  // ---- outer products over the warp's samples: e0 = [inp,1]^T a0b, e1 = h0c^T a1b
  float w2c[4][3];  // W2c rows n = 8nt + g
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int c = 0; c < 3; ++c) w2c[nt][c] = cvec[CVec::w2 + (8 * nt + g) * 3 + c];
  float e0[1][4][4], e1[2][4][4];
  zero_d(e0);
  zero_d(e1);
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int k0 = ks * 8;
    uint32_t ah[2][4], al[2][4], bh0[4], bh1[4], bl0[4], bl1[4];
    {  // dW0c (+ db0c via the ones column) += [inp,1]^T a0b
      uint32_t a1h[1][4], a1l[1][4];
      frag_a(rows, ROW, K::oA0, k0, 0, a1h[0], a1l[0]);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) frag_b(rows, ROW, K::oB0, k0, nt * 8, bh0[nt], bh1[nt], bl0[nt], bl1[nt]);
      mma3_sweep(e0, a1h, a1l, bh0, bh1, bl0, bl1);
    }
    {  // dW1c += h0c^T a1b, a1b[k][n] = m1_k(n) ? sum_c W2c[n][c] y_bar_k[c] : 0
      const float* r0 = rows + (k0 + t) * ROW;
      const float* r1 = rows + (k0 + t + 4) * ROW;
      const uint32_t mk0 = reinterpret_cast<const uint32_t*>(r0 + K::oM)[0];
      const uint32_t mk1 = reinterpret_cast<const uint32_t*>(r1 + K::oM)[0];
      const float y00 = r0[K::oY], y01 = r0[K::oY + 1], y02 = r0[K::oY + 2];
      const float y10 = r1[K::oY], y11 = r1[K::oY + 1], y12 = r1[K::oY + 2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int n = nt * 8 + g;
        const float v0 = fmaf(w2c[nt][0], y00, fmaf(w2c[nt][1], y01, w2c[nt][2] * y02));
        const float v1 = fmaf(w2c[nt][0], y10, fmaf(w2c[nt][1], y11, w2c[nt][2] * y12));
        split_fast(((mk0 >> n) & 1u) ? v0 : 0.f, bh0[nt], bl0[nt]);
        split_fast(((mk1 >> n) & 1u) ? v1 : 0.f, bh1[nt], bl1[nt]);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) frag_a(rows, ROW, K::oA1, k0, mt * 16, ah[mt], al[mt]);
      mma3_sweep(e1, ah, al, bh0, bh1, bl0, bl1);
    }
  }
  // column sums over the warp: reduce the 8 lanes sharing t
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) accb2[c] += __shfl_xor_sync(0xffffffffu, accb2[c], o);
  }
  __syncthreads();
  constexpr int NCP = S::NMLP - S::NG;
  float* red = rows_all;
  {
    float* mine = red + (size_t)wid * NCP;
    const int o = S::NG;
    if (lane < S::oCW0 - S::NG) mine[lane] = 0.f;  // alignment padding
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) frag_d_store(e0[0][nt], mine + (S::oCW0 - o), 0, nt * 8, S::IN_C + 1);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) frag_d_store(e1[mt][nt], mine + (S::oCW1 - o), mt * 16, nt * 8, GSB_HID);
    {
      const int q = rs_chunk(), j = 8 * (q >> 1) + 2 * t + (q & 1);
      mine[S::oCb1 - o + j] = sb1;
#pragma unroll
      for (int c = 0; c < 3; ++c) mine[S::oCW2 - o + j * 3 + c] = sw2[c];
    }
    if (lane == 0) {  // y_bar is quad-replicated: lane 0's sum covers every row once
#pragma unroll
      for (int c = 0; c < 3; ++c) mine[S::oCb2 - o + c] = accb2[c];
    }
  }
  __syncthreads();
  const int slot = w.mlp_slots > 0 ? (int)(blockIdx.x % (unsigned)w.mlp_slots) : (int)blockIdx.x;
  float* out = w.mlp_part + (size_t)slot * S::NMLPP + S::NG;
  for (int i = threadIdx.x; i < NCP; i += WARPS * 32) {
    float a = 0.f;
#pragma unroll
    for (int k = 0; k < WARPS; ++k) a += red[(size_t)k * NCP + i];
    if (w.mlp_slots > 0)
      atomicAdd(out + i, a);
    else
      out[i] = a;
  }
}

}  // namespace tc
}  // namespace gsb
