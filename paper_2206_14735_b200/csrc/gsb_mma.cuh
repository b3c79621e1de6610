// gsb_mma.cuh -- mma.sync m16n8k8 TF32 helpers of the float32 decoders
// (gsb_tc.cuh): tf32 splits for 3xTF32 (hi*hi + hi*lo + lo*hi, ~fp32
// accuracy), the MMA itself, and fragment loads / stores from sample-major
// shared-memory rows (the weight-gradient outer products).
#pragma once

#include "gsb_mlp.cuh"

namespace gsb {

__device__ __forceinline__ uint32_t tf32_of(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32_of(x);
  lo = tf32_of(x - __uint_as_float(hi));
}
// per-use split: hi = x as is (mma.sync reads the top 19 bits of a tf32
// operand, i.e. trunc(x)), lo = x - trunc(x) exact, also passed raw:
// |x - trunc(x) - trunc(lo)| <= 2^-21 |x|
__device__ __forceinline__ void split_fast(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x);
  lo = __float_as_uint(x - __uint_as_float(hi & 0xffffe000u));
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

}  // namespace gsb
