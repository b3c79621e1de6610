// gsb_common.cuh -- device building blocks shared by the step kernels.
//
// Compiled with --fmad=false: every multiply-add that the reference performs
// as two rounded numpy/numba operations stays two rounded operations here;
// the MLP and interpolation hot loops use explicit fma() where fusing is
// harmless (those values are only compared within tolerance).
#pragma once

#include "gsb_pcg_tables.cuh"
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gsb.h"

#define GSB_HID 32  // decoders.HIDDEN_WIDTH (gs/decoders.py:22)

namespace gsb {

// ---------------------------------------------------------------------------
// MLP block layout (arena order, gs/decoders.py:40-49, weights stored (in, out)):
// geom W0 (IN,32), b0, W1 (32,32), b1, W2 (32,1), b2, pad to a multiple of 4,
// colour W0 (CC+3,32), b0, W1, b1, W2 (32,3), b2.
#define GSB_MLP_MAX 3200

template <int NL_, int CG_, int CC_>
struct Shape {
  static constexpr int NL = NL_, CG = CG_, CC = CC_;
  static constexpr int IN_G = NL * CG;
  static constexpr int IN_C = CC + 3;
  static constexpr int oGW0 = 0;
  static constexpr int oGb0 = oGW0 + IN_G * GSB_HID;
  static constexpr int oGW1 = oGb0 + GSB_HID;
  static constexpr int oGb1 = oGW1 + GSB_HID * GSB_HID;
  static constexpr int oGW2 = oGb1 + GSB_HID;
  static constexpr int oGb2 = oGW2 + GSB_HID;
  static constexpr int NG = oGb2 + 1;
  static constexpr int oCW0 = (NG + 3) / 4 * 4;  // colour net starts 16-byte aligned
  static constexpr int oCb0 = oCW0 + IN_C * GSB_HID;
  static constexpr int oCW1 = oCb0 + GSB_HID;
  static constexpr int oCb1 = oCW1 + GSB_HID * GSB_HID;
  static constexpr int oCW2 = oCb1 + GSB_HID;
  static constexpr int oCb2 = oCW2 + GSB_HID * 3;
  static constexpr int NMLP = oCb2 + 3;
  static constexpr int NMLPP = (NMLP + 3) / 4 * 4;  // stride of the MLP partial rows (16-byte aligned)
  static_assert(NMLP <= GSB_MLP_MAX, "MLP block exceeds constant buffer");
};

// ---------------------------------------------------------------------------
// numpy PCG64 (XSL-RR 128/64), gs/seeds.py:28-30 -> Generator.random():
// state advances before each output; double = (x >> 11) * 2^-53.

typedef unsigned __int128 u128;
__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

struct Pcg {
  u128 state, inc;
  __device__ __forceinline__ void init(const gsb_pcg64_t& g) {
    state = ((u128)g.state_hi << 64) | (u128)g.state_lo;
    inc = ((u128)g.inc_hi << 64) | (u128)g.inc_lo;
  }
  // jump ahead by delta draws: for each set bit k, state -> M_k state + inc P_k
  // (gsb_pcg_tables.cuh; exact mod 2^128, equal to square-and-multiply)
  __device__ __forceinline__ void advance(uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0;
    for (int k = 0; delta != 0; ++k, delta >>= 1) {
      if (delta & 1) {
        const u128 Mk = ((u128)kPcgMultPow[k][0] << 64) | (u128)kPcgMultPow[k][1];
        const u128 Pk = ((u128)kPcgPlusPow[k][0] << 64) | (u128)kPcgPlusPow[k][1];
        acc_mult *= Mk;
        acc_plus = acc_plus * Mk + inc * Pk;
      }
    }
    state = acc_mult * state + acc_plus;
  }
  __device__ __forceinline__ uint64_t next64() {
    state = state * pcg_mult() + inc;
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ __forceinline__ double next_double() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
};

// ---------------------------------------------------------------------------
// grid lattice (gs/diffcore.py:704-767)

struct LevelDev {
  const void* feat;
  void* grad;
  int nx, ny, nz, C;
  double ox, oy, oz, vs, inv_vs, eps;
};

struct Loc {
  int64_t base;     // flat vertex index of corner 0
  double fx, fy, fz;
};

// local = (p - origin) / vs (gs/diffcore.py:740), correctly rounded without
// a division: with inv = RN(1/vs) (computed on the host), q = RN(d inv) is
// within 1 ulp of d/vs, the remainder r = d - q vs is exact under an FMA, and
// RN(q + r inv) is the correctly rounded quotient (Markstein's theorem; no
// underflow/overflow for lattice coordinates).  So floor() -- the voxel
// index -- always equals the reference's, at 1 DMUL + 2 DFMA per axis and no
// slow-path call.
template <bool EXACT>
__device__ __forceinline__ double axis_local(double p, double o, double vs, double inv) {
  const double d = p - o;
  const double q = d * inv;
  const double r = fma(-q, vs, d);
  return fma(r, inv, q);
}

template <bool EXACT>
__device__ __forceinline__ Loc locate(const LevelDev& L, double px, double py, double pz,
                                      int* status) {
  double lx = axis_local<EXACT>(px, L.ox, L.vs, L.inv_vs);
  double ly = axis_local<EXACT>(py, L.oy, L.vs, L.inv_vs);
  double lz = axis_local<EXACT>(pz, L.oz, L.vs, L.inv_vs);
  if (lx < -L.eps || ly < -L.eps || lz < -L.eps || lx > (L.nx - 1) + L.eps ||
      ly > (L.ny - 1) + L.eps || lz > (L.nz - 1) + L.eps || !(lx == lx && ly == ly && lz == lz)) {
    if (status) atomicOr(status + GSB_ST_BOUNDS, 1);
  }
  int cx = (int)floor(lx), cy = (int)floor(ly), cz = (int)floor(lz);
  cx = max(min(cx, L.nx - 2), 0);
  cy = max(min(cy, L.ny - 2), 0);
  cz = max(min(cz, L.nz - 2), 0);
  Loc r;
  r.base = ((int64_t)cx * L.ny + cy) * L.nz + cz;
  r.fx = lx - cx;
  r.fy = ly - cy;
  r.fz = lz - cz;
  return r;
}

// corner k = 4dx + 2dy + dz (gs/diffcore.py:731-735) -> flat offset
__device__ __forceinline__ int64_t corner_off(const LevelDev& L, int k) {
  return (int64_t)((k >> 2) & 1) * L.ny * L.nz + (int64_t)((k >> 1) & 1) * L.nz + (k & 1);
}

// ---------------------------------------------------------------------------
// row loads / vector reductions

template <typename T, int C>
__device__ __forceinline__ void load_row(const T* __restrict__ p, T (&v)[C]) {
  if constexpr (sizeof(T) == 4 && C % 4 == 0) {
#pragma unroll
    for (int c = 0; c < C; c += 4) {
      float4 x = __ldg(reinterpret_cast<const float4*>(p + c));
      v[c] = x.x; v[c + 1] = x.y; v[c + 2] = x.z; v[c + 3] = x.w;
    }
  } else if constexpr (sizeof(T) == 4 && C % 2 == 0) {
#pragma unroll
    for (int c = 0; c < C; c += 2) {
      float2 x = __ldg(reinterpret_cast<const float2*>(p + c));
      v[c] = x.x; v[c + 1] = x.y;
    }
  } else if constexpr (sizeof(T) == 8 && C % 2 == 0) {
#pragma unroll
    for (int c = 0; c < C; c += 2) {
      double2 x = __ldg(reinterpret_cast<const double2*>(p + c));
      v[c] = x.x; v[c + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c) v[c] = __ldg(p + c);
  }
}

__device__ __forceinline__ void red_add_v4(float* a, float x, float y, float z, float w) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(x), "f"(y), "f"(z),
               "f"(w)
               : "memory");
}
__device__ __forceinline__ void red_add_v2(float* a, float x, float y) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(a), "f"(x), "f"(y) : "memory");
}

template <typename T, int C>
__device__ __forceinline__ void red_row(T* p, const T (&v)[C]) {
  if constexpr (sizeof(T) == 4 && C % 4 == 0) {
#pragma unroll
    for (int c = 0; c < C; c += 4) red_add_v4(p + c, v[c], v[c + 1], v[c + 2], v[c + 3]);
  } else if constexpr (sizeof(T) == 4 && C == 6) {
    // 24-byte rows: a 16-byte and an 8-byte red, in the order the row's
    // alignment allows (2 reds instead of 3)
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      red_add_v4(p, v[0], v[1], v[2], v[3]);
      red_add_v2(p + 4, v[4], v[5]);
    } else {
      red_add_v2(p, v[0], v[1]);
      red_add_v4(p + 2, v[2], v[3], v[4], v[5]);
    }
  } else if constexpr (sizeof(T) == 4 && C % 2 == 0) {
#pragma unroll
    for (int c = 0; c < C; c += 2) red_add_v2(p + c, v[c], v[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c) atomicAdd(p + c, v[c]);
  }
}

template <typename T>
__device__ __forceinline__ T sigmoid_raw(T x) {  // gs/diffcore.py:445-451
  if (x >= T(0)) return T(1) / (T(1) + exp(-x));
  T ex = exp(x);
  return ex / (T(1) + ex);
}

// Division without the IEEE slow-path subroutine call (used where values are
// only compared within tolerance): float -> __fdividef (2 ulp), double ->
// Newton-refined reciprocal + one remainder correction (faithful).
__device__ __forceinline__ float fdiv(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double fdiv(double a, double b) {
  double y = (double)__frcp_rn((float)b);
  y = fma(fma(-b, y, 1.0), y, y);
  y = fma(fma(-b, y, 1.0), y, y);
  const double q = a * y;
  return fma(fma(-q, b, a), y, q);
}

// logistic function for the colour head, call-free
template <typename T>
__device__ __forceinline__ T sigmoid_fast(T x) {
  if (x >= T(0)) return fdiv(T(1), T(1) + exp(-x));
  const T ex = exp(x);
  return fdiv(ex, T(1) + ex);
}

template <typename T>
__device__ __forceinline__ T sgn(T x) {
  return x > T(0) ? T(1) : (x < T(0) ? T(-1) : T(0));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace gsb
