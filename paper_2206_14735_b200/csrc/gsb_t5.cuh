// gsb_t5.cuh -- decoder layers on the 5th-generation tensor cores (tcgen05).
//
// A CTA of 128 threads owns a tile of 128 samples: thread = sample = TMEM
// lane.  Per-sample work (point, grid location, trilinear gather, epilogue)
// is lane-per-sample as in gsb_tc.cuh; each 32-wide layer is ONE elected
// thread issuing tcgen05.mma kind::tf32 with
//   A = activations (M = 128 samples x K) in TMEM, written by tcgen05.st,
//   B = weights (N = 32 x K) in shared memory, canonical K-major no-swizzle
//       tiles built once per step by k_wfrag and staged by a TMA bulk copy,
//   D = fp32 accumulator (128 lanes x 32 columns) in TMEM, read back with
//       tcgen05.ld.32x32b (thread t reads its own lane).
// 3xTF32 split precision (Ahi Bhi + Ahi Blo + Alo Bhi, ~fp32 accuracy) as in
// the mma.sync path.  TMEM columns: D [0, 32), A hi [32, 64), A lo [64, 96).
// tools/tc05_test.cu measured this TS form at 57 TFMA/s effective on chained
// layers vs 37 for the register-chained mma.sync form.
#pragma once

#include "gsb_tc.cuh"

namespace gsb {
namespace t5 {

using tc::smem_u32;

// division by a loop-invariant divisor (samples per ray): multiply-high
// with a precomputed magic number (round-up method, exact for every 32-bit
// n and d >= 1) instead of the generic ~20-instruction sequence per sample
struct FastDiv {
  uint32_t d, m, sh;
  __device__ __forceinline__ explicit FastDiv(uint32_t d_) : d(d_) {
    sh = d_ > 1 ? 32u - (uint32_t)__clz(d_ - 1u) : 0u;  // ceil(log2 d)
    m = d_ > 1 ? (uint32_t)((((1ull << 32) * ((1ull << sh) - d_)) / d_) + 1ull) : 0u;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (sh == 0) return n;
    const uint32_t t = __umulhi(n, m);
    return (t + ((n - t) >> 1)) >> (sh - 1);
  }
  __device__ __forceinline__ uint32_t mod(uint32_t n, uint32_t q) const { return n - q * d; }
};

constexpr int kTile = 128;         // samples per CTA = TMEM lanes
constexpr int kCtaPerSm = 4;       // 128 TMEM columns each: 4 x 128 = 512
constexpr uint32_t kCols = 128;
// taped forward: TMEM columns D [0, 32), A hi / lo [32, 96), and the two
// finest levels' spatial Jacobians [96, 128)
constexpr int kJacLevels = 2;
constexpr uint32_t kJacCol = 96;

// kind::tf32, D f32, A/B K-major, M = 128, N = 32 (or 16)
__host__ __device__ constexpr uint32_t idesc(uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
constexpr uint32_t kIdesc = idesc(32);

// shared-memory matrix descriptor, SWIZZLE_NONE, descriptor version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
template <uint32_t NN = 32>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc(NN)), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// all threads' TMEM stores visible to the MMA issued after this
__device__ __forceinline__ void cta_sync_tmem() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
}

#define GSB_R(i) "r"(__float_as_uint(v[i]))
__device__ __forceinline__ void st8(uint32_t ta, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), GSB_R(0),
               GSB_R(1), GSB_R(2), GSB_R(3), GSB_R(4), GSB_R(5), GSB_R(6), GSB_R(7)
               : "memory");
}
__device__ __forceinline__ void st16(uint32_t ta, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          ta),
      GSB_R(0), GSB_R(1), GSB_R(2), GSB_R(3), GSB_R(4), GSB_R(5), GSB_R(6), GSB_R(7), GSB_R(8), GSB_R(9), GSB_R(10),
      GSB_R(11), GSB_R(12), GSB_R(13), GSB_R(14), GSB_R(15)
      : "memory");
}
__device__ __forceinline__ void st32(uint32_t ta, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
      GSB_R(0), GSB_R(1), GSB_R(2), GSB_R(3), GSB_R(4), GSB_R(5), GSB_R(6), GSB_R(7), GSB_R(8), GSB_R(9), GSB_R(10),
      GSB_R(11), GSB_R(12), GSB_R(13), GSB_R(14), GSB_R(15), GSB_R(16), GSB_R(17), GSB_R(18), GSB_R(19),
      GSB_R(20), GSB_R(21), GSB_R(22), GSB_R(23), GSB_R(24), GSB_R(25), GSB_R(26), GSB_R(27), GSB_R(28),
      GSB_R(29), GSB_R(30), GSB_R(31)
      : "memory");
}
#undef GSB_R
__device__ __forceinline__ void ld32(uint32_t ta, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(ta)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void ld16(uint32_t ta, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// several TMEM loads in flight, one wait (a single asm statement, so no use
// of the loaded registers can be scheduled before the wait)
__device__ __forceinline__ void ld32x2(uint32_t a0, uint32_t a1, float (&v0)[32], float (&v1)[32]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(a0), "r"(a1)
      : "memory");
  #pragma unroll
  for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(r[0 + i]);
  #pragma unroll
  for (int i = 0; i < 32; ++i) v1[i] = __uint_as_float(r[32 + i]);
}
__device__ __forceinline__ void ld8(uint32_t ta, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// hi = x itself: the tensor core reads the top 19 bits of a tf32 operand
// (truncation), so the operand it sees is trunc(x) and lo = x - trunc(x) is
// exact (>= 0, < 2^-10 |x|; its own truncation leaves <= 2^-21 |x|).  No
// rounding op, and hi needs no register of its own: 1.338 -> 1.292 ms per
// step over rounding hi (half away at bit 13) as round 1 did.
__device__ __forceinline__ void split2(float x, float& hi, float& lo) {
  hi = x;
  lo = x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

// A hi / lo (K = 8 KS columns) to TMEM columns [32, 32 + 8KS) / [64, 64 + 8KS)
template <int KS>
__device__ __forceinline__ void store_a(uint32_t tl, const float* x) {
  float h[8 * KS], l[8 * KS];
#pragma unroll
  for (int i = 0; i < 8 * KS; ++i) split2(x[i], h[i], l[i]);
  if constexpr (KS == 1) {
    st8(tl + 32, h);
    st8(tl + 64, l);
  } else if constexpr (KS == 2) {
    st16(tl + 32, h);
    st16(tl + 64, l);
  } else {
    static_assert(KS == 4, "K");
    st32(tl + 32, h);
    st32(tl + 64, l);
  }
}

// D[0, NN) = A (TMEM) x B (smem tiles bh / bl, NN x K, K = 8 KS), 3xTF32
template <int KS, uint32_t NN = 32>
__device__ __forceinline__ void issue_layer(uint32_t tmem, uint32_t bh, uint32_t bl) {
  constexpr uint32_t sbo = KS * 8 * 32;  // 8 rows x K fp32
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const uint32_t off = kk * 256;  // two 128-byte core matrices per k-step of 8
    mma_ts<NN>(tmem, tmem + 64 + kk * 8, sdesc(bh + off, 128, sbo), kk > 0 ? 1u : 0u);
    mma_ts<NN>(tmem, tmem + 32 + kk * 8, sdesc(bl + off, 128, sbo), 1u);
    mma_ts<NN>(tmem, tmem + 32 + kk * 8, sdesc(bh + off, 128, sbo), 1u);
  }
}

// ---------------------------------------------------------------------------
// no-grad SDF at listed samples (importance passes, gs/renderer.py:330-340):
// persistent CTAs, one 128-sample tile per iteration

struct SdfT5 {
  static constexpr int NW = tc::UmmaW::W1L + 1024;  // W0^T, W1^T tiles only
  static constexpr size_t smem() { return (size_t)(NW + tc::GVec::N) * 4; }
};

template <class S>
__global__ void __launch_bounds__(kTile) k_sdf_eval_t5(Ws<float> w, Geo G, int M, int Nc,
                                                      const double* __restrict__ dep,
                                                      double* __restrict__ phi,
                                                      const int32_t* __restrict__ list,
                                                      const int32_t* __restrict__ list_count) {
  using F = tc::Fr<S>;
  constexpr int KG = F::KG;
  const FastDiv fdc((uint32_t)Nc);
  extern __shared__ __align__(128) float t5_smem[];
  float* sw = t5_smem;                 // UmmaW block
  float* svec = t5_smem + SdfT5::NW;  // GVec block
  __shared__ __align__(8) uint64_t s_bar[2];  // [0] weight staging, [1] MMA completion
  __shared__ uint32_t s_tmem;
  const int64_t total = list ? (int64_t)(*list_count) : (int64_t)M * Nc;
  const int64_t ntiles = (total + kTile - 1) / kTile;
  if ((int64_t)blockIdx.x >= ntiles) return;  // block-uniform, before any TMEM allocation
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    tc::mbar_init(&s_bar[0]);
    tc::mbar_init(&s_bar[1]);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    constexpr uint32_t wb = SdfT5::NW * 4, vb = tc::GVec::N * 4;
    tc::mbar_expect(&s_bar[0], wb + vb);
    tc::bulk_g2s(sw, w.wfrag + tc::kUmmaBaseU4, wb, &s_bar[0]);
    tc::bulk_g2s(svec, reinterpret_cast<const float*>(w.wfrag + tc::kVecBase), vb, &s_bar[0]);
  }
  const uint32_t tmem = s_tmem;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);  // this warp's 32 lanes
  const uint32_t w0h = smem_u32(sw + tc::UmmaW::W0H), w0l = smem_u32(sw + tc::UmmaW::W0L);
  const uint32_t w1h = smem_u32(sw + tc::UmmaW::W1H), w1l = smem_u32(sw + tc::UmmaW::W1L);
  uint32_t phase = 0;
  bool staged = false;
  // one tile's lane-per-sample inputs: (ray, slot) and z at the sample point
  auto gather = [&](int64_t tile, float (&z)[8 * KG], int& ray, int& slot, bool& act) {
    const int64_t s = tile * kTile + tid;
    act = s < total;
    ray = 0;
    slot = 0;
    if (act) {
      if (list) {
        const int32_t e = list[s];
        ray = e / GSB_KMAX;
        slot = e % GSB_KMAX;
      } else {
        const uint32_t q = fdc.div((uint32_t)s);
        ray = (int)q;
        slot = (int)fdc.mod((uint32_t)s, q);
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
#pragma unroll
    for (int i = S::IN_G; i < 8 * KG; ++i) z[i] = 0.f;
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      // bounds / NaN flag from the finest level only: the points are clipped
      // to the clamp box (half a finest voxel inside the grid box on every
      // side), so every level passes unless the point is NaN, which every
      // level catches alike (the other levels' compares compile away)
      const Loc q = locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2],
                                  (act && l == S::NL - 1) ? w.status : nullptr);
      gather_fast<float, S::CG>(G.lv[l], compact<float>(q), z + l * S::CG);
    }
  };
  float z[8 * KG];
  int ray, slot;
  bool act;
  gather(blockIdx.x, z, ray, slot, act);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    store_a<KG>(tl, z);
    cta_sync_tmem();
    if (!staged) {
      tc::mbar_wait(&s_bar[0], 0);
      staged = true;
    }
    if (tid == 0) {
      issue_layer<KG>(tmem, w0h, w0l);
      commit(&s_bar[1]);
    }
    // software pipeline: the next tile's gathers overlap this tile's MMAs
    const int cur_ray = ray, cur_slot = slot;
    const bool cur_act = act;
    if (tile + gridDim.x < ntiles) gather(tile + gridDim.x, z, ray, slot, act);
    tc::mbar_wait(&s_bar[1], phase);
    phase ^= 1u;
    fence_after();
    float h[32];
    ld32(tl, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) h[n] = fmaxf(h[n] + svec[tc::GVec::b0 + n], 0.f);
    store_a<4>(tl, h);
    cta_sync_tmem();
    if (tid == 0) {
      issue_layer<4>(tmem, w1h, w1l);
      commit(&s_bar[1]);
    }
    tc::mbar_wait(&s_bar[1], phase);
    phase ^= 1u;
    fence_after();
    ld32(tl, h);
    float acc = svec[tc::GVec::b2];
#pragma unroll
    for (int n = 0; n < 32; ++n) acc = fmaf(fmaxf(h[n] + svec[tc::GVec::b1 + n], 0.f), svec[tc::GVec::w2 + n], acc);
    if (cur_act) phi[(int64_t)cur_ray * w.ld + cur_slot] = (double)acc;
  }
  fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
}


// ---------------------------------------------------------------------------
// taped forward (same contract as tc::k_fwd_tc): per sample phi, dphi/dx and
// colour, plus dphi/dz for pose refinement.  Six chained tcgen05 layers per
// 128-sample tile: z W0, h0 W1, delta1 W1^T, delta0 W0^T (N = 16), then the
// colour decoder [f_c, r] W0c, h0c W1c; the 32 -> 1 / 32 -> 3 heads and the
// grid-space gradient are per-lane epilogues.  The next tile's gathers
// overlap the last MMA.

// Staged form (STG): the finest level's 8 corner rows of the NEXT tile are
// copied HBM -> shared memory with cp.async (16 B per row, thread-private
// slots [corner][lane]) while this tile's six MMA rounds run, so its gather
// reads them from shared memory; the next tile's point is formed during this
// tile's gather (its depth / ray loads overlap the coarse-level loads) and
// parked in shared memory.  16 KB + 1.5 KB per CTA: still 4 CTAs per SM.
struct FwdT5 {
  static constexpr int kVecEnd = tc::UmmaW::NFWD + tc::GVec::N + tc::CVec::N;  // floats
  static constexpr int kStg = kVecEnd;                 // float4 [8][kTile]
  static constexpr int kPt = kStg + 8 * kTile * 4;     // float [3][kTile]
  static constexpr size_t smem(bool stg = false) { return (size_t)(stg ? kPt + 3 * kTile : kVecEnd) * 4; }
};
static_assert(FwdT5::kVecEnd % 4 == 0, "staging rows 16-byte aligned");

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <class S, int CPS = kCtaPerSm, bool STG = false, bool DBG = false>
__global__ void __launch_bounds__(kTile, CPS) k_fwd_t5(Ws<float> w, Geo G, int M, int N,
                                                 const double* __restrict__ dep,
                                                 const float* __restrict__ spts, int nsp) {
  using F = tc::Fr<S>;
  using U = tc::UmmaW;
  constexpr int KG = F::KG, KC = F::KC;
  static_assert(8 * KG <= 16 && 8 * KC <= 16, "input widths");
  static_assert(!STG || (S::CG == 4 && S::NL >= kJacLevels), "staged form: 16-byte finest rows");
  const FastDiv fdn((uint32_t)N);
  extern __shared__ __align__(128) float t5_smem[];
  float* sw = t5_smem;
  const float* gvec = t5_smem + U::NFWD;
  const float* cvec = gvec + tc::GVec::N;
  __shared__ __align__(8) uint64_t s_bar[2];  // [0] weight staging, [1] MMA completion
  __shared__ uint32_t s_tmem;
  const int64_t MN = (int64_t)M * N, NS = MN + nsp;
  const int64_t ntiles = (NS + kTile - 1) / kTile;
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t first = blockIdx.x, stride = gridDim.x;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    tc::mbar_init(&s_bar[0]);
    tc::mbar_init(&s_bar[1]);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    constexpr uint32_t wb = U::NFWD * 4, vb = (tc::GVec::N + tc::CVec::N) * 4;
    tc::mbar_expect(&s_bar[0], wb + vb);
    tc::bulk_g2s(sw, w.wfrag + tc::kUmmaBaseU4, wb, &s_bar[0]);
    tc::bulk_g2s(t5_smem + U::NFWD, reinterpret_cast<const float*>(w.wfrag + tc::kVecBase), vb, &s_bar[0]);
  }
  const uint32_t tmem = s_tmem;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  uint64_t* bar_d = &s_bar[1];
  auto sa = [&](int off) { return smem_u32(sw + off); };
  uint32_t phase = 0;
  auto run = [&](auto issue) {  // all lanes' A stores -> one thread issues -> wait for D
    cta_sync_tmem();
    if (tid == 0) {
      if (!(DBG && (w.dbg & 16))) issue();
      commit(bar_d);
    }
  };
  auto wait_d = [&]() {
    tc::mbar_wait(bar_d, phase);
    phase ^= 1u;
    fence_after();
  };
  // lane-per-sample inputs of one tile
  int64_t s;
  int ray;
  bool act;
  LocT<float> loc[S::NL];
  float z[8 * KG], inp[8 * KC];
  auto sample_of = [&](int64_t tile, int64_t& s_, int& ray_, bool& act_) {
    s_ = ((w.sweep & 1) ? ntiles - 1 - tile : tile) * kTile + tid;  // backward sweep: L2 reuse
    act_ = s_ < NS;
    ray_ = act_ && s_ < MN ? (int)fdn.div((uint32_t)s_) : -1;
  };
  auto point_of = [&](int64_t s_, int ray_, bool act_, float (&p)[3]) {
    if (ray_ >= 0) {
      taped_point<float>(w.o + ray_ * 3, w.r + ray_ * 3,
                         dep[(int64_t)ray_ * w.ld + (int)fdn.mod((uint32_t)s_, (uint32_t)ray_)], G.lo, G.hi, p);
    } else if (act_) {
#pragma unroll
      for (int a = 0; a < 3; ++a) p[a] = spts[(s_ - MN) * 3 + a];
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) p[a] = (float)G.lo[a];
    }
  };
  float4* stg = reinterpret_cast<float4*>(t5_smem + FwdT5::kStg);
  float* spt = t5_smem + FwdT5::kPt;
  // STG: issue the finest level's corner copies for the point p (this
  // thread's slots), park p
  auto stage = [&](const float (&p)[3]) {
    cp_async_wait_all();  // (no-op: the previous copies were consumed)
    const LevelDev& L = G.lv[S::NL - 1];
    const LocT<float> q = compact<float>(locate<false>(L, (double)p[0], (double)p[1], (double)p[2], nullptr));
    const float* F = reinterpret_cast<const float*>(L.feat) + (int64_t)q.base * S::CG;
#pragma unroll
    for (int k = 0; k < 8; ++k) cp_async16(stg + k * kTile + tid, F + corner_off(L, k) * S::CG);
    cp_async_commit();
#pragma unroll
    for (int a = 0; a < 3; ++a) spt[a * kTile + tid] = p[a];
  };
  auto gather = [&](int64_t tile) {
    sample_of(tile, s, ray, act);
    float p[3];
    if constexpr (STG) {
#pragma unroll
      for (int a = 0; a < 3; ++a) p[a] = spt[a * kTile + tid];
    } else {
      point_of(s, ray, act, p);
    }
    // STG: the next tile's point (its loads overlap this tile's gathers)
    const int64_t nt = tile + stride;
    float pn[3];
    if constexpr (STG) {
      if (nt < ntiles) {
        int64_t sn;
        int rn;
        bool an;
        sample_of(nt, sn, rn, an);
        point_of(sn, rn, an, pn);
      }
    }
#pragma unroll
    for (int i = 0; i < 8 * KG; ++i) z[i] = 0.f;
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      loc[l] = compact<float>(locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2],
                                            (act && l == S::NL - 1) ? w.status : nullptr));  // as in the SDF pass
      if (DBG && (w.dbg & 8)) {
#pragma unroll
        for (int c = 0; c < S::CG; ++c) z[l * S::CG + c] = 1e-3f * (float)c + loc[l].fx;
      } else if (l >= S::NL - kJacLevels && S::CG == 4) {
        // the two finest levels keep their spatial Jacobian (this lane's
        // TMEM columns [96, 128), 16 per level, 12 used) so grad phi does
        // not re-read their corners
        float J[16];
        if (STG && l == S::NL - 1) {
          cp_async_wait_all();
          float r[8][S::CG];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 x = stg[k * kTile + tid];
            r[k][0] = x.x;
            r[k][1] = x.y;
            r[k][2] = x.z;
            r[k][3] = x.w;
          }
          jac_from_rows<float, S::CG>(loc[l], r, z + l * S::CG, reinterpret_cast<float(&)[3 * S::CG]>(J));
        } else {
          gather_jac<float, S::CG>(G.lv[l], loc[l], z + l * S::CG, reinterpret_cast<float(&)[3 * S::CG]>(J));
        }
#pragma unroll
        for (int i = 3 * S::CG; i < 16; ++i) J[i] = 0.f;
        st16(tl + kJacCol + 16 * (l - (S::NL - kJacLevels)), J);
      } else {
        gather_fast<float, S::CG>(G.lv[l], loc[l], z + l * S::CG);
      }
    }
    const int cr = ray < 0 ? 0 : ray;  // smoothness points: harmless colour, not stored
    const Loc qc = locate<false>(G.col, (double)p[0], (double)p[1], (double)p[2], nullptr);
#pragma unroll
    for (int i = 0; i < 8 * KC; ++i) inp[i] = 0.f;
    if (DBG && (w.dbg & 8)) {
#pragma unroll
      for (int c = 0; c < S::CC; ++c) inp[c] = 1e-3f * (float)c + (float)qc.fx;
    } else {
      gather_fast<float, S::CC>(G.col, compact<float>(qc), inp);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) inp[S::CC + a] = w.r[cr * 3 + a];
    if constexpr (STG) {
      if (nt < ntiles) stage(pn);
    }
  };
  if constexpr (STG) {
    int64_t s0;
    int r0;
    bool a0;
    sample_of(first, s0, r0, a0);
    float p0[3];
    point_of(s0, r0, a0, p0);
    stage(p0);
  }
  if (first < ntiles) gather(first);
  tc::mbar_wait(&s_bar[0], 0);
  for (int64_t tile = first; tile < ntiles; tile += stride) {
    float h[32];
    uint32_t m0 = 0u;
    // ---- geometry layer 0 / 1 (gs/decoders.py:40-60)
    store_a<KG>(tl, z);
    run([&] { issue_layer<KG>(tmem, sa(U::W0H), sa(U::W0L)); });
    wait_d();
    ld32(tl, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float v = h[n] + gvec[tc::GVec::b0 + n];
      const bool pos = v > 0.f;
      h[n] = pos ? v : 0.f;
      m0 |= (uint32_t)pos << n;
    }
    store_a<4>(tl, h);
    run([&] { issue_layer<4>(tmem, sa(U::W1H), sa(U::W1L)); });
    wait_d();
    ld32(tl, h);
    float phi = gvec[tc::GVec::b2];
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float v = h[n] + gvec[tc::GVec::b1 + n];
      const bool pos = v > 0.f;
      phi = fmaf(pos ? v : 0.f, gvec[tc::GVec::w2 + n], phi);
      h[n] = pos ? gvec[tc::GVec::w2 + n] : 0.f;  // delta1
    }
    // ---- dphi/dz = W0 ((W1 delta1) . m0)
    store_a<4>(tl, h);
    run([&] { issue_layer<4>(tmem, sa(U::W1NH), sa(U::W1NL)); });
    wait_d();
    ld32(tl, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) h[n] = ((m0 >> n) & 1u) ? h[n] : 0.f;
    store_a<4>(tl, h);
    run([&] { issue_layer<4, 16>(tmem, sa(U::W0NH), sa(U::W0NL)); });
    wait_d();
    float gz[16];
    ld16(tl, gz);
    float gr[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      if (DBG && (w.dbg & 72)) continue;
      if (l >= S::NL - kJacLevels && S::CG == 4) {
        float J[16];
        ld16(tl + kJacCol + 16 * (l - (S::NL - kJacLevels)), J);
        level_dx_jac<float, S::CG>(G.lv[l], reinterpret_cast<const float(&)[3 * S::CG]>(J), gz + l * S::CG, gr);
      } else {
        level_dx_fast<float, S::CG>(G.lv[l], loc[l], gz + l * S::CG, gr);
      }
    }
    // ---- colour: sigmoid(MLP_c([f_c, r]))  (gs/decoders.py:86-99)
    if (act && ray >= 0 && w.scolf) {  // the colour features, for the colour backward
#pragma unroll
      for (int c = 0; c < S::CC; c += 2)
        *reinterpret_cast<float2*>(w.scolf + s * S::CC + c) = make_float2(inp[c], inp[c + 1]);
    }
    store_a<KC>(tl, inp);
    run([&] { issue_layer<KC>(tmem, sa(U::C0H), sa(U::C0L)); });
    wait_d();
    ld32(tl, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) h[n] = fmaxf(h[n] + cvec[tc::CVec::b0 + n], 0.f);
    store_a<4>(tl, h);
    run([&] { issue_layer<4>(tmem, sa(U::C1H), sa(U::C1L)); });
    const int64_t cs = s;
    const int cray = ray;
    const bool cact = act;
    if (tile + stride < ntiles) gather(tile + stride);  // overlaps the last MMA
    wait_d();
    ld32(tl, h);
    float y[3] = {cvec[tc::CVec::b2], cvec[tc::CVec::b2 + 1], cvec[tc::CVec::b2 + 2]};
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float v = fmaxf(h[n] + cvec[tc::CVec::b1 + n], 0.f);
#pragma unroll
      for (int c = 0; c < 3; ++c) y[c] = fmaf(v, cvec[tc::CVec::w2 + n * 3 + c], y[c]);
    }
    if (cact) {
      w.sphi[cs] = phi;
#pragma unroll
      for (int a = 0; a < 3; ++a) w.sgphi[cs * 3 + a] = gr[a];
      if (cray >= 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) w.scol[cs * 3 + c] = sigmoid_fast(y[c]);
        if (w.pose_g) {
#pragma unroll
          for (int i = 0; i < S::IN_G; ++i) w.pose_g[cs * S::IN_G + i] = gz[i];
        }
      }
    }
  }
  if constexpr (STG) cp_async_wait_all();
  fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
}


// ---------------------------------------------------------------------------
// geometry backward (same contract as tc::k_bwd_geom_tc): the six
// sample-major layers on tcgen05, two independent layers per commit
//   S1: z W0 -> h0, m0          | v W0 -> q0 = (v W0) . m0
//   S2: h0 W1 -> h1, m1         | q0 W1 -> dd1 = (q0 W1) . m1
//   S3: delta1 W1^T -> delta0 = (.) . m0
//   S4: delta0 W0^T -> dphi/dz (N = 16, stays in TMEM until the scatter)
// column sums (db0, db1, dW2) as warp butterfly reduce-scatters; the
// weight-gradient outer products (contraction over samples) stay on
// mma.sync over the sample-major rows, as in the tc kernel.  256 TMEM
// columns: D0 [0,32), D1 [32,64), A1 hi/lo [64,128), A2 hi/lo [128,192);
// 104 KB shared memory: 2 CTAs per SM (3 CTAs with 128 columns, 5 MMA rounds
// and a 168-register cap measured slower: 432 vs 390 us).  Persistent: a CTA
// loops over tiles and keeps its MLP-gradient sums (outer-product fragments
// in the lanes' spare TMEM columns, column sums in registers) across them
// -- no extra shared memory, so L1 keeps its share for the gathers -- so
// the CTA reduction and
// the L2 reds into the partial rows happen once per CTA instead of once per
// 128-sample tile (GSB_DBG attribution: that per-tile reduction was 47 of
// 376 us).

struct GeoT5 {
  static constexpr int ROW = 104;  // 104 % 32 = 8: fragment loads conflict-free (88 measured slower)
  static constexpr int oA0 = 16, oM = 33, oB0 = 40, oA1 = 72;  // p z + v, m1 bits, delta0, p h0 + q0
  static constexpr int NW = tc::UmmaW::W0NL + 512;              // geometry tiles only
  static constexpr uint32_t kCols2 = 256;
  static constexpr int kCtaPerSm = 2;
  static constexpr uint32_t kAcc = 192;  // TMEM columns [192, 240): the lane's dW0 / dW1 fragment sums
  template <class S>
  static constexpr size_t smem() { return (size_t)(NW + tc::GVec::N) * 4 + (size_t)kTile * ROW * 4; }
};

// running sums of a warp's mma.sync D fragments (tiles of m16n8) kept in the
// lane's own TMEM row: 16 fragment values per call, columns [col, col + 16)
__device__ __forceinline__ void tmem_acc16(uint32_t ta, float (&d)[4][4]) {
  float cur[16];
  ld16(ta, cur);
#pragma unroll
  for (int i = 0; i < 16; ++i) cur[i] += d[i >> 2][i & 3];
  st16(ta, cur);
}
__device__ __forceinline__ void tmem_get16(uint32_t ta, float (&d)[4][4]) {
  float cur[16];
  ld16(ta, cur);
#pragma unroll
  for (int i = 0; i < 16; ++i) d[i >> 2][i & 3] = cur[i];
}

// x (W columns) as tf32 hi / lo to TMEM columns chi / clo of this warp's lanes
template <int W>
__device__ __forceinline__ void store_hl(uint32_t tl, uint32_t chi, uint32_t clo, const float* x) {
  float h[W], l[W];
#pragma unroll
  for (int i = 0; i < W; ++i) split2(x[i], h[i], l[i]);
  if constexpr (W == 8) {
    st8(tl + chi, h);
    st8(tl + clo, l);
  } else if constexpr (W == 16) {
    st16(tl + chi, h);
    st16(tl + clo, l);
  } else {
    static_assert(W == 32, "W");
    st32(tl + chi, h);
    st32(tl + clo, l);
  }
}
template <int KS, uint32_t NN = 32>
__device__ __forceinline__ void issue_at(uint32_t d, uint32_t ahi, uint32_t alo, uint32_t bh, uint32_t bl) {
  constexpr uint32_t sbo = KS * 8 * 32;
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const uint32_t off = kk * 256;
    mma_ts<NN>(d, alo + kk * 8, sdesc(bh + off, 128, sbo), kk > 0 ? 1u : 0u);
    mma_ts<NN>(d, ahi + kk * 8, sdesc(bl + off, 128, sbo), 1u);
    mma_ts<NN>(d, ahi + kk * 8, sdesc(bh + off, 128, sbo), 1u);
  }
}
// column sums over the warp: lane l returns sum over lanes of v[l]
__device__ __forceinline__ float warp_colsum32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = up ? v[i] : v[i + o];
      v[i] = (up ? v[i + o] : v[i]) + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}

template <class S, bool DBG = false>
__global__ void __launch_bounds__(kTile, 2) k_bwd_geom_t5(Ws<float> w, Geo G, int M, int N,
                                                         const double* __restrict__ dep,
                                                         const float* __restrict__ spts, int nsp,
                                                         int agg_levels) {
  using F = tc::Fr<S>;
  using U = tc::UmmaW;
  using K = GeoT5;
  constexpr int KG = F::KG, ROW = K::ROW;
  constexpr int NGP = (S::NG + 3) / 4 * 4;
  static_assert(S::IN_G <= 16 && 8 * KG <= 16, "geometry input width");
  const FastDiv fdn((uint32_t)N);
  extern __shared__ __align__(128) float t5_smem[];
  float* sw = t5_smem;
  const float* gvec = t5_smem + K::NW;
  float* rows_all = t5_smem + K::NW + tc::GVec::N;
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(K::kCols2)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    tc::mbar_init(&s_bar[0]);
    tc::mbar_init(&s_bar[1]);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    constexpr uint32_t wb = K::NW * 4, vb = tc::GVec::N * 4;
    tc::mbar_expect(&s_bar[0], wb + vb);
    tc::bulk_g2s(sw, w.wfrag + tc::kUmmaBaseU4, wb, &s_bar[0]);
    tc::bulk_g2s(t5_smem + K::NW, reinterpret_cast<const float*>(w.wfrag + tc::kVecBase), vb, &s_bar[0]);
  }
  const uint32_t tmem = s_tmem;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  {  // zero the fragment sums (TMEM columns [kAcc, kAcc + 48) of this warp's lanes)
    float zz[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) zz[i] = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) st16(tl + K::kAcc + 16 * j, zz);
  }
  auto sa = [&](int off) { return smem_u32(sw + off); };
  float* rows = rows_all + warp * 32 * ROW;
  float* myrow = rows + lane * ROW;
  const int64_t MN = (int64_t)M * N, NS = MN + nsp;
  const int64_t ntiles = (NS + kTile - 1) / kTile;
  uint32_t phase = 0;
  auto mma_round = [&](auto issue) {
    cta_sync_tmem();
    if (tid == 0) {
      if (!(DBG && (w.dbg & 16))) issue();
      commit(&s_bar[1]);
    }
    tc::mbar_wait(&s_bar[1], phase);
    phase ^= 1u;
    fence_after();
  };
  // column sums (db0, db1, dW2 per lane = column; db2) summed over the tiles
  float sum_b0 = 0.f, sum_b1 = 0.f, sum_w2 = 0.f, sum_p = 0.f;
  bool weights_ready = false;
  // persistent: tiles blockIdx, blockIdx + grid, ... (the sweep maps them
  // last-to-first: the cells the forward touched last are still in L2)
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t tt = (w.sweep & 2) ? ntiles - 1 - tile : tile;
    const int64_t s = tt * kTile + tid;
    const bool active = s < NS;
    __syncwarp();  // the previous tile's outer products are done with this warp's rows
    // ---- per sample: point, z and v in one pass over the corners
    LocT<float> loc[S::NL];
    float p = 0.f, u[3] = {0.f, 0.f, 0.f};
    {
      float pt[3];
      if (active) {
        p = w.pbar[s];
#pragma unroll
        for (int a = 0; a < 3; ++a) u[a] = w.ubar[s * 3 + a];
        if (s < MN) {
          const int ray = (int)fdn.div((uint32_t)s);
          taped_point<float>(w.o + ray * 3, w.r + ray * 3,
                             dep[(int64_t)ray * w.ld + (int)fdn.mod((uint32_t)s, (uint32_t)ray)], G.lo, G.hi, pt);
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
          if (DBG && (w.dbg & 8)) {
#pragma unroll
            for (int c = 0; c < S::CG; ++c) row[c] = 1e-3f * (float)(c + k);
          } else {
            load_row<float, S::CG>(Fp + corner_off(L, k) * S::CG, row);
          }
#pragma unroll
          for (int c = 0; c < S::CG; ++c) {
            z[l * S::CG + c] = fmaf(wk[k], row[c], z[l * S::CG + c]);
            v[l * S::CG + c] = fmaf(ju[k], row[c], v[l * S::CG + c]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 16; i += 2)
        *reinterpret_cast<float2*>(myrow + K::oA0 + i) = make_float2(fmaf(p, z[i], v[i]), fmaf(p, z[i + 1], v[i + 1]));
      store_hl<8 * KG>(tl, 64, 96, z);
      store_hl<8 * KG>(tl, 128, 160, v);
    }
    if (!weights_ready) {
      tc::mbar_wait(&s_bar[0], 0);
      weights_ready = true;
    }
    // S1
    mma_round([&] {
      issue_at<KG>(tmem, tmem + 64, tmem + 96, sa(U::W0H), sa(U::W0L));
      issue_at<KG>(tmem + 32, tmem + 128, tmem + 160, sa(U::W0H), sa(U::W0L));
    });
    float h[32], q[32];
    uint32_t m0 = 0u, m1 = 0u;
    ld32x2(tl, tl + 32, h, q);
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float x = h[n] + gvec[tc::GVec::b0 + n];
      const bool pos = x > 0.f;
      h[n] = pos ? x : 0.f;
      q[n] = pos ? q[n] : 0.f;
      m0 |= (uint32_t)pos << n;
    }
#pragma unroll
    for (int n = 0; n < 32; n += 2)
      *reinterpret_cast<float2*>(myrow + K::oA1 + n) = make_float2(fmaf(p, h[n], q[n]), fmaf(p, h[n + 1], q[n + 1]));
    store_hl<32>(tl, 64, 96, h);
    store_hl<32>(tl, 128, 160, q);
    // S2
    mma_round([&] {
      issue_at<4>(tmem, tmem + 64, tmem + 96, sa(U::W1H), sa(U::W1L));
      issue_at<4>(tmem + 32, tmem + 128, tmem + 160, sa(U::W1H), sa(U::W1L));
    });
    ld32x2(tl, tl + 32, h, q);
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float x = h[n] + gvec[tc::GVec::b1 + n];
      const bool pos = x > 0.f;
      m1 |= (uint32_t)pos << n;
      q[n] = (pos ? p * x : 0.f) + (pos ? q[n] : 0.f);  // dW2: p relu(h1) + dd1
      h[n] = pos ? gvec[tc::GVec::w2 + n] : 0.f;        // delta1
    }
    myrow[K::oM] = __uint_as_float(m1);
    sum_w2 += warp_colsum32(q);
    store_hl<32>(tl, 64, 96, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) h[n] *= p;
    sum_b1 += warp_colsum32(h);
    // S3
    mma_round([&] { issue_at<4>(tmem, tmem + 64, tmem + 96, sa(U::W1NH), sa(U::W1NL)); });
    ld32(tl, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) h[n] = ((m0 >> n) & 1u) ? h[n] : 0.f;
#pragma unroll
    for (int n = 0; n < 32; n += 2) *reinterpret_cast<float2*>(myrow + K::oB0 + n) = make_float2(h[n], h[n + 1]);
    store_hl<32>(tl, 64, 96, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) h[n] *= p;
    sum_b0 += warp_colsum32(h);
    // S4 (dphi/dz to D0 [0, 16)); the outer products overlap it
    cta_sync_tmem();
    if (tid == 0) {
      issue_at<4, 16>(tmem, tmem + 64, tmem + 96, sa(U::W0NH), sa(U::W0NL));
      commit(&s_bar[1]);
    }
    __syncwarp();
    // ---- outer products over the warp's samples: dW0 += A0^T delta0, dW1 += A1^T delta1
    if (!(DBG && (w.dbg & 2))) {
      const int g = lane >> 2, t = lane & 3;
      float d0[1][4][4], d1[2][4][4];
      tc::zero_d(d0);
      tc::zero_d(d1);
      const float w2l = gvec[tc::GVec::w2 + lane];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k0 = ks * 8;
        const uint32_t mk0 = __float_as_uint(rows[(k0 + t) * ROW + K::oM]);
        const uint32_t mk1 = __float_as_uint(rows[(k0 + t + 4) * ROW + K::oM]);
        uint32_t ah[2][4], al[2][4], bh0[4], bh1[4], bl0[4], bl1[4];
        {
          uint32_t a1h[1][4], a1l[1][4];
          frag_a(rows, ROW, K::oA0, k0, 0, a1h[0], a1l[0]);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) frag_b(rows, ROW, K::oB0, k0, nt * 8, bh0[nt], bh1[nt], bl0[nt], bl1[nt]);
          tc::mma3_sweep(d0, a1h, a1l, bh0, bh1, bl0, bl1);
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int n = nt * 8 + g;
          const float w2n = __shfl_sync(0xffffffffu, w2l, n);
          split_fast(((mk0 >> n) & 1u) ? w2n : 0.f, bh0[nt], bl0[nt]);
          split_fast(((mk1 >> n) & 1u) ? w2n : 0.f, bh1[nt], bl1[nt]);
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) frag_a(rows, ROW, K::oA1, k0, mt * 16, ah[mt], al[mt]);
        tc::mma3_sweep(d1, ah, al, bh0, bh1, bl0, bl1);
      }
      // this tile's products into the lane's running sums in TMEM
      tmem_acc16(tl + K::kAcc, d0[0]);
      tmem_acc16(tl + K::kAcc + 16, d1[0]);
      tmem_acc16(tl + K::kAcc + 32, d1[1]);
    }
    float accp = p;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) accp += __shfl_xor_sync(0xffffffffu, accp, o);
    sum_p += accp;
    // ---- grid scatter: theta_l[idx_k] += g_l (p w_k + ju_k)
    tc::mbar_wait(&s_bar[1], phase);
    phase ^= 1u;
    fence_after();
    float gz[16];
    ld16(tl, gz);
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      const LocT<float> lq = loc[l];
      float wk[8], ju[8], coef[8];
      corner_w_ju(lq, (float)G.lv[l].inv_vs, u, wk, ju);
#pragma unroll
      for (int k = 0; k < 8; ++k) coef[k] = fmaf(p, wk[k], ju[k]);
      if (!(DBG && (w.dbg & 1)))
        scatter_level<float, S::CG>(G.lv[l], lq, gz + l * S::CG, coef, active,
                                    (DBG && (w.dbg & 128)) && l == S::NL - 1, w.det_keys,
                                    w.det_vals, s * (S::NL + 1) + l);
    }
  }
  // ---- CTA reduction of the running sums -> MLP partial slot (once per CTA)
  float d0[1][4][4], d1[2][4][4];
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tmem_get16(tl + K::kAcc, d0[0]);
  tmem_get16(tl + K::kAcc + 16, d1[0]);
  tmem_get16(tl + K::kAcc + 32, d1[1]);
  fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(K::kCols2) : "memory");
  if (DBG && (w.dbg & 4)) return;
  float* acc_all = rows_all;  // [4 warps][NGP] over the (now idle) sample rows
  {
    float* acc = acc_all + (size_t)warp * NGP;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) frag_d_store(d0[0][nt], acc + S::oGW0, 0, nt * 8, S::IN_G);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) frag_d_store(d1[mt][nt], acc + S::oGW1, mt * 16, nt * 8, GSB_HID);
    acc[S::oGb0 + lane] = sum_b0;
    acc[S::oGb1 + lane] = sum_b1;
    acc[S::oGW2 + lane] = sum_w2;
    if (lane == 0) acc[S::oGb2] = sum_p;
  }
  __syncthreads();
  const int slot = w.mlp_slots > 0 ? (int)(blockIdx.x % (unsigned)w.mlp_slots) : (int)blockIdx.x;
  float* out = w.mlp_part + (size_t)slot * S::NMLPP;
  for (int i = tid; i < S::NG; i += kTile) {
    float a = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) a += acc_all[(size_t)k * NGP + i];
    if (w.mlp_slots > 0)
      atomicAdd(out + i, a);
    else
      out[i] = a;
  }
}


// ---------------------------------------------------------------------------
// colour backward (same contract as tc::k_bwd_color_tc): the sample-major
// colour layers on tcgen05, one 128-sample tile per CTA
//   R1: [f_c, r] W0c -> h0c, m0
//   R2: h0c W1c -> h1c, m1; 32 -> 3 head, sigmoid, y_bar, a1_bar per lane
//   R3: a1_bar W1c^T -> a0_bar = (.) . m0
//   R4: a0_bar W0c^T (N = 16) -> [f_bar, view-direction cotangent]
// column sums (dW2c, db1c, db2c) as butterflies; the dW0c (+ db0c via the
// ones column) and dW1c outer products stay on mma.sync over the rows.

struct ColT5 {
  static constexpr int ROW = 104;
  static constexpr int oA0 = 0, oB0 = 16, oA1 = 48, oY = 80, oM = 88;
  static constexpr int W0 = tc::UmmaW::C0H, NW = tc::UmmaW::N - tc::UmmaW::C0H;  // colour tiles
  static constexpr int kCtaPerSm = 2;
  static constexpr uint32_t kCols = 256;  // D [0,32), A hi/lo [32,96), fragment sums [96, 144),
  static constexpr uint32_t kAcc = 96;    // dW2c lane partials [144, 240)
  static constexpr uint32_t kW2 = 144;
  template <class S>
  static constexpr size_t smem() { return (size_t)(NW + tc::CVec::N) * 4 + (size_t)kTile * ROW * 4; }
};

template <class S, bool DBG = false>
__global__ void __launch_bounds__(kTile, 2) k_bwd_color_t5(Ws<float> w, Geo G, int M, int N,
                                                          const double* __restrict__ dep) {
  using F = tc::Fr<S>;
  using U = tc::UmmaW;
  using K = ColT5;
  constexpr int KC = F::KC, ROW = K::ROW;
  constexpr int NCP = S::NMLP - S::NG, o = S::NG;
  static_assert(S::IN_C + 1 <= 16 && 8 * KC <= 16 && S::CC <= 8 && S::CC % 2 == 0, "colour input width");
  static_assert(S::oCb0 == S::oCW0 + S::IN_C * GSB_HID, "db0c is the ones row of dW0c");
  const FastDiv fdn((uint32_t)N);
  extern __shared__ __align__(128) float t5_smem[];
  float* sw = t5_smem - K::W0;  // indexed by UmmaW offsets
  const float* cvec = t5_smem + K::NW;
  float* rows_all = t5_smem + K::NW + tc::CVec::N;
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(K::kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    tc::mbar_init(&s_bar[0]);
    tc::mbar_init(&s_bar[1]);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    constexpr uint32_t wb = K::NW * 4, vb = tc::CVec::N * 4;
    tc::mbar_expect(&s_bar[0], wb + vb);
    tc::bulk_g2s(t5_smem, reinterpret_cast<const float*>(w.wfrag + tc::kUmmaBaseU4) + K::W0, wb, &s_bar[0]);
    tc::bulk_g2s(t5_smem + K::NW, reinterpret_cast<const float*>(w.wfrag + tc::kVecBase) + tc::GVec::N, vb,
                 &s_bar[0]);
  }
  const uint32_t tmem = s_tmem;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  {  // zero the fragment sums (TMEM columns [kAcc, kAcc + 48) of this warp's lanes)
    float zz[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) zz[i] = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) st16(tl + K::kAcc + 16 * j, zz);
#pragma unroll
    for (int j = 0; j < 6; ++j) st16(tl + K::kW2 + 16 * j, zz);
  }
  auto sa = [&](int off) { return smem_u32(sw + off); };
  float* rows = rows_all + warp * 32 * ROW;
  float* myrow = rows + lane * ROW;
  const int64_t NS = (int64_t)M * N;
  const int64_t ntiles = (NS + kTile - 1) / kTile;
  uint32_t phase = 0;
  auto mma_round = [&](auto issue) {
    cta_sync_tmem();
    if (tid == 0) {
      if (!(DBG && (w.dbg & 16))) issue();
      commit(&s_bar[1]);
    }
    tc::mbar_wait(&s_bar[1], phase);
    phase ^= 1u;
    fence_after();
  };
  // column sums (dW2c, db1c per lane = column; db2c) summed over the tiles
  float sum_w2[3] = {0.f, 0.f, 0.f}, sum_b1 = 0.f, sum_b2[3] = {0.f, 0.f, 0.f};
  bool weights_ready = false;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t tt = (w.sweep & 4) ? ntiles - 1 - tile : tile;
    const int64_t s = tt * kTile + tid;
    const bool active = s < NS;
    const int ray = active ? (int)fdn.div((uint32_t)s) : 0;
    __syncwarp();  // the previous tile's outer products are done with this warp's rows
    LocT<float> q;
    float cb[3], cc3[3];
    {
      float pt[3];
      taped_point<float>(w.o + ray * 3, w.r + ray * 3,
                         active ? dep[(int64_t)ray * w.ld + (int)fdn.mod((uint32_t)s, (uint32_t)ray)] : 0.0, G.lo, G.hi,
                         pt);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        cb[c] = active ? w.cbar[s * 3 + c] : 0.f;
        // the colour the taped forward stored: sigmoid of the same head
        // (same MMA operands and order, so the same bits as recomputing it)
        cc3[c] = active ? w.scol[s * 3 + c] : 0.f;
      }
      q = compact<float>(locate<false>(G.col, (double)pt[0], (double)pt[1], (double)pt[2], nullptr));
      float inp[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) inp[i] = 0.f;
      if (DBG && (w.dbg & 8)) {
#pragma unroll
        for (int c = 0; c < S::CC; ++c) inp[c] = 1e-3f * (float)c + q.fx;
      } else if (w.scolf) {  // kept by the taped forward (the same gather, bit for bit)
#pragma unroll
        for (int c = 0; c < S::CC; c += 2) {
          const float2 f = active ? *reinterpret_cast<const float2*>(w.scolf + s * S::CC + c)
                                  : make_float2(0.f, 0.f);
          inp[c] = f.x;
          inp[c + 1] = f.y;
        }
      } else {
        gather_fast<float, S::CC>(G.col, q, inp);
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) inp[S::CC + a] = w.r[ray * 3 + a];
      inp[S::IN_C] = 1.f;  // ones column: db0c rides on the dW0c outer product (zero weight row in W0c^T)
#pragma unroll
      for (int i = 0; i < 16; i += 2) *reinterpret_cast<float2*>(myrow + K::oA0 + i) = make_float2(inp[i], inp[i + 1]);
      store_hl<8 * KC>(tl, 32, 64, inp);
    }
    if (!weights_ready) {
      tc::mbar_wait(&s_bar[0], 0);
      weights_ready = true;
    }
    // R1
    mma_round([&] { issue_at<KC>(tmem, tmem + 32, tmem + 64, sa(U::C0H), sa(U::C0L)); });
    float h[32];
    uint32_t m0 = 0u, m1 = 0u;
    ld32(tl, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float x = h[n] + cvec[tc::CVec::b0 + n];
      const bool pos = x > 0.f;
      h[n] = pos ? x : 0.f;
      m0 |= (uint32_t)pos << n;
    }
#pragma unroll
    for (int n = 0; n < 32; n += 2) *reinterpret_cast<float2*>(myrow + K::oA1 + n) = make_float2(h[n], h[n + 1]);
    store_hl<32>(tl, 32, 64, h);
    // R2
    mma_round([&] { issue_at<4>(tmem, tmem + 32, tmem + 64, sa(U::C1H), sa(U::C1L)); });
    ld32(tl, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float x = h[n] + cvec[tc::CVec::b1 + n];
      const bool pos = x > 0.f;
      h[n] = pos ? x : 0.f;
      m1 |= (uint32_t)pos << n;
    }
    float yb[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      yb[c] = cb[c] * (cc3[c] * (1.f - cc3[c]));
      myrow[K::oY + c] = yb[c];
    }
    myrow[K::oM] = __uint_as_float(m1);
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // dW2c[n][c] = sum_s h1c[n] y_bar[c]: the lane's own
      float v[32];                 // running vector in TMEM, reduced over lanes once per CTA
      ld32(tl + K::kW2 + 32 * c, v);
#pragma unroll
      for (int n = 0; n < 32; ++n) v[n] = fmaf(h[n], yb[c], v[n]);
      st32(tl + K::kW2 + 32 * c, v);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float a = yb[c];
#pragma unroll
      for (int sh = 1; sh < 32; sh <<= 1) a += __shfl_xor_sync(0xffffffffu, a, sh);
      sum_b2[c] += a;
    }
    // a1_bar = (y_bar W2c^T) . m1
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float* w2 = cvec + tc::CVec::w2 + n * 3;
      const float v = fmaf(w2[0], yb[0], fmaf(w2[1], yb[1], w2[2] * yb[2]));
      h[n] = ((m1 >> n) & 1u) ? v : 0.f;
    }
    store_hl<32>(tl, 32, 64, h);
    sum_b1 += warp_colsum32(h);
    // R3
    mma_round([&] { issue_at<4>(tmem, tmem + 32, tmem + 64, sa(U::C1NH), sa(U::C1NL)); });
    ld32(tl, h);
#pragma unroll
    for (int n = 0; n < 32; ++n) h[n] = ((m0 >> n) & 1u) ? h[n] : 0.f;
#pragma unroll
    for (int n = 0; n < 32; n += 2) *reinterpret_cast<float2*>(myrow + K::oB0 + n) = make_float2(h[n], h[n + 1]);
    store_hl<32>(tl, 32, 64, h);
    // R4: [f_bar, r_bar] to D [0, 16); the outer products overlap it
    cta_sync_tmem();
    if (tid == 0) {
      issue_at<4, 16>(tmem, tmem + 32, tmem + 64, sa(U::C0NH), sa(U::C0NL));
      commit(&s_bar[1]);
    }
    __syncwarp();
    // ---- outer products over the warp's samples: e0 = [inp,1]^T a0b, e1 = h0c^T a1b
    if (!(DBG && (w.dbg & 2))) {
      const int g = lane >> 2, t = lane & 3;
      float w2c[4][3];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int c = 0; c < 3; ++c) w2c[nt][c] = cvec[tc::CVec::w2 + (8 * nt + g) * 3 + c];
      float e0[1][4][4], e1[2][4][4];
      tc::zero_d(e0);
      tc::zero_d(e1);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k0 = ks * 8;
        uint32_t ah[2][4], al[2][4], bh0[4], bh1[4], bl0[4], bl1[4];
        {
          uint32_t a1h[1][4], a1l[1][4];
          frag_a(rows, ROW, K::oA0, k0, 0, a1h[0], a1l[0]);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) frag_b(rows, ROW, K::oB0, k0, nt * 8, bh0[nt], bh1[nt], bl0[nt], bl1[nt]);
          tc::mma3_sweep(e0, a1h, a1l, bh0, bh1, bl0, bl1);
        }
        {
          const float* r0 = rows + (k0 + t) * ROW;
          const float* r1 = rows + (k0 + t + 4) * ROW;
          const uint32_t mk0 = __float_as_uint(r0[K::oM]);
          const uint32_t mk1 = __float_as_uint(r1[K::oM]);
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
          tc::mma3_sweep(e1, ah, al, bh0, bh1, bl0, bl1);
        }
      }
      // this tile's products into the lane's running sums in TMEM
      tmem_acc16(tl + K::kAcc, e0[0]);
      tmem_acc16(tl + K::kAcc + 16, e1[0]);
      tmem_acc16(tl + K::kAcc + 32, e1[1]);
    }
    // ---- colour grid scatter: theta_c[idx_k] += w_k f_bar
    tc::mbar_wait(&s_bar[1], phase);
    phase ^= 1u;
    fence_after();
    float fb[16];
    ld16(tl, fb);
    {
      float wk[8];
      corner_w(q, wk);
      if (!(DBG && (w.dbg & 1)))
        scatter_level<float, S::CC>(G.col, q, fb, wk, active, false, w.det_keys, w.det_vals,
                                    s * (S::NL + 1) + S::NL);
    }
    if (w.pose_fb && active) {  // pose refinement: f_bar and the view-direction cotangent
      float* po = w.pose_fb + s * 12;
#pragma unroll
      for (int c = 0; c < S::IN_C; ++c) po[c] = fb[c];
    }
  }
  // ---- CTA reduction of the running sums -> MLP partial slot (colour block, once per CTA)
  float e0[1][4][4], e1[2][4][4];
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float v[32];
    ld32(tl + K::kW2 + 32 * c, v);
    sum_w2[c] = warp_colsum32(v);
  }
  tmem_get16(tl + K::kAcc, e0[0]);
  tmem_get16(tl + K::kAcc + 16, e1[0]);
  tmem_get16(tl + K::kAcc + 32, e1[1]);
  fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(K::kCols) : "memory");
  if (DBG && (w.dbg & 4)) return;
  float* acc_all = rows_all;  // [4 warps][NCP] over the (now idle) sample rows
  {
    float* acc = acc_all + (size_t)warp * NCP;
    if (lane < S::oCW0 - S::NG) acc[lane] = 0.f;  // alignment padding
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) frag_d_store(e0[0][nt], acc + (S::oCW0 - o), 0, nt * 8, S::IN_C + 1);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) frag_d_store(e1[mt][nt], acc + (S::oCW1 - o), mt * 16, nt * 8, GSB_HID);
    acc[S::oCb1 - o + lane] = sum_b1;
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[S::oCW2 - o + lane * 3 + c] = sum_w2[c];
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[S::oCb2 - o + c] = sum_b2[c];
    }
  }
  __syncthreads();
  const int slot = w.mlp_slots > 0 ? (int)(blockIdx.x % (unsigned)w.mlp_slots) : (int)blockIdx.x;
  // from the 16-byte aligned colour block start, 4 parameters per vector red
  float* out = w.mlp_part + (size_t)slot * S::NMLPP;
  if (w.mlp_slots == 0 && tid < S::oCW0 - S::NG) out[S::NG + tid] = 0.f;  // per-CTA rows: padding
  for (int i = S::oCW0 + tid * 4; i < S::NMLP; i += kTile * 4) {
    float a[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      a[e] = 0.f;
      if (i + e < S::NMLP) {
#pragma unroll
        for (int k = 0; k < 4; ++k) a[e] += acc_all[(size_t)k * NCP + (i + e - o)];
      }
    }
    if (w.mlp_slots > 0)
      red_add_v4(out + i, a[0], a[1], a[2], a[3]);
    else
      *reinterpret_cast<float4*>(out + i) = make_float4(a[0], a[1], a[2], a[3]);
  }
}

}  // namespace t5
}  // namespace gsb
