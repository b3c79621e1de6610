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

constexpr int kTile = 128;         // samples per CTA = TMEM lanes
constexpr int kCtaPerSm = 4;       // 128 TMEM columns each: 4 x 128 = 512
constexpr uint32_t kCols = 128;

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
// hi = x rounded to tf32 (half away at bit 13); lo = x - hi exact (the tensor
// core reads its top 19 bits)
__device__ __forceinline__ void split2(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
  lo = x - hi;
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
  static constexpr size_t smem() { return (size_t)(tc::UmmaW::N + tc::GVec::N) * 4; }
};

template <class S>
__global__ void __launch_bounds__(kTile) k_sdf_eval_t5(Ws<float> w, Geo G, int M, int Nc,
                                                      const double* __restrict__ dep,
                                                      double* __restrict__ phi,
                                                      const int32_t* __restrict__ list,
                                                      const int32_t* __restrict__ list_count) {
  using F = tc::Fr<S>;
  constexpr int KG = F::KG;
  extern __shared__ __align__(128) float t5_smem[];
  float* sw = t5_smem;                 // UmmaW block
  float* svec = t5_smem + tc::UmmaW::N;  // GVec block
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
    constexpr uint32_t wb = tc::UmmaW::N * 4, vb = tc::GVec::N * 4;
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
        ray = (int)((uint32_t)s / (uint32_t)Nc);
        slot = (int)((uint32_t)s % (uint32_t)Nc);
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
      const Loc q = locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2], act ? w.status : nullptr);
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

struct FwdT5 {
  static constexpr size_t smem() { return (size_t)(tc::UmmaW::N + tc::GVec::N + tc::CVec::N) * 4; }
};

template <class S, int CPS>
__global__ void __launch_bounds__(kTile, CPS) k_fwd_t5(Ws<float> w, Geo G, int M, int N,
                                                 const double* __restrict__ dep,
                                                 const float* __restrict__ spts, int nsp) {
  using F = tc::Fr<S>;
  using U = tc::UmmaW;
  constexpr int KG = F::KG, KC = F::KC;
  static_assert(8 * KG <= 16 && 8 * KC <= 16, "input widths");
  extern __shared__ __align__(128) float t5_smem[];
  float* sw = t5_smem;
  const float* gvec = t5_smem + U::N;
  const float* cvec = gvec + tc::GVec::N;
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ uint32_t s_tmem;
  const int64_t MN = (int64_t)M * N, NS = MN + nsp;
  const int64_t ntiles = (NS + kTile - 1) / kTile;
  if ((int64_t)blockIdx.x >= ntiles) return;
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
    constexpr uint32_t wb = U::N * 4, vb = (tc::GVec::N + tc::CVec::N) * 4;
    tc::mbar_expect(&s_bar[0], wb + vb);
    tc::bulk_g2s(sw, w.wfrag + tc::kUmmaBaseU4, wb, &s_bar[0]);
    tc::bulk_g2s(t5_smem + U::N, reinterpret_cast<const float*>(w.wfrag + tc::kVecBase), vb, &s_bar[0]);
  }
  const uint32_t tmem = s_tmem;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  auto sa = [&](int off) { return smem_u32(sw + off); };
  uint32_t phase = 0;
  auto run = [&](auto issue) {  // all lanes' A stores -> one thread issues -> wait for D
    cta_sync_tmem();
    if (tid == 0) {
      issue();
      commit(&s_bar[1]);
    }
  };
  auto wait_d = [&]() {
    tc::mbar_wait(&s_bar[1], phase);
    phase ^= 1u;
    fence_after();
  };
  // lane-per-sample inputs of one tile
  int64_t s;
  int ray;
  bool act;
  LocT<float> loc[S::NL];
  float z[8 * KG], inp[8 * KC];
  auto gather = [&](int64_t tile) {
    s = tile * kTile + tid;
    act = s < NS;
    ray = -1;
    float p[3];
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
#pragma unroll
    for (int i = 0; i < 8 * KG; ++i) z[i] = 0.f;
#pragma unroll
    for (int l = 0; l < S::NL; ++l) {
      loc[l] = compact<float>(locate<false>(G.lv[l], (double)p[0], (double)p[1], (double)p[2],
                                            act ? w.status : nullptr));
      gather_fast<float, S::CG>(G.lv[l], loc[l], z + l * S::CG);
    }
    const int cr = ray < 0 ? 0 : ray;  // smoothness points: harmless colour, not stored
    const Loc qc = locate<false>(G.col, (double)p[0], (double)p[1], (double)p[2], nullptr);
#pragma unroll
    for (int i = 0; i < 8 * KC; ++i) inp[i] = 0.f;
    gather_fast<float, S::CC>(G.col, compact<float>(qc), inp);
#pragma unroll
    for (int a = 0; a < 3; ++a) inp[S::CC + a] = w.r[cr * 3 + a];
  };
  gather(blockIdx.x);
  tc::mbar_wait(&s_bar[0], 0);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
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
    for (int l = 0; l < S::NL; ++l) level_dx_fast<float, S::CG>(G.lv[l], loc[l], gz + l * S::CG, gr);
    // ---- colour: sigmoid(MLP_c([f_c, r]))  (gs/decoders.py:86-99)
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
    if (tile + gridDim.x < ntiles) gather(tile + gridDim.x);  // overlaps the last MMA
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
  fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
}

}  // namespace t5
}  // namespace gsb
