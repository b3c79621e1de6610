// gsb_step.cuh -- one training step (objective + backward) for one (T, Shape).
#pragma once

#include "gsb_host.cuh"
#include "gsb_tc.cuh"
#include "gsb_t5.cuh"
#include "gsb_pose.cuh"

#include <cub/cub.cuh>

#include <cstdlib>

#define GSB_CHECK(x)                           \
  do {                                         \
    cudaError_t e__ = (x);                     \
    if (e__ != cudaSuccess) return GSB_E_CUDA; \
  } while (0)
#define GSB_LAUNCHED()         \
  do {                         \
    gsb::host::note_launch(); \
    GSB_CHECK(cudaGetLastError()); \
  } while (0)

#define GSB_LAUNCHED_T(name)                  \
  do {                                        \
    GSB_LAUNCHED();                           \
    gsb::host::timing_point(name, stream);    \
  } while (0)

namespace gsb {

// no-grad SDF kernel form (A/B runs): GSB_T5=0 mma.sync everywhere, 1 tcgen05
// everywhere, 2 (default, measured best) tcgen05 for the coarse pass (590 k samples,
// ~10 tiles per persistent CTA) and mma.sync for the 74 k-sample importance passes
inline int t5_mode() {
  static const int v = [] {
    const char* e = std::getenv("GSB_T5");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}
inline bool use_t5(bool coarse = true) { return t5_mode() == 1 || (t5_mode() == 2 && coarse); }
// taped forward form: GSB_T5_FWD=0 mma.sync (tc::k_fwd_tc); > 0 tcgen05
// (t5::k_fwd_t5, 4 CTAs per SM, register cap 128); 3: 3 CTAs per SM, 170
// registers (A/B, measured slower: 196 vs 181 us); 5: finest-level corners
// staged in shared memory with cp.async one tile ahead (A/B, measured
// slower: 221 vs 182 us -- the 4 x 56 KB carve-out leaves L1 28 KB for the
// coarse-level gathers).
// geometry backward form: GSB_T5_BWD=1 (default) tcgen05 (t5::k_bwd_geom_t5), 0 mma.sync
inline bool use_t5_bwd() {
  static const bool v = [] {
    const char* e = std::getenv("GSB_T5_BWD");
    return e ? std::atoi(e) != 0 : true;
  }();
  return v;
}
// colour backward form: GSB_T5_COL=1 (default) tcgen05 (t5::k_bwd_color_t5), 0 mma.sync
inline bool use_t5_col() {
  static const bool v = [] {
    const char* e = std::getenv("GSB_T5_COL");
    return e ? std::atoi(e) != 0 : true;
  }();
  return v;
}
inline int t5_fwd_mode() {
  static const int v = [] {
    const char* e = std::getenv("GSB_T5_FWD");
    return e ? std::atoi(e) : 4;
  }();
  return v;
}
inline int sm_count() {
  static const int v = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return v;
}
// deterministic scatter scratch: entries (sample slot, level, corner)
struct DetLayout {
  int64_t n;
  size_t keys_in, keys_out, idx_in, idx_out, vals, temp, temp_bytes, total;
};
template <typename T>
inline DetLayout det_layout(const host::Sizes& z, int nl) {
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  DetLayout L;
  L.n = ((int64_t)z.NS + 64) * (nl + 1) * 8;
  size_t o = 0;
  L.keys_in = o;
  o = up(o + (size_t)L.n * 8);
  L.keys_out = o;
  o = up(o + (size_t)L.n * 8);
  L.idx_in = o;
  o = up(o + (size_t)L.n * 4);
  L.idx_out = o;
  o = up(o + (size_t)L.n * 4);
  L.vals = o;
  o = up(o + (size_t)L.n * 8 * sizeof(T));
  L.temp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, L.temp_bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)L.n);
  L.temp = o;
  o = up(o + L.temp_bytes);
  L.total = o;
  return L;
}

// lanes per ray of the importance rounds (GSB_IMP_G: 8, 16 or 32).  Measured
// at config 2 (three rounds per step): 32 -> 116 us, 16 -> 108.5 us, 8 -> 134 us
inline int imp_group() {
  static const int v = [] {
    const char* e = std::getenv("GSB_IMP_G");
    const int g = e ? std::atoi(e) : 16;
    return (g == 8 || g == 32) ? g : 16;
  }();
  return v;
}
template <typename T>
inline cudaError_t launch_importance(int G, Ws<T> w, int M, int K, int A, int ray_base, const double* dep,
                                     const double* phi, double* dep_out, double* phi_out, const T* log_s,
                                     gsb_pcg64_t rng, int want_list, int count_final, double trunc,
                                     const uint64_t* row_states, int32_t* evl_count, cudaStream_t stream) {
  const int rpb = 128 / G;
  const size_t smem = (size_t)rpb * imp_row_bytes(K + A, A);
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(M + rpb - 1) / rpb, 128, smem, stream>>>(w, M, K, A, ray_base, dep, phi, dep_out, phi_out, log_s,
                                                      rng, w.evl, evl_count, w.evl_cap, want_list,
                                                      count_final, trunc, row_states);
    return cudaGetLastError();
  };
  if (G == 8) return go(k_importance_dev<T, 8>);
  if (G == 16) return go(k_importance_dev<T, 16>);
  return go(k_importance_dev<T, 32>);
}

// persistent tcgen05 SDF evaluation over `cap` (upper bound of) samples
template <class S>
inline cudaError_t launch_sdf_t5(Ws<float> w, Geo G, int M, int Nc, const double* dep, double* phi,
                                 const int32_t* list, const int32_t* list_count, int64_t cap,
                                 cudaStream_t stream) {
  const int64_t tiles = (cap + t5::kTile - 1) / t5::kTile;
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count() * t5::kCtaPerSm);
  if (grid <= 0) return cudaSuccess;
  t5::k_sdf_eval_t5<S><<<grid, t5::kTile, t5::SdfT5::smem(), stream>>>(w, G, M, Nc, dep, phi, list,
                                                                        list_count);
  return cudaGetLastError();
}

// float32 step start: ray setup (blocks [0, nrb)) and the decoder weight
// tiles / fragments (k_wfrag's blocks after them) in one launch
template <typename T, class S>
__global__ void __launch_bounds__(128) k_setup(gsb_dataset_t D, const int64_t* __restrict__ ids, int M,
                                               int ray_base, Ws<T> w, Geo G, int Nc, double nearv,
                                               double max_depth, int has_ff, double ff, gsb_pcg64_t rng,
                                               PcgRounds imp, int nfin, int nrb, const float* __restrict__ mlp) {
  if ((int)blockIdx.x < nrb)
    ray_setup_block<T>(D, ids, M, ray_base, w, G, Nc, nearv, max_depth, has_ff, ff, rng, imp, blockIdx.x, nfin);
  else
    tc::wfrag_block<S>(mlp, w.wfrag, (int)blockIdx.x - nrb);
}

namespace host {

template <typename T, class S>
int run_step(const gsb_model_t* model, const gsb_dataset_t* data, const gsb_step_t* st,
             cudaStream_t stream) {
  const size_t esz = sizeof(T);
  timing_point(nullptr, stream);
  Sizes z = sizes_of(model, st->n_rays, st->n_coarse, st->n_rounds, st->n_add, st->n_smooth);
  if (S::NMLP != z.nmlp) return GSB_E_ARG;
  size_t need = 0;
  Ws<T> w = carve<T>(st->workspace, z, &need);
  if (need > st->workspace_bytes) return GSB_E_ARG;
  // the colour backward reads the colour features the taped forward kept
  // only when both are the tcgen05 kernels (the A/B forms re-gather)
  if (!(sizeof(T) == 4 && t5_fwd_mode() > 0 && use_t5_col())) w.scolf = nullptr;
  Geo G = geo_of(model, esz);
  T* params = reinterpret_cast<T*>(model->params);
  T* grads = reinterpret_cast<T*>(model->grads);
  const T* mlp = params + model->mlp_offset;  // staged into shared memory by each CTA
  constexpr bool F32 = sizeof(T) == 4;  // float32: decoders on the tensor cores (gsb_tc.cuh)
  constexpr int TW = 4;                  // warps per CTA of the float32 sample kernels
  const float* mlp32 = reinterpret_cast<const float*>(mlp);
  DetLayout DL{};
  if (st->det_work && (st->phases & 2)) {  // deterministic scatter: entries instead of atomics
    DL = det_layout<T>(z, S::NL);
    if (DL.total > st->det_work_bytes || DL.n > INT32_MAX) return GSB_E_ARG;
    unsigned char* db = reinterpret_cast<unsigned char*>(st->det_work);
    w.det_keys = reinterpret_cast<uint64_t*>(db + DL.keys_in);
    w.det_vals = reinterpret_cast<T*>(db + DL.vals);
  }
  if constexpr (F32) {
    if (st->pose_work) {  // pose refinement: keep dphi/dz and colour-input cotangents
      const PoseLayout PL = pose_layout<T>(z, S::IN_G);
      if (PL.total > st->pose_work_bytes) return GSB_E_ARG;
      unsigned char* sc = reinterpret_cast<unsigned char*>(st->pose_work);
      w.pose_g = reinterpret_cast<T*>(sc + PL.g);
      w.pose_fb = reinterpret_cast<T*>(sc + PL.fb);
    }
    static_assert(tc::kFragBufU4 == 4096 + 68 + 3072, "workspace carve");
    if (!(st->phases & 1)) {  // otherwise k_setup builds them with the rays
      tc::k_wfrag<S><<<tc::wfrag_blocks<S>(), 128, 0, stream>>>(mlp32, w.wfrag);
      GSB_LAUNCHED_T("k_wfrag");
    }
  }
  const size_t smem_sdf = (size_t)S::NG * esz;
  const size_t smem_fwd = ((size_t)(S::NMLP + 3) / 4 * 4 + 128 * FwdRow<T, S>::ROW) * esz;
  const int M = z.M, N = z.N, Nc = st->n_coarse, A = st->n_add, R = st->n_rounds;
  const int nsp = 2 * z.S;
  double* dep_final = w.dep[R % 2];
  const T* log_s = params + model->log_s_offset;
  if (st->phases & 1) {
    PcgRounds imp{};
    imp.n = R;
    imp.A = A;
    for (int r = 0; r < R; ++r) imp.r[r] = st->rng_importance[r];
    const int nrb = (M + kRaySetupRays - 1) / kRaySetupRays, nfin = (S::NMLP + 31) / 32;
    if constexpr (F32) {
      k_setup<T, S><<<nrb + tc::wfrag_blocks<S>(), 128, 0, stream>>>(
          *data, st->ray_ids, M, st->ray_base, w, G, Nc, st->near, st->max_depth, st->has_fixed_far,
          st->fixed_far, st->rng_stratify, imp, nfin, nrb, mlp32);
    } else {
      k_ray_setup<T><<<nrb, 128, 0, stream>>>(*data, st->ray_ids, M, st->ray_base, w, G, Nc, st->near,
                                              st->max_depth, st->has_fixed_far, st->fixed_far,
                                              st->rng_stratify, imp, nfin);
    }
    GSB_LAUNCHED_T("k_ray_setup");
    if (R > 0) {
      int64_t n0 = (int64_t)M * Nc;
      int blocks = (int)((n0 + 127) / 128);
      if constexpr (F32) {
        if (use_t5()) {
          GSB_CHECK(launch_sdf_t5<S>(w, G, M, Nc, w.dep[0], w.phi[0], nullptr, nullptr, n0, stream));
        } else {
          GSB_CHECK(cudaFuncSetAttribute(tc::k_sdf_eval_tc<S, TW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tc::SdfTc<S, TW>::smem()));
          tc::k_sdf_eval_tc<S, TW><<<blocks, TW * 32, tc::SdfTc<S, TW>::smem(), stream>>>(
              w, G, M, Nc, mlp32, w.dep[0], w.phi[0], nullptr, nullptr);
        }
      } else
        k_sdf_eval<T, S, false><<<blocks, 128, smem_sdf, stream>>>(w, G, M, Nc, w.dep[0],
                                                                   w.phi[0], nullptr, nullptr, mlp);
      GSB_LAUNCHED_T("k_sdf_eval");
      int cur = 0, K = Nc;
      for (int rnd = 0; rnd < R; ++rnd) {
        const bool need_phi = rnd < R - 1;
        int32_t* evl_n = w.evl_count + rnd;  // zeroed by k_ray_setup
        GSB_CHECK(launch_importance<T>(imp_group(), w, M, K, A, st->ray_base, w.dep[cur], w.phi[cur],
                                       w.dep[1 - cur], w.phi[1 - cur], log_s, st->rng_importance[rnd],
                                       need_phi ? 1 : 0, rnd == R - 1 ? 1 : 0, st->truncation,
                                       w.imp_state + (int64_t)rnd * M * 2, evl_n, stream));
        GSB_LAUNCHED_T("k_importance_dev");
        if (need_phi) {
          int64_t cap = (int64_t)M * A;
          int b2 = (int)((cap + 127) / 128);
          if constexpr (F32) {
            if (use_t5(false))
              GSB_CHECK(launch_sdf_t5<S>(w, G, M, Nc, w.dep[1 - cur], w.phi[1 - cur], w.evl, evl_n,
                                         cap, stream));
            else
              tc::k_sdf_eval_tc<S, TW><<<b2, TW * 32, tc::SdfTc<S, TW>::smem(), stream>>>(
                  w, G, M, Nc, mlp32, w.dep[1 - cur], w.phi[1 - cur], w.evl, evl_n);
          } else
            k_sdf_eval<T, S, false><<<b2, 128, smem_sdf, stream>>>(
                w, G, M, Nc, w.dep[1 - cur], w.phi[1 - cur], w.evl, evl_n, mlp);
          GSB_LAUNCHED_T("k_sdf_eval");
        }
        cur = 1 - cur;
        K += A;
      }
    }
    if (R == 0) {  // otherwise counted by the last importance round
      k_counts<T><<<(M + 127) / 128, 128, 0, stream>>>(w, M, N, dep_final, st->truncation);
      GSB_LAUNCHED_T("k_counts");
    }
  }
  if (st->phases & 2) {
    // bit 2 / bit 3 split the backward phase for communication overlap: part A
    // = taped forward, render, geometry backward (the geometry grids' grads are
    // final after it); part B = colour backward and the finalize kernels
    const bool runA = (st->phases & 12) != 8, runB = (st->phases & 12) != 4;
    const T* spts = reinterpret_cast<const T*>(st->smooth_pts);
    int64_t ns = z.NS;
    int fb = (int)((ns + 127) / 128);
    // tile sweep directions (Ws::sweep, GSB_SWEEP): the geometry backward runs
    // its tiles last-to-first, so it starts on the grid cells the forward
    // touched last (still in L2): 372 -> 369 us; the other bits measured neutral
    static const int kSweep = [] {
      const char* e = std::getenv("GSB_SWEEP");
      return e ? std::atoi(e) : 2;
    }();
    w.sweep = kSweep;
    static const int kDbg = [] {
      const char* e = std::getenv("GSB_DBG");
      return e ? std::atoi(e) : 0;
    }();
    w.dbg = kDbg;
    if (runA) {
    if constexpr (F32) {
      constexpr int FW = 4;  // warps per CTA of the taped forward
      if (const int cps = t5_fwd_mode(); cps > 0) {
        // 4 CTAs per SM (128 registers) by default; GSB_T5_FWD=3: 3 CTAs, 170 registers (A/B)
        const int64_t tiles = (ns + t5::kTile - 1) / t5::kTile;
        const int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count() * (cps == 3 ? 3 : t5::kCtaPerSm));
        if (grid > 0) {
          bool staged = false;
          if constexpr (S::CG == 4 && S::NL >= 2) {
            if (cps == 5) {
              GSB_CHECK(cudaFuncSetAttribute(t5::k_fwd_t5<S, t5::kCtaPerSm, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)t5::FwdT5::smem(true)));
              t5::k_fwd_t5<S, t5::kCtaPerSm, true>
                  <<<grid, t5::kTile, t5::FwdT5::smem(true), stream>>>(w, G, M, N, dep_final, spts, nsp);
              staged = true;
            }
          }
          if (staged) {
          } else if (cps == 3) {
            t5::k_fwd_t5<S, 3><<<grid, t5::kTile, t5::FwdT5::smem(), stream>>>(w, G, M, N, dep_final, spts, nsp);
          } else if (w.dbg) {  // GSB_DBG attribution knobs (measurement only)
            t5::k_fwd_t5<S, t5::kCtaPerSm, false, true>
                <<<grid, t5::kTile, t5::FwdT5::smem(), stream>>>(w, G, M, N, dep_final, spts, nsp);
          } else {
            t5::k_fwd_t5<S><<<grid, t5::kTile, t5::FwdT5::smem(), stream>>>(w, G, M, N, dep_final, spts, nsp);
          }
        }
      } else {
        GSB_CHECK(cudaFuncSetAttribute(tc::k_fwd_tc<S, FW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)tc::FwdTc<S, FW>::smem()));
        tc::k_fwd_tc<S, FW><<<(int)((ns + FW * 32 - 1) / (FW * 32)), FW * 32, tc::FwdTc<S, FW>::smem(),
                              stream>>>(w, G, M, N, mlp32, dep_final, spts, nsp);
      }
    } else {
      GSB_CHECK(cudaFuncSetAttribute(k_fwd<T, S, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fwd));
      k_fwd<T, S, false><<<fb, 128, smem_fwd, stream>>>(w, G, M, N, dep_final, spts, nsp, mlp);
    }
    GSB_LAUNCHED_T("k_fwd");
    }
    LossW L;
    L.rgb = st->w_rgb;
    L.depth = st->w_depth;
    L.sdf = st->w_sdf;
    L.fs = st->w_fs;
    L.eik = st->w_eik;
    L.smooth = st->w_smooth;
    L.trunc = st->truncation;
    L.alpha = st->fs_alpha;
    L.m_global = st->m_global;
    L.smooth_global = st->smooth_global;
    if (runA) {
      // the smoothness pairs ride in k_render's trailing blocks
      const size_t smem_render = (size_t)4 * kRenderRows * N * esz;
      GSB_CHECK(cudaFuncSetAttribute(k_render<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_render));
      k_render<T><<<(M + 3) / 4 + (z.S + 127) / 128, 128, smem_render, stream>>>(
          w, M, N, dep_final, params, model->log_s_offset, L, z.S, z.MN);
      GSB_LAUNCHED_T("k_render");
      if (w.det_keys)  // every slot starts empty (~0 sorts last and is skipped)
        GSB_CHECK(cudaMemsetAsync(w.det_keys, 0xff, (size_t)DL.n * 8, stream));
    }
    // backward kernels: persistent grids
    constexpr int WG = sizeof(T) == 4 ? 4 : 2;
    const int per_cta = WG * 32;
    int nb_geo = (int)std::min<int64_t>((ns + per_cta - 1) / per_cta, (int64_t)num_sms() * 2);
    int nb_col = (int)std::min<int64_t>((z.MN + per_cta - 1) / per_cta, (int64_t)num_sms() * 2);
    nb_geo = std::max(1, std::min(nb_geo, kNbMax));
    nb_col = std::max(1, std::min(nb_col, kNbMax));
    if constexpr (F32) {
      constexpr int WGEO = 4;  // one 32-sample batch per warp
      nb_geo = (int)((ns + WGEO * 32 - 1) / (WGEO * 32));
      nb_col = (int)((z.MN + per_cta - 1) / per_cta);
      const size_t smem_g = tc::GeoTc<S, WGEO>::smem();
      constexpr int WCOL = 4;  // 2 x 4 warps beat 2 x 6 (322 vs 367 us): L1 for the gathers
      nb_col = (int)((z.MN + WCOL * 32 - 1) / (WCOL * 32));
      const size_t smem_c = tc::ColTc<S, WCOL>::smem();
      GSB_CHECK(cudaFuncSetAttribute(tc::k_bwd_geom_tc<S, WGEO>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_g));
      GSB_CHECK(cudaFuncSetAttribute(tc::k_bwd_color_tc<S, WCOL>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c));
      // MLP partials: red.add into kMlpSlots L2-resident rows instead of one row per CTA
      static const int kMlpSlots = [] {
        const char* e = std::getenv("GSB_MLP_SLOTS");
        const int v = e ? std::atoi(e) : 64;
        return v < 1 ? 1 : (v > kNbMax ? kNbMax : v);
      }();
      w.mlp_slots = w.det_keys ? 0 : kMlpSlots;  // deterministic mode: per-CTA rows
      if (use_t5_bwd())  // persistent: two CTAs per SM loop over the 128-sample tiles
        nb_geo = (int)std::min<int64_t>((ns + t5::kTile - 1) / t5::kTile,
                                        (int64_t)sm_count() * t5::GeoT5::kCtaPerSm);
      if (use_t5_col())
        nb_col = (int)std::min<int64_t>((z.MN + t5::kTile - 1) / t5::kTile,
                                        (int64_t)sm_count() * t5::ColT5::kCtaPerSm);
      if (runA) {
        if (w.mlp_slots)
          GSB_CHECK(cudaMemsetAsync(w.mlp_part, 0, (size_t)kMlpSlots * S::NMLPP * sizeof(T), stream));
        if (use_t5_bwd()) {
          const size_t smem_t5 = t5::GeoT5::smem<S>();
          // the runtime-knob instantiation in production too: without the
          // knob branches the compiler schedules the gather differently (255
          // vs 236 registers) and the kernel measured slower, 311 vs 297 us
          auto kern = t5::k_bwd_geom_t5<S, true>;
          GSB_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t5));
          kern<<<nb_geo, t5::kTile, smem_t5, stream>>>(w, G, M, N, dep_final, spts, nsp, 2);
        } else {
          tc::k_bwd_geom_tc<S, WGEO><<<nb_geo, WGEO * 32, smem_g, stream>>>(w, G, M, N, mlp32,
                                                                            dep_final, spts, nsp, 2);
        }
        GSB_LAUNCHED_T("k_bwd_geom");
      }
      if (runB) {
        if (use_t5_col()) {
          const size_t smem_t5 = t5::ColT5::smem<S>();
          auto kern = w.dbg ? t5::k_bwd_color_t5<S, true> : t5::k_bwd_color_t5<S>;
          GSB_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t5));
          kern<<<nb_col, t5::kTile, smem_t5, stream>>>(w, G, M, N, dep_final);
        } else {
          tc::k_bwd_color_tc<S, WCOL><<<nb_col, WCOL * 32, smem_c, stream>>>(w, G, M, N, mlp32, dep_final);
        }
        GSB_LAUNCHED_T("k_bwd_color");
      }
      if (w.mlp_slots) {
        nb_geo = std::min(nb_geo, kMlpSlots);
        nb_col = std::min(nb_col, kMlpSlots);
      }
    } else {
      constexpr int CW = S::NMLP - S::oCW0;
      size_t smem_g = ((size_t)(S::NG + 3) / 4 * 4 + (size_t)WG * 32 * GeoRow<T, S>::ROW) * esz;
      size_t smem_c = ((size_t)(CW + 3) / 4 * 4 + (size_t)WG * 32 * ColRow<T, S>::ROW) * esz;
      GSB_CHECK(cudaFuncSetAttribute(k_bwd_geom<T, S, WG>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_g));
      GSB_CHECK(cudaFuncSetAttribute(k_bwd_color<T, S, WG>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c));
      if (runA) {
        k_bwd_geom<T, S, WG><<<nb_geo, per_cta, smem_g, stream>>>(w, G, M, N, dep_final, spts, nsp,
                                                                 2, mlp);
        GSB_LAUNCHED_T("k_bwd_geom");
      }
      if (runB) {
        k_bwd_color<T, S, WG><<<nb_col, per_cta, smem_c, stream>>>(w, G, M, N, dep_final, mlp);
        GSB_LAUNCHED_T("k_bwd_color");
      }
    }
    if (!runB) return GSB_OK;  // part A only: the caller overlaps the geometry-grid exchange
    if (w.det_keys) {  // stable sort by grad row, then per-row sums in (sample, level, corner) order
      unsigned char* db = reinterpret_cast<unsigned char*>(st->det_work);
      int32_t* idx_in = reinterpret_cast<int32_t*>(db + DL.idx_in);
      int32_t* idx_out = reinterpret_cast<int32_t*>(db + DL.idx_out);
      uint64_t* keys_out = reinterpret_cast<uint64_t*>(db + DL.keys_out);
      const int nb = (int)((DL.n + 255) / 256);
      k_det_iota<<<nb, 256, 0, stream>>>(idx_in, DL.n);
      GSB_LAUNCHED_T("k_det_iota");
      size_t tb = DL.temp_bytes;
      GSB_CHECK(cub::DeviceRadixSort::SortPairs(db + DL.temp, tb, w.det_keys, keys_out, idx_in, idx_out,
                                                (int)DL.n, 0, 64, stream));
      GSB_LAUNCHED_T("cub_radix_sort");
      const uintptr_t col_lo = reinterpret_cast<uintptr_t>(G.col.grad);
      const uintptr_t col_hi = col_lo + (uintptr_t)G.col.nx * G.col.ny * G.col.nz * G.col.C * sizeof(T);
      k_det_reduce<T><<<nb, 256, 0, stream>>>(keys_out, idx_out, w.det_vals, DL.n, S::CG, S::CC, col_lo, col_hi);
      GSB_LAUNCHED_T("k_det_reduce");
    }
    static_assert(FIN_SPLIT == 16, "workspace carve");
    const int nloss = (std::max(M, z.S) + 255) / 256;
    // MLP-partial reduction and loss reduction in one launch
    if (nb_geo <= 256 && nb_col <= 256) {  // few (slot) rows: one pass, 8 warps per 32 parameters
      k_finalize<T, S, false><<<(S::NMLP + 31) / 32 + nloss, 256, 0, stream>>>(
          w, grads, model->mlp_offset, nb_geo, nb_col, M, z.S, params, model->log_s_offset, L, nloss);
    } else {
      // tickets: zeroed by the step's ray setup, and each launch leaves them zero
      if (!(st->phases & 1))
        GSB_CHECK(cudaMemsetAsync(w.fin_cnt, 0, (S::NMLP + 31) / 32 * sizeof(unsigned), stream));
      k_finalize<T, S, true><<<(S::NMLP + 31) / 32 * FIN_SPLIT + nloss, 256, 0, stream>>>(
          w, grads, model->mlp_offset, nb_geo, nb_col, M, z.S, params, model->log_s_offset, L, nloss);
    }
    GSB_LAUNCHED_T("k_finalize");
  }
  return GSB_OK;
}

// ---------------------------------------------------------------------------
// geometry-only evaluation / fit on point lists: the sphere pre-fit
// (decoders.geometric_init, gs/decoders.py:102-177) and dense SDF queries.
// They reuse the taped kernels with zero rays: every sample is a "point"
// sample (the smoothness-point path), so phi is exactly the step's phi.

template <typename T>
Ws<T> carve_sdf(void* ws, int64_t n, int nmlp, size_t* bytes, bool grad = true) {
  Carver<T> c;
  c.base = reinterpret_cast<unsigned char*>(ws);
  Ws<T> w{};
  w.ld = 1;
  w.status = c.template take<int32_t>(GSB_N_STATUS);
  w.parts = c.template take<double>(16);       // [0]: fit loss
  w.o = c.template take<T>(4);                 // dummy ray for the (unused) colour branch
  w.r = c.template take<T>(4);
  w.sphi = c.template take<T>(n);
  w.sgphi = c.template take<T>(n * 3);
  w.pbar = c.template take<T>(grad ? n : 1);
  w.ubar = c.template take<T>(grad ? n * 3 : 1);
  const int64_t nb = grad ? std::max<int64_t>(kNbMax, (n + 127) / 128) : 1;
  w.nb_max = (int)nb;
  w.mlp_part = c.template take<T>(nb * ((nmlp + 3) / 4 * 4));
  w.wfrag = c.template take<uint4>(4096 + 68 + 3072);
  w.fin_red = c.template take<double>((int64_t)16 * nmlp);
  w.fin_cnt = c.template take<unsigned>((nmlp + 31) / 32);
  if (bytes) *bytes = c.off;
  return w;
}

// p_bar = d/dphi [mean_batch (phi - t)^2 + mean_anchor (phi - t)^2] with the
// reference's vjp arithmetic: g = 1/n, then g*err + g*err (gs/diffcore.py:354-572)
template <typename T>
__global__ void k_fit_seed(Ws<T> w, const T* __restrict__ target, int64_t nb, int64_t na) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nb + na) return;
  const T inv = T(1) / (T)(i < nb ? nb : na);
  const T err = w.sphi[i] - target[i];
  const T g = inv * err;
  w.pbar[i] = g + g;
#pragma unroll
  for (int a = 0; a < 3; ++a) w.ubar[i * 3 + a] = T(0);
  atomicAdd(&w.parts[0], (double)(err * err) * (double)inv);
}

template <typename T, class S>
int sdf_forward(const gsb_model_t* model, Ws<T>& w, const T* pts, int64_t n, cudaStream_t stream) {
  const size_t esz = sizeof(T);
  Geo G = geo_of(model, esz);
  const T* mlp = reinterpret_cast<const T*>(model->params) + model->mlp_offset;
  const int blocks = (int)((n + 127) / 128);
  if constexpr (sizeof(T) == 4) {
    constexpr int TW = 4;
    tc::k_wfrag<S><<<tc::Fr<S>::NALL + 1 + tc::UmmaW::kTiles, 128, 0, stream>>>(mlp, w.wfrag);
    GSB_LAUNCHED_T("k_wfrag");
    GSB_CHECK(cudaFuncSetAttribute(tc::k_fwd_tc<S, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)tc::FwdTc<S, TW>::smem()));
    tc::k_fwd_tc<S, TW><<<blocks, TW * 32, tc::FwdTc<S, TW>::smem(), stream>>>(w, G, 0, 1, mlp, nullptr,
                                                                             pts, (int)n);
  } else {
    const size_t smem_fwd = ((size_t)(S::NMLP + 3) / 4 * 4 + 128 * FwdRow<T, S>::ROW) * esz;
    GSB_CHECK(cudaFuncSetAttribute(k_fwd<T, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_fwd));
    k_fwd<T, S, false><<<blocks, 128, smem_fwd, stream>>>(w, G, 0, 1, nullptr, pts, (int)n, mlp);
  }
  GSB_LAUNCHED_T("k_fwd");
  return GSB_OK;
}

template <typename T, class S>
int run_sdf_points(const gsb_model_t* model, const void* points, int64_t n, void* phi_out, void* ws,
                   size_t ws_bytes, cudaStream_t stream) {
  if (S::NMLP != nmlp_of(model) || n <= 0 || n > INT32_MAX) return GSB_E_ARG;
  timing_point(nullptr, stream);
  size_t need = 0;
  Ws<T> w = carve_sdf<T>(ws, n, S::NMLP, &need, false);
  if (need > ws_bytes) return GSB_E_ARG;
  w.sphi = reinterpret_cast<T*>(phi_out);
  GSB_CHECK(cudaMemsetAsync(w.status, 0, GSB_N_STATUS * sizeof(int32_t), stream));
  return sdf_forward<T, S>(model, w, reinterpret_cast<const T*>(points), n, stream);
}

template <typename T, class S>
int run_sdf_fit(const gsb_model_t* model, const void* points, const void* targets, int64_t nb,
                int64_t na, void* ws, size_t ws_bytes, double* loss_out, cudaStream_t stream) {
  const int64_t n = nb + na;
  if (S::NMLP != nmlp_of(model) || nb <= 0 || na < 0 || n > INT32_MAX) return GSB_E_ARG;
  timing_point(nullptr, stream);
  size_t need = 0;
  Ws<T> w = carve_sdf<T>(ws, n, S::NMLP, &need);
  if (need > ws_bytes) return GSB_E_ARG;
  GSB_CHECK(cudaMemsetAsync(w.status, 0, GSB_N_STATUS * sizeof(int32_t), stream));
  GSB_CHECK(cudaMemsetAsync(w.parts, 0, 16 * sizeof(double), stream));
  const T* pts = reinterpret_cast<const T*>(points);
  int rc = sdf_forward<T, S>(model, w, pts, n, stream);
  if (rc != GSB_OK) return rc;
  k_fit_seed<T><<<(int)((n + 255) / 256), 256, 0, stream>>>(w, reinterpret_cast<const T*>(targets), nb, na);
  GSB_LAUNCHED_T("k_fit_seed");
  Geo G = geo_of(model, sizeof(T));
  T* grads = reinterpret_cast<T*>(model->grads);
  const T* mlp = reinterpret_cast<const T*>(model->params) + model->mlp_offset;
  int nb_geo;
  if constexpr (sizeof(T) == 4) {
    constexpr int WGEO = 4;
    nb_geo = (int)((n + WGEO * 32 - 1) / (WGEO * 32));
    const size_t smem_g = tc::GeoTc<S, WGEO>::smem();
    GSB_CHECK(cudaFuncSetAttribute(tc::k_bwd_geom_tc<S, WGEO>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_g));
    tc::k_bwd_geom_tc<S, WGEO><<<nb_geo, WGEO * 32, smem_g, stream>>>(w, G, 0, 1, mlp, nullptr, pts,
                                                                      (int)n, 2);
  } else {
    constexpr int WG = 2;
    nb_geo = (int)std::min<int64_t>((n + WG * 32 - 1) / (WG * 32), (int64_t)num_sms() * 2);
    nb_geo = std::max(1, std::min(nb_geo, kNbMax));
    const size_t smem_g = ((size_t)(S::NG + 3) / 4 * 4 + (size_t)WG * 32 * GeoRow<T, S>::ROW) * sizeof(T);
    GSB_CHECK(cudaFuncSetAttribute(k_bwd_geom<T, S, WG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_g));
    k_bwd_geom<T, S, WG><<<nb_geo, WG * 32, smem_g, stream>>>(w, G, 0, 1, nullptr, pts, (int)n, 2, mlp);
  }
  GSB_LAUNCHED_T("k_bwd_geom");
  GSB_CHECK(cudaMemsetAsync(w.fin_cnt, 0, (S::NMLP + 31) / 32 * sizeof(unsigned), stream));
  k_finalize_mlp2<T, S><<<dim3((S::NMLP + 31) / 32, FIN_SPLIT), 256, 0, stream>>>(w, grads, model->mlp_offset,
                                                                                nb_geo, 0);
  GSB_LAUNCHED_T("k_finalize_mlp");
  if (loss_out)
    GSB_CHECK(cudaMemcpyAsync(loss_out, w.parts, sizeof(double), cudaMemcpyDeviceToDevice, stream));
  return GSB_OK;
}

// ---- dense SDF volume (mesher.sdf_volume, gs/mesher.py:114-133): vertex
// (i, j, k) at lo + (i, j, k) * res in f64 (numpy's lo + arange * res), cast
// to the dtype, decoded in chunks of kVolChunk points; float32 output
constexpr int64_t kVolChunk = int64_t(1) << 22;

template <typename T>
__global__ void k_grid_points(double lx, double ly, double lz, double res, int64_t ny, int64_t nz,
                              int64_t start, int64_t count, T* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int64_t g = start + t;
  const int64_t k = g % nz, j = (g / nz) % ny, i = g / (ny * nz);
  out[t * 3] = (T)(lx + (double)i * res);
  out[t * 3 + 1] = (T)(ly + (double)j * res);
  out[t * 3 + 2] = (T)(lz + (double)k * res);
}

template <typename T>
__global__ void k_to_f32(const T* __restrict__ in, int64_t n, float* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) out[t] = (float)in[t];
}

template <typename T>
size_t sdf_volume_ws(int nmlp) {
  size_t b = 0;
  carve_sdf<T>(nullptr, kVolChunk, nmlp, &b, false);
  return align_up(b) + align_up((size_t)kVolChunk * 3 * sizeof(T)) + align_up((size_t)kVolChunk * sizeof(T));
}

template <typename T, class S>
int run_sdf_volume(const gsb_model_t* model, const double* lo, double res, int64_t nx, int64_t ny,
                   int64_t nz, float* vol, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (S::NMLP != nmlp_of(model) || nx <= 0 || ny <= 0 || nz <= 0) return GSB_E_ARG;
  if (ws_bytes < sdf_volume_ws<T>(S::NMLP)) return GSB_E_ARG;
  size_t b = 0;
  unsigned char* base = reinterpret_cast<unsigned char*>(ws);
  Ws<T> w = carve_sdf<T>(base, kVolChunk, S::NMLP, &b, false);
  T* pts = reinterpret_cast<T*>(base + align_up(b));
  T* phi = reinterpret_cast<T*>(base + align_up(b) + align_up((size_t)kVolChunk * 3 * sizeof(T)));
  GSB_CHECK(cudaMemsetAsync(w.status, 0, GSB_N_STATUS * sizeof(int32_t), stream));
  const int64_t total = nx * ny * nz;
  for (int64_t s0 = 0; s0 < total; s0 += kVolChunk) {
    const int64_t n = std::min(kVolChunk, total - s0);
    k_grid_points<T><<<(int)((n + 255) / 256), 256, 0, stream>>>(lo[0], lo[1], lo[2], res, ny, nz, s0, n,
                                                                pts);
    GSB_LAUNCHED_T("k_grid_points");
    w.sphi = sizeof(T) == 4 ? reinterpret_cast<T*>(vol + s0) : phi;
    const int rc = sdf_forward<T, S>(model, w, pts, n, stream);
    if (rc != GSB_OK) return rc;
    if (sizeof(T) != 4) {
      k_to_f32<T><<<(int)((n + 255) / 256), 256, 0, stream>>>(phi, n, vol + s0);
      GSB_LAUNCHED_T("k_to_f32");
    }
  }
  return GSB_OK;
}

// pose gradients of the step just run on (model, data, st): SURVEY.md 8f #3
template <typename T, class S>
int run_pose_grad(const gsb_model_t* model, const gsb_dataset_t* data, const gsb_step_t* st,
                  const gsb_pose_t* pose, void* scratch, size_t scratch_bytes, cudaStream_t stream) {
  if (S::NMLP != nmlp_of(model)) return GSB_E_ARG;
  const Sizes z = sizes_of(model, st->n_rays, st->n_coarse, st->n_rounds, st->n_add, st->n_smooth);
  const PoseLayout PL = pose_layout<T>(z, S::IN_G);
  if (PL.total > scratch_bytes) return GSB_E_ARG;
  size_t need = 0;
  Ws<T> w = carve<T>(st->workspace, z, &need);
  if (need > st->workspace_bytes) return GSB_E_ARG;
  // the colour backward reads the colour features the taped forward kept
  // only when both are the tcgen05 kernels (the A/B forms re-gather)
  if (!(sizeof(T) == 4 && t5_fwd_mode() > 0 && use_t5_col())) w.scolf = nullptr;
  if (z.M == 0) return GSB_OK;
  const Geo G = geo_of(model, sizeof(T));
  const T* params = reinterpret_cast<const T*>(model->params);
  T* grads = reinterpret_cast<T*>(model->grads);
  const double* dep = w.dep[st->n_rounds % 2];
  unsigned char* sc = reinterpret_cast<unsigned char*>(scratch);
  T* xbar = reinterpret_cast<T*>(sc + PL.xbar);
  double* rbar = reinterpret_cast<double*>(sc + PL.rbar);
  bool fast = false;
  if constexpr (sizeof(T) == 4) {
    // the step stored dphi/dz and the colour-input cotangents in this scratch
    fast = st->pose_work == scratch;
    if (fast) {
      w.pose_g = reinterpret_cast<T*>(sc + PL.g);
      w.pose_fb = reinterpret_cast<T*>(sc + PL.fb);
      k_pose_fast<S><<<(int)((z.MN + 127) / 128), 128, 0, stream>>>(w, G, z.M, z.N, dep, xbar);
      GSB_LAUNCHED_T("k_pose_fast");
    }
  }
  if (!fast) {
    using R = FwdRow<T, S>;
    const size_t smem = ((size_t)(S::NMLP + 3) / 4 * 4 + 128 * R::ROW) * sizeof(T);
    GSB_CHECK(cudaFuncSetAttribute(k_pose_xbar<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_pose_xbar<T, S><<<(int)((z.MN + 127) / 128), 128, smem, stream>>>(w, G, z.M, z.N, dep,
                                                                        params + model->mlp_offset, xbar);
    GSB_LAUNCHED_T("k_pose_xbar");
  }
  k_pose_ray<T><<<(z.M + 3) / 4, 128, 0, stream>>>(w, *data, st->ray_ids, z.M, z.N, dep, xbar, rbar);
  GSB_LAUNCHED_T("k_pose_ray");
  k_pose_frames<T><<<pose->n_frames, 1024, 0, stream>>>(z.M, *pose, params, rbar, grads);
  GSB_LAUNCHED_T("k_pose_frames");
  return GSB_OK;
}

}  // namespace host
}  // namespace gsb
