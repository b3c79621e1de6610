// gsb_host.cuh -- host-side helpers shared by the ABI and the step TUs.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>

#include "gsb_kernels.cuh"

namespace gsb {
namespace host {

constexpr int kNbMax = 1024;  // max CTAs of the backward kernels (partials slots)

// kernels launched by this library (process-wide; gsb_launch_count)
void note_launch();
// opt-in per-kernel CUDA-event timing (gsb_timing_enable): records an event on
// `s` after each production launch; name == nullptr marks the start of a call
void timing_point(const char* name, cudaStream_t s);

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

struct Sizes {
  int M, N, ld, S;
  int64_t MN, NS;
  int nmlp;
};

template <typename T>
struct Carver {
  size_t off = 0;
  unsigned char* base;
  template <typename U>
  U* take(int64_t count) {
    U* p = base ? reinterpret_cast<U*>(base + off) : nullptr;
    off = align_up(off + (size_t)count * sizeof(U));
    return p;
  }
};

template <typename T>
Ws<T> carve(void* ws, const Sizes& z, size_t* bytes, int64_t* off_parts = nullptr,
            int64_t* off_counts = nullptr, int64_t* off_status = nullptr,
            int64_t* off_dep = nullptr, int64_t* off_wts = nullptr, int rounds = 0) {
  Carver<T> c;
  c.base = reinterpret_cast<unsigned char*>(ws);
  Ws<T> w;
  w.mlp_slots = 0;
  w.sweep = 0;
  w.dbg = 0;
  w.det_keys = nullptr;
  w.det_vals = nullptr;
  w.pose_g = nullptr;
  w.pose_fb = nullptr;
  w.ld = z.ld;
  // small, externally visible blocks first
  size_t o_parts = c.off;
  w.parts = c.template take<double>(16);
  size_t o_counts = c.off;
  w.counts = c.template take<long long>(8);
  size_t o_status = c.off;
  w.status = c.template take<int32_t>(GSB_N_STATUS);
  w.evl_count = c.template take<int32_t>(GSB_MAX_ROUNDS);  // one list counter per importance round
  w.o = c.template take<T>(z.M * 3);
  w.r = c.template take<T>(z.M * 3);
  w.od = c.template take<double>(z.M * 3);
  w.rd = c.template take<double>(z.M * 3);
  w.nearv = c.template take<double>(z.M);
  w.farv = c.template take<double>(z.M);
  w.col = c.template take<T>(z.M * 3);
  w.dray = c.template take<double>(z.M);
  w.valid = c.template take<int32_t>(z.M);
  w.cnt = c.template take<int32_t>(z.M * 3);
  size_t o_dep[2];
  for (int b = 0; b < 2; ++b) {
    o_dep[b] = c.off;
    w.dep[b] = c.template take<double>((int64_t)z.M * z.ld);
  }
  for (int b = 0; b < 2; ++b) w.phi[b] = c.template take<double>((int64_t)z.M * z.ld);
  w.evl_cap = (int64_t)z.M * z.ld;
  w.evl = c.template take<int32_t>(w.evl_cap);
  w.sphi = c.template take<T>(z.NS);
  w.sgphi = c.template take<T>(z.NS * 3);
  w.scol = c.template take<T>(z.MN * 3);
  w.scolf = c.template take<T>(z.MN * 8);  // colour features (CC <= 8)
  w.pbar = c.template take<T>(z.NS);
  w.ubar = c.template take<T>(z.NS * 3);
  w.cbar = c.template take<T>(z.MN * 3);
  size_t o_wts = c.off;
  w.wts = c.template take<T>(z.MN);
  w.ray_part = c.template take<double>((int64_t)z.M * 8);
  w.smooth_part = c.template take<double>(z.S > 0 ? z.S : 1);
  // partial weight-gradient slots: one per backward CTA (float32 path: one
  // CTA per 128 samples), at least kNbMax for the persistent float64 kernels
  const int64_t nb = std::max<int64_t>(kNbMax, (z.NS + 127) / 128);
  w.nb_max = (int)nb;
  w.mlp_part = c.template take<T>(nb * ((z.nmlp + 3) / 4 * 4));
  w.wfrag = c.template take<uint4>(4096 + 68 + 3072);  // tc::kFragBufU4: fragments + vector block
  w.fin_red = c.template take<double>((int64_t)16 * z.nmlp);  // FIN_SPLIT x NMLP
  w.fin_cnt = c.template take<unsigned>((z.nmlp + 31) / 32);
  w.loss_red = c.template take<double>((int64_t)((std::max(z.M, z.S) + 255) / 256 + 1) * 8);
  w.loss_cnt = c.template take<unsigned>(4);
  w.imp_state = c.template take<uint64_t>((int64_t)GSB_MAX_ROUNDS * z.M * 2);
  if (bytes) *bytes = c.off;
  if (off_parts) *off_parts = (int64_t)o_parts;
  if (off_counts) *off_counts = (int64_t)o_counts;
  if (off_status) *off_status = (int64_t)o_status;
  if (off_dep) *off_dep = (int64_t)o_dep[rounds % 2];
  if (off_wts) *off_wts = (int64_t)o_wts;
  return w;
}

inline LevelDev level_dev(const gsb_level_t& L, void* params, void* grads, size_t esz) {
  LevelDev d;
  d.feat = reinterpret_cast<unsigned char*>(params) + L.offset * esz;
  d.grad = grads ? reinterpret_cast<unsigned char*>(grads) + L.offset * esz : nullptr;
  d.nx = L.nx;
  d.ny = L.ny;
  d.nz = L.nz;
  d.C = L.channels;
  d.ox = L.ox;
  d.oy = L.oy;
  d.oz = L.oz;
  d.vs = L.voxel;
  d.inv_vs = 1.0 / L.voxel;
  int mx = L.nx > L.ny ? L.nx : L.ny;
  mx = mx > L.nz ? mx : L.nz;
  d.eps = 1e-9 * (double)mx;  // gs/diffcore.py:742
  return d;
}

inline Geo geo_of(const gsb_model_t* m, size_t esz) {
  Geo G;
  for (int l = 0; l < m->n_levels; ++l) G.lv[l] = level_dev(m->levels[l], m->params, m->grads, esz);
  G.col = level_dev(m->color, m->params, m->grads, esz);
  for (int a = 0; a < 3; ++a) {
    G.lo[a] = m->lo_c[a];
    G.hi[a] = m->hi_c[a];
  }
  return G;
}

inline int nmlp_of(const gsb_model_t* m) {
  int in_g = m->n_levels * m->levels[0].channels, in_c = m->color.channels + 3;
  int ng = in_g * 32 + 32 + 1024 + 32 + 32 + 1;
  return (ng + 3) / 4 * 4 + in_c * 32 + 32 + 1024 + 32 + 96 + 3;
}

inline Sizes sizes_of(const gsb_model_t* m, int M, int Nc, int R, int A, int S) {
  Sizes z;
  z.M = M;
  z.N = Nc + R * A;
  z.ld = z.N;
  z.S = S;
  z.MN = (int64_t)M * z.N;
  z.NS = z.MN + 2 * (int64_t)S;
  z.nmlp = nmlp_of(m);
  return z;
}


}  // namespace host
}  // namespace gsb
