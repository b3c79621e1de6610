// gsb.cu -- C ABI (include/gsb.h) over the GO-Surf step kernels.
#include <cuda_runtime.h>

#include <type_traits>

#include "gsb_step.cuh"
#include "gsb_mesh.cuh"
#include "gsb_scene.cuh"

#include <atomic>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace gsb {
namespace host {
static std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// per-kernel timing: an event after every production launch; the duration of
// a launch is the gap to the previous mark (the call's start mark or the
// previous kernel) on the same stream
struct Mark {
  const char* name;
  cudaEvent_t ev;
};
static std::mutex g_tm;
static bool g_timing = false;
static std::vector<Mark> g_marks;
static std::vector<cudaEvent_t> g_pool;

void timing_point(const char* name, cudaStream_t s) {
  if (!g_timing) return;
  std::lock_guard<std::mutex> lk(g_tm);
  cudaEvent_t e;
  if (g_pool.empty()) {
    if (cudaEventCreate(&e) != cudaSuccess) return;
  } else {
    e = g_pool.back();
    g_pool.pop_back();
  }
  cudaEventRecord(e, s);
  g_marks.push_back({name, e});
}
}  // namespace host
}  // namespace gsb

using namespace gsb;


using namespace gsb::host;

#define GSB_DECL(name)                                                                  \
  extern "C" int name(const gsb_model_t* m, const gsb_dataset_t* d, const gsb_step_t* st, \
                      cudaStream_t s);
GSB_DECL(gsb_step_f446)
GSB_DECL(gsb_step_d446)
GSB_DECL(gsb_step_f222)
GSB_DECL(gsb_step_d222)
#define GSB_DECL_SDF(tag)                                                                       \
  extern "C" int gsb_step_##tag##_sdf_points(const gsb_model_t*, const void*, int64_t, void*,  \
                                             void*, size_t, cudaStream_t);                     \
  extern "C" int gsb_step_##tag##_sdf_fit(const gsb_model_t*, const void*, const void*, int64_t, \
                                          int64_t, void*, size_t, double*, cudaStream_t);
#define GSB_DECL_VOL(tag)                                                                          \
  extern "C" int gsb_step_##tag##_sdf_volume(const gsb_model_t*, const double*, double, int64_t, int64_t, \
                                             int64_t, float*, void*, size_t, cudaStream_t);
#define GSB_DECL_POSE(tag)                                                                      \
  extern "C" int gsb_step_##tag##_pose_grad(const gsb_model_t*, const gsb_dataset_t*, const gsb_step_t*, \
                                            const gsb_pose_t*, void*, size_t, cudaStream_t);
GSB_DECL_POSE(f446)
GSB_DECL_POSE(d446)
GSB_DECL_POSE(f222)
GSB_DECL_POSE(d222)
GSB_DECL_VOL(f446)
GSB_DECL_VOL(d446)
GSB_DECL_VOL(f222)
GSB_DECL_VOL(d222)
GSB_DECL_SDF(f446)
GSB_DECL_SDF(d446)
GSB_DECL_SDF(f222)
GSB_DECL_SDF(d222)

namespace gsb_abi {

// twin: explicit uniforms / outputs

template <typename T>
int dispatch_shape(const gsb_model_t* m, const gsb_dataset_t* d, const gsb_step_t* st,
                   cudaStream_t s) {
  const int nl = m->n_levels, cg = m->levels[0].channels, cc = m->color.channels;
  for (int l = 0; l < nl; ++l)
    if (m->levels[l].channels != cg) return GSB_E_ARG;
  const bool f = sizeof(T) == 4;
  if (nl == 4 && cg == 4 && cc == 6) return f ? gsb_step_f446(m, d, st, s) : gsb_step_d446(m, d, st, s);
  if (nl == 2 && cg == 2 && cc == 2) return f ? gsb_step_f222(m, d, st, s) : gsb_step_d222(m, d, st, s);
  return GSB_E_ARG;
}

// shape tag of a model: 0 = (4,4,6), 1 = (2,2,2), -1 unsupported
inline int shape_tag(const gsb_model_t* m) {
  const int nl = m->n_levels, cg = m->levels[0].channels, cc = m->color.channels;
  for (int l = 0; l < nl; ++l)
    if (m->levels[l].channels != cg) return -1;
  if (nl == 4 && cg == 4 && cc == 6) return 0;
  if (nl == 2 && cg == 2 && cc == 2) return 1;
  return -1;
}

template <typename T>
void regions_of(const Sizes& z, int rounds, int64_t* o) {
  unsigned char* base = reinterpret_cast<unsigned char*>(4096);  // never dereferenced
  size_t b = 0;
  Ws<T> w = carve<T>(base, z, &b);
  auto off = [&](const void* p) { return (int64_t)(reinterpret_cast<const unsigned char*>(p) - base); };
  o[GSB_R_PARTS] = off(w.parts);
  o[GSB_R_COUNTS] = off(w.counts);
  o[GSB_R_STATUS] = off(w.status);
  o[GSB_R_DEPTHS] = off(w.dep[rounds % 2]);
  o[GSB_R_WEIGHTS] = off(w.wts);
  o[GSB_R_PHI] = off(w.sphi);
  o[GSB_R_GPHI] = off(w.sgphi);
  o[GSB_R_COLOR] = off(w.scol);
  o[GSB_R_PBAR] = off(w.pbar);
  o[GSB_R_UBAR] = off(w.ubar);
  o[GSB_R_CBAR] = off(w.cbar);
  o[GSB_R_RAY_O] = off(w.o);
  o[GSB_R_RAY_R] = off(w.r);
  o[GSB_R_RAY_FAR] = off(w.farv);
}

}  // namespace gsb_abi
using namespace gsb_abi;

extern "C" {

int gsb_version(void) { return 1; }

uint64_t gsb_launch_count(void) { return gsb::host::g_launches.load(); }

int gsb_timing_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(gsb::host::g_tm);
  gsb::host::g_timing = on != 0;
  return GSB_OK;
}

int gsb_timing_collect(int32_t max_kernels, char* names, double* total_ms, int64_t* launches,
                       int32_t* n_kernels) {
  using namespace gsb::host;
  if (max_kernels <= 0 || !names || !total_ms || !launches || !n_kernels) return GSB_E_ARG;
  std::lock_guard<std::mutex> lk(g_tm);
  if (!g_marks.empty() && cudaEventSynchronize(g_marks.back().ev) != cudaSuccess) return GSB_E_CUDA;
  int n = 0;
  for (size_t i = 1; i < g_marks.size(); ++i) {
    if (!g_marks[i].name) continue;  // start mark of a call
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, g_marks[i - 1].ev, g_marks[i].ev) != cudaSuccess) return GSB_E_CUDA;
    int k = 0;
    while (k < n && std::strncmp(names + 64 * k, g_marks[i].name, 63) != 0) ++k;
    if (k == n) {
      if (n == max_kernels) continue;
      std::strncpy(names + 64 * k, g_marks[i].name, 63);
      names[64 * k + 63] = 0;
      total_ms[k] = 0.0;
      launches[k] = 0;
      ++n;
    }
    total_ms[k] += ms;
    launches[k] += 1;
  }
  for (auto& m : g_marks) g_pool.push_back(m.ev);
  g_marks.clear();
  *n_kernels = n;
  return GSB_OK;
}

int gsb_sdf_workspace_size(const gsb_model_t* model, int64_t n_points, size_t* bytes) {
  if (!model || !bytes || n_points <= 0) return GSB_E_ARG;
  const int nmlp = nmlp_of(model);
  if (model->precision == 0)
    carve_sdf<float>(nullptr, n_points, nmlp, bytes);
  else
    carve_sdf<double>(nullptr, n_points, nmlp, bytes);
  return GSB_OK;
}

int gsb_sdf_points(const gsb_model_t* model, const void* points, int64_t n, void* phi_out,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (!model || !points || !phi_out || !workspace) return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool f = model->precision == 0;
  switch (shape_tag(model)) {
    case 0:
      return f ? gsb_step_f446_sdf_points(model, points, n, phi_out, workspace, workspace_bytes, s)
               : gsb_step_d446_sdf_points(model, points, n, phi_out, workspace, workspace_bytes, s);
    case 1:
      return f ? gsb_step_f222_sdf_points(model, points, n, phi_out, workspace, workspace_bytes, s)
               : gsb_step_d222_sdf_points(model, points, n, phi_out, workspace, workspace_bytes, s);
    default:
      return GSB_E_ARG;
  }
}

int gsb_render_frames(const gsb_scene_t* scene, const double* poses, int32_t n_frames, int32_t height,
                      int32_t width, double fx, double fy, double cx, double cy, double max_t,
                      const double* noise, double sigma0, const gsb_render_opts_t* opts, uint8_t* colors,
                      uint16_t* depth_mm, void* stream) {
  if (!scene || !poses || !opts || !colors || !depth_mm || n_frames < 0 || height <= 0 || width <= 0)
    return GSB_E_ARG;
  if (scene->n_prims < 1 || scene->n_prims > GSB_SCENE_MAX_PRIMS || scene->n_ops < 1 ||
      scene->n_ops > GSB_SCENE_MAX_OPS)
    return GSB_E_ARG;
  int sp = 0;  // validate the program: indices, stack depth, one result
  for (int i = 0; i < scene->n_ops; ++i) {
    const int op = scene->op[i][0], arg = scene->op[i][1];
    if (op == 0) {
      if (arg < 0 || arg >= scene->n_prims || ++sp > GSB_SCENE_MAX_STACK) return GSB_E_ARG;
    } else if (op == 1) {
      if (sp < 1) return GSB_E_ARG;
    } else if (op == 2) {
      if (arg < 1 || arg > sp) return GSB_E_ARG;
      sp -= arg - 1;
    } else {
      return GSB_E_ARG;
    }
  }
  if (sp != 1 || (sigma0 > 0.0 && !noise)) return GSB_E_ARG;
  const int64_t n = (int64_t)n_frames * height * width;
  if (n == 0) return GSB_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  k_render_frames<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(*scene, poses, n, height, width, fx, fy, cx, cy,
                                                              max_t, noise, sigma0, *opts, colors, depth_mm);
  note_launch();
  timing_point("k_render_frames", s);
  return cudaGetLastError() == cudaSuccess ? GSB_OK : GSB_E_CUDA;
}

int gsb_pose_table(const gsb_model_t* model, const gsb_pose_t* pose, double* table, double* table_f64,
                   void* stream) {
  if (!model || !pose || !table || !table_f64 || pose->n_frames < 0) return GSB_E_ARG;
  if (pose->n_frames == 0) return GSB_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int b = (pose->n_frames + 127) / 128;
  if (model->precision == 0)
    k_pose_table<float><<<b, 128, 0, s>>>(*pose, reinterpret_cast<const float*>(model->params), table, table_f64);
  else
    k_pose_table<double><<<b, 128, 0, s>>>(*pose, reinterpret_cast<const double*>(model->params), table,
                                           table_f64);
  note_launch();
  timing_point("k_pose_table", s);
  return cudaGetLastError() == cudaSuccess ? GSB_OK : GSB_E_CUDA;
}

int gsb_det_scratch_size(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse, int32_t n_rounds,
                         int32_t n_add, int32_t n_smooth, size_t* bytes) {
  if (!model || !bytes || n_rays < 0) return GSB_E_ARG;
  const Sizes z = sizes_of(model, n_rays, n_coarse, n_rounds, n_add, n_smooth);
  *bytes = model->precision == 0 ? det_layout<float>(z, model->n_levels).total
                                 : det_layout<double>(z, model->n_levels).total;
  return GSB_OK;
}

int gsb_pose_scratch_size(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse, int32_t n_rounds,
                          int32_t n_add, size_t* bytes) {
  if (!model || !bytes || n_rays < 0) return GSB_E_ARG;
  const Sizes z = sizes_of(model, n_rays, n_coarse, n_rounds, n_add, 0);
  const int in_g = model->n_levels * model->levels[0].channels;
  *bytes = model->precision == 0 ? pose_scratch_bytes<float>(z, in_g) : pose_scratch_bytes<double>(z, in_g);
  return GSB_OK;
}

int gsb_pose_grad(const gsb_model_t* model, const gsb_dataset_t* data, const gsb_step_t* step,
                  const gsb_pose_t* pose, void* scratch, size_t scratch_bytes, void* stream) {
  if (!model || !data || !step || !pose || !scratch) return GSB_E_ARG;
  if (pose->n_frames != data->n_frames) return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool f = model->precision == 0;
  switch (shape_tag(model)) {
    case 0:
      return f ? gsb_step_f446_pose_grad(model, data, step, pose, scratch, scratch_bytes, s)
               : gsb_step_d446_pose_grad(model, data, step, pose, scratch, scratch_bytes, s);
    case 1:
      return f ? gsb_step_f222_pose_grad(model, data, step, pose, scratch, scratch_bytes, s)
               : gsb_step_d222_pose_grad(model, data, step, pose, scratch, scratch_bytes, s);
    default:
      return GSB_E_ARG;
  }
}

int gsb_sdf_volume_workspace_size(const gsb_model_t* model, size_t* bytes) {
  if (!model || !bytes) return GSB_E_ARG;
  const int nmlp = nmlp_of(model);
  *bytes = model->precision == 0 ? sdf_volume_ws<float>(nmlp) : sdf_volume_ws<double>(nmlp);
  return GSB_OK;
}

int gsb_sdf_volume(const gsb_model_t* model, const double* lo_host, double resolution, int64_t nx,
                   int64_t ny, int64_t nz, float* vol, void* workspace, size_t workspace_bytes,
                   void* stream) {
  if (!model || !lo_host || !vol || !workspace || !(resolution > 0.0)) return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool f = model->precision == 0;
  switch (shape_tag(model)) {
    case 0:
      return f ? gsb_step_f446_sdf_volume(model, lo_host, resolution, nx, ny, nz, vol, workspace,
                                          workspace_bytes, s)
               : gsb_step_d446_sdf_volume(model, lo_host, resolution, nx, ny, nz, vol, workspace,
                                          workspace_bytes, s);
    case 1:
      return f ? gsb_step_f222_sdf_volume(model, lo_host, resolution, nx, ny, nz, vol, workspace,
                                          workspace_bytes, s)
               : gsb_step_d222_sdf_volume(model, lo_host, resolution, nx, ny, nz, vol, workspace,
                                          workspace_bytes, s);
    default:
      return GSB_E_ARG;
  }
}

// ---- marching cubes
static size_t mc_layout(int64_t cells, size_t* o_counts, size_t* o_offsets, size_t* o_mm, size_t* o_tmp,
                        size_t* tmp_bytes) {
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int32_t*)nullptr, (int32_t*)nullptr, (int)cells);
  size_t off = 0;
  *o_counts = off;
  off = align_up(off + (size_t)cells * 4);
  *o_offsets = off;
  off = align_up(off + (size_t)cells * 4);
  *o_mm = off;
  off = align_up(off + 16);
  *o_tmp = off;
  off = align_up(off + tb);
  *tmp_bytes = tb;
  return off;
}

int gsb_mc_workspace_size(int64_t nx, int64_t ny, int64_t nz, size_t* bytes) {
  if (!bytes || nx < 2 || ny < 2 || nz < 2) return GSB_E_ARG;
  const int64_t cells = (nx - 1) * (ny - 1) * (nz - 1);
  if (cells >= INT32_MAX) return GSB_E_ARG;
  size_t a, b, c, d, t;
  *bytes = mc_layout(cells, &a, &b, &c, &d, &t);
  return GSB_OK;
}

__global__ void k_mc_total(const int32_t* counts, const int32_t* offsets, int64_t cells, const int* mm,
                           int64_t* total, float* minmax) {
  total[0] = (int64_t)offsets[cells - 1] + counts[cells - 1];
  for (int q = 0; q < 2; ++q) {
    const int i = mm[q];
    minmax[q] = __int_as_float(i >= 0 ? i : i ^ 0x7fffffff);
  }
}

int gsb_mc_count(const float* vol, int64_t nx, int64_t ny, int64_t nz, float level, const int8_t* table,
                 void* workspace, size_t workspace_bytes, int64_t* total, float* minmax, void* stream) {
  if (!vol || !table || !workspace || !total || !minmax || nx < 2 || ny < 2 || nz < 2) return GSB_E_ARG;
  const int64_t cells = (nx - 1) * (ny - 1) * (nz - 1);
  if (cells >= INT32_MAX) return GSB_E_ARG;
  size_t oc, oo, om, ot, tb;
  if (mc_layout(cells, &oc, &oo, &om, &ot, &tb) > workspace_bytes) return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* w = reinterpret_cast<unsigned char*>(workspace);
  int32_t* counts = reinterpret_cast<int32_t*>(w + oc);
  int32_t* offsets = reinterpret_cast<int32_t*>(w + oo);
  int* mm = reinterpret_cast<int*>(w + om);
  const int init[2] = {INT_MAX, INT_MIN};
  GSB_CHECK(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
  mesh::k_mc_count<<<(int)((cells + 255) / 256), 256, 0, s>>>(vol, nx, ny, nz, level, table, counts, mm);
  GSB_LAUNCHED();
  GSB_CHECK(cub::DeviceScan::ExclusiveSum(w + ot, tb, counts, offsets, (int)cells, s));
  k_mc_total<<<1, 1, 0, s>>>(counts, offsets, cells, mm, total, minmax);
  GSB_LAUNCHED();
  return GSB_OK;
}

int gsb_mc_emit(const float* vol, int64_t nx, int64_t ny, int64_t nz, float level, double ox, double oy,
                double oz, double resolution, const int8_t* table, void* workspace, size_t workspace_bytes,
                double* verts, int64_t* keys, void* stream) {
  if (!vol || !table || !workspace || !verts || nx < 2 || ny < 2 || nz < 2) return GSB_E_ARG;
  const int64_t cells = (nx - 1) * (ny - 1) * (nz - 1);
  size_t oc, oo, om, ot, tb;
  if (mc_layout(cells, &oc, &oo, &om, &ot, &tb) > workspace_bytes) return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* w = reinterpret_cast<unsigned char*>(workspace);
  mesh::k_mc_emit<<<(int)((cells + 255) / 256), 256, 0, s>>>(
      vol, nx, ny, nz, level, ox, oy, oz, resolution, table, reinterpret_cast<const int32_t*>(w + oc),
      reinterpret_cast<const int32_t*>(w + oo), verts, keys);
  GSB_LAUNCHED();
  return GSB_OK;
}

// ---- exact nearest neighbours
static size_t nn_layout(int64_t nr, int64_t ncells, size_t o[6], size_t* tmp_bytes, int* bits) {
  int b = 1;
  while (b < 63 && (int64_t(1) << b) < ncells) ++b;
  *bits = b;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, (const int64_t*)nullptr, (int64_t*)nullptr,
                                  (const int64_t*)nullptr, (int64_t*)nullptr, (int)nr, 0, b);
  size_t off = 0;
  for (int k = 0; k < 4; ++k) {
    o[k] = off;
    off = align_up(off + (size_t)nr * 8);
  }
  o[4] = off;
  off = align_up(off + (size_t)(ncells + 1) * 8);
  o[5] = off;
  off = align_up(off + tb);
  *tmp_bytes = tb;
  return off;
}

int gsb_nn_workspace_size(int64_t n_ref, int64_t nx, int64_t ny, int64_t nz, size_t* bytes) {
  if (!bytes || n_ref <= 0 || n_ref >= INT32_MAX || nx <= 0 || ny <= 0 || nz <= 0) return GSB_E_ARG;
  size_t o[6], tb;
  int bits;
  *bytes = nn_layout(n_ref, nx * ny * nz, o, &tb, &bits);
  return GSB_OK;
}

int gsb_nearest_neighbors(const double* query, int64_t nq, const double* ref, int64_t nr, const double* lo_host,
                          double cell, int64_t nx, int64_t ny, int64_t nz, void* workspace,
                          size_t workspace_bytes, double* out_d, int64_t* out_i, void* stream) {
  if (!query || !ref || !lo_host || !workspace || !out_d || !out_i || nr <= 0 || nq < 0 || !(cell > 0.0))
    return GSB_E_ARG;
  const int64_t ncells = nx * ny * nz;
  size_t o[6], tb;
  int bits;
  if (nn_layout(nr, ncells, o, &tb, &bits) > workspace_bytes) return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* w = reinterpret_cast<unsigned char*>(workspace);
  int64_t* cid = reinterpret_cast<int64_t*>(w + o[0]);
  int64_t* idx = reinterpret_cast<int64_t*>(w + o[1]);
  int64_t* scid = reinterpret_cast<int64_t*>(w + o[2]);
  int64_t* order = reinterpret_cast<int64_t*>(w + o[3]);
  int64_t* starts = reinterpret_cast<int64_t*>(w + o[4]);
  mesh::k_nn_cells<<<(int)((nr + 255) / 256), 256, 0, s>>>(ref, nr, lo_host[0], lo_host[1], lo_host[2], cell,
                                                           nx, ny, nz, cid, idx);
  GSB_LAUNCHED();
  GSB_CHECK(cub::DeviceRadixSort::SortPairs(w + o[5], tb, cid, scid, idx, order, (int)nr, 0, bits, s));
  mesh::k_nn_starts<<<(int)((ncells + 1 + 255) / 256), 256, 0, s>>>(scid, nr, ncells, starts);
  GSB_LAUNCHED();
  if (nq > 0) {
    mesh::k_nn_query<<<(int)((nq + 127) / 128), 128, 0, s>>>(query, nq, ref, order, starts, lo_host[0],
                                                             lo_host[1], lo_host[2], cell, nx, ny, nz,
                                                             out_d, out_i);
    GSB_LAUNCHED();
  }
  return GSB_OK;
}

__global__ void k_fill_u64(unsigned long long* p, int64_t n, unsigned long long v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

int gsb_raster_zbuffer(const double* u, const double* v, const double* z, const int64_t* faces,
                       int64_t n_faces, int32_t height, int32_t width, double* zbuf, void* stream) {
  if (!u || !v || !z || !faces || !zbuf || height <= 0 || width <= 0 || n_faces < 0) return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t np = (int64_t)height * width;
  unsigned long long* zb = reinterpret_cast<unsigned long long*>(zbuf);
  k_fill_u64<<<(int)((np + 255) / 256), 256, 0, s>>>(zb, np, 0x7ff0000000000000ull);  // +inf
  GSB_LAUNCHED();
  if (n_faces > 0) {
    mesh::k_raster_zbuffer<<<(int)((n_faces + 127) / 128), 128, 0, s>>>(u, v, z, faces, n_faces, height,
                                                                        width, zb);
    GSB_LAUNCHED();
  }
  return GSB_OK;
}

int gsb_sdf_fit_step(const gsb_model_t* model, const void* points, const void* targets,
                     int64_t n_batch, int64_t n_anchor, void* workspace, size_t workspace_bytes,
                     double* loss_out, void* stream) {
  if (!model || !points || !targets || !workspace) return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool f = model->precision == 0;
  switch (shape_tag(model)) {
    case 0:
      return f ? gsb_step_f446_sdf_fit(model, points, targets, n_batch, n_anchor, workspace,
                                       workspace_bytes, loss_out, s)
               : gsb_step_d446_sdf_fit(model, points, targets, n_batch, n_anchor, workspace,
                                       workspace_bytes, loss_out, s);
    case 1:
      return f ? gsb_step_f222_sdf_fit(model, points, targets, n_batch, n_anchor, workspace,
                                       workspace_bytes, loss_out, s)
               : gsb_step_d222_sdf_fit(model, points, targets, n_batch, n_anchor, workspace,
                                       workspace_bytes, loss_out, s);
    default:
      return GSB_E_ARG;
  }
}

int gsb_step_workspace_size(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse,
                            int32_t n_rounds, int32_t n_add, int32_t n_smooth, size_t* bytes) {
  if (!model || !bytes || n_rays <= 0 || n_coarse < 2 || n_rounds < 0 || n_add < 0) return GSB_E_ARG;
  if (n_coarse + n_rounds * n_add > GSB_KMAX || n_add > GSB_AMAX || n_rounds > GSB_MAX_ROUNDS)
    return GSB_E_ARG;
  Sizes z = sizes_of(model, n_rays, n_coarse, n_rounds, n_add, n_smooth);
  if (model->precision == 0)
    carve<float>(nullptr, z, bytes);
  else
    carve<double>(nullptr, z, bytes);
  return GSB_OK;
}

int gsb_step_workspace_layout(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse,
                              int32_t n_rounds, int32_t n_add, int32_t n_smooth,
                              int64_t* parts_off, int64_t* counts_off, int64_t* status_off,
                              int64_t* depths_off, int64_t* weights_off, int32_t* ld) {
  if (!model) return GSB_E_ARG;
  Sizes z = sizes_of(model, n_rays, n_coarse, n_rounds, n_add, n_smooth);
  size_t b = 0;
  if (model->precision == 0)
    carve<float>(nullptr, z, &b, parts_off, counts_off, status_off, depths_off, weights_off,
                 n_rounds);
  else
    carve<double>(nullptr, z, &b, parts_off, counts_off, status_off, depths_off, weights_off,
                  n_rounds);
  if (ld) *ld = z.ld;
  return GSB_OK;
}

int gsb_step_workspace_regions(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse,
                               int32_t n_rounds, int32_t n_add, int32_t n_smooth,
                               int64_t* offsets) {
  if (!model || !offsets) return GSB_E_ARG;
  Sizes z = sizes_of(model, n_rays, n_coarse, n_rounds, n_add, n_smooth);
  if (model->precision == 0)
    regions_of<float>(z, n_rounds, offsets);
  else
    regions_of<double>(z, n_rounds, offsets);
  return GSB_OK;
}

int gsb_train_step(const gsb_model_t* model, const gsb_dataset_t* data, const gsb_step_t* step,
                   void* stream) {
  if (!model || !data || !step || !step->workspace) return GSB_E_ARG;
  if (step->n_coarse + step->n_rounds * step->n_add > GSB_KMAX || step->n_add > GSB_AMAX ||
      step->n_rounds > GSB_MAX_ROUNDS || step->n_coarse < 2)
    return GSB_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (model->precision == 0) return dispatch_shape<float>(model, data, step, s);
  return dispatch_shape<double>(model, data, step, s);
}

int gsb_adam_step(int32_t precision, void* params, void* grads, void* m, void* v, int64_t n,
                  const int64_t* seg_begin_host, const double* seg_lr_host, int32_t n_seg,
                  double beta1, double beta2, double eps, double c1, double c2,
                  const double* guard, double guard_threshold, const int32_t* guard_status,
                  int32_t* status, void* stream) {
  if (n_seg < 1 || n_seg > GSB_ADAM_MAX_SEGS || !status) return GSB_E_ARG;
  AdamSegs sg;
  sg.n = n_seg;
  for (int i = 0; i < n_seg; ++i) {
    sg.begin[i] = seg_begin_host[i];
    sg.lr[i] = seg_lr_host[i];
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  AdamConst k;
  k.b1 = beta1;
  k.b2 = beta2;
  k.eps = eps;
  k.c1 = c1;
  k.c2 = c2;
  k.ib1 = 1.0 - beta1;  // same rounding as numba's (1.0 - b1)
  k.ib2 = 1.0 - beta2;
  k.inv_c1 = 1.0 / c1;
  k.inv_c2 = 1.0 / c2;
  // persistent grid: exactly the resident blocks (no partial last wave).
  // (Four vectors in flight per thread instead of two measured slower:
  // 437 vs 351 us at config 2.)
  // float32: 256-bit accesses (k_adam8) unless GSB_ADAM_V8=0 (A/B)
  static const bool v8 = [] {
    const char* e = std::getenv("GSB_ADAM_V8");
    return e ? std::atoi(e) != 0 : true;
  }();
  const bool use8 = precision == 0 && v8 &&
                    ((reinterpret_cast<uintptr_t>(params) | reinterpret_cast<uintptr_t>(grads) |
                      reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 31u) == 0;
  static int resident[3] = {0, 0, 0};
  int& res = resident[use8 ? 2 : (precision == 0 ? 0 : 1)];
  if (res == 0) {
    if (use8)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, k_adam8<>, 256, 0);
    else if (precision == 0)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, k_adam<float>, 256, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, k_adam<double>, 256, 0);
    if (res <= 0) res = 1;
  }
  int blocks = num_sms() * res;
  timing_point(nullptr, s);
  if (use8)
    k_adam8<><<<blocks, 256, 0, s>>>((float*)params, (float*)grads, (float*)m, (float*)v, n, sg,
                                     k, guard, guard_threshold, guard_status, status);
  else if (precision == 0)
    k_adam<float><<<blocks, 256, 0, s>>>((float*)params, (float*)grads, (float*)m, (float*)v, n, sg,
                                         k, guard, guard_threshold, guard_status, status);
  else
    k_adam<double><<<blocks, 256, 0, s>>>((double*)params, (double*)grads, (double*)m, (double*)v,
                                          n, sg, k, guard, guard_threshold, guard_status, status);
  GSB_LAUNCHED();
  timing_point("k_adam", s);
  return GSB_OK;
}

// ------------------------------------------------------------------ twins

__global__ void k_pcg_fill(gsb_pcg64_t rng, int64_t offset, int64_t n, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  Pcg g;
  g.init(rng);
  g.advance((uint64_t)(offset + i));
  out[i] = g.next_double();
}

int gsb_pcg64_random(const gsb_pcg64_t* rng, int64_t offset, int64_t n, double* out, void* stream) {
  if (!rng || n < 0) return GSB_E_ARG;
  if (n == 0) return GSB_OK;
  k_pcg_fill<<<(int)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      *rng, offset, n, out);
  GSB_LAUNCHED();
  return GSB_OK;
}

__global__ void k_ray_batch_twin(gsb_dataset_t D, const int64_t* ids, int n, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  PixelRay P = pixel_ray(D, ids[i]);
  double* o = out + (int64_t)i * 12;
  o[0] = (double)P.frame;
  o[1] = (double)P.u;
  o[2] = (double)P.v;
  o[3] = P.col[0];
  o[4] = P.col[1];
  o[5] = P.col[2];
  o[6] = P.depth_ray;
  o[7] = (double)P.valid;
  o[8] = P.dir[0];
  o[9] = P.dir[1];
  o[10] = P.dir[2];
  o[11] = P.scale;
}

int gsb_smooth_points(const gsb_model_t* model, const gsb_dataset_t* data, const double* poses,
                      const int64_t* row_cum, const int16_t* valid_u, const int64_t* pick,
                      const double* jitter, const double* normals, int32_t count, double delta,
                      void* out, void* stream) {
  if (!model || !data || !poses || !row_cum || !valid_u || !pick || !jitter || !normals || !out ||
      count < 0)
    return GSB_E_ARG;
  if (count == 0) return GSB_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n_rows = (int64_t)data->n_frames * data->height;
  const int blocks = (count + 127) / 128;
  if (model->precision == 0) {
    Geo G = geo_of(model, 4);
    k_smooth_points<float><<<blocks, 128, 0, s>>>(*data, poses, row_cum, n_rows, valid_u, pick, jitter,
                                                  normals, count, delta, G, (float*)out);
  } else {
    Geo G = geo_of(model, 8);
    k_smooth_points<double><<<blocks, 128, 0, s>>>(*data, poses, row_cum, n_rows, valid_u, pick,
                                                   jitter, normals, count, delta, G, (double*)out);
  }
  GSB_LAUNCHED();
  return GSB_OK;
}

int gsb_ray_batch(const gsb_dataset_t* data, const int64_t* ray_ids, int32_t n, double* out,
                  void* stream) {
  if (!data || n < 0) return GSB_E_ARG;
  if (n == 0) return GSB_OK;
  k_ray_batch_twin<<<(n + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      *data, ray_ids, n, out);
  GSB_LAUNCHED();
  return GSB_OK;
}

}  // extern "C"

template <typename T>
__global__ void k_gather_twin(const T* feat, int C, const int64_t* idx8, const double* w8,
                              int64_t n, T* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int c = 0; c < C; ++c) {
    T acc = T(0);
    for (int k = 0; k < 8; ++k)
      acc = (T)((double)acc + w8[i * 8 + k] * (double)feat[idx8[i * 8 + k] * C + c]);
    out[i * C + c] = acc;
  }
}

extern "C" {

int gsb_gather_weighted(int32_t precision, const void* feat, int32_t channels,
                        const int64_t* idx8, const double* w8, int64_t n, void* out,
                        void* stream) {
  if (n < 0 || channels <= 0) return GSB_E_ARG;
  if (n == 0) return GSB_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int b = (int)((n + 127) / 128);
  if (precision == 0)
    k_gather_twin<float><<<b, 128, 0, s>>>((const float*)feat, channels, idx8, w8, n, (float*)out);
  else
    k_gather_twin<double><<<b, 128, 0, s>>>((const double*)feat, channels, idx8, w8, n,
                                            (double*)out);
  GSB_LAUNCHED();
  return GSB_OK;
}

}  // extern "C"

template <typename T>
__global__ void k_scatter_twin(const int64_t* idx8, const double* w8, const T* g, int C, int64_t n,
                               T* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < 8; ++k)
    for (int c = 0; c < C; ++c)
      atomicAdd(out + idx8[i * 8 + k] * C + c, (T)(w8[i * 8 + k] * (double)g[i * C + c]));
}

extern "C" {

int gsb_scatter_weighted(int32_t precision, const int64_t* idx8, const double* w8, const void* g,
                         int32_t channels, int64_t n, void* out, void* stream) {
  if (n < 0 || channels <= 0) return GSB_E_ARG;
  if (n == 0) return GSB_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int b = (int)((n + 127) / 128);
  if (precision == 0)
    k_scatter_twin<float><<<b, 128, 0, s>>>(idx8, w8, (const float*)g, channels, n, (float*)out);
  else
    k_scatter_twin<double><<<b, 128, 0, s>>>(idx8, w8, (const double*)g, channels, n,
                                             (double*)out);
  GSB_LAUNCHED();
  return GSB_OK;
}

}  // extern "C"

template <typename T, int C>
__global__ void k_grid_sample_twin(LevelDev L, const T* pts, int64_t n, T* out, int32_t* status) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  Loc q = locate<true>(L, (double)pts[i * 3], (double)pts[i * 3 + 1], (double)pts[i * 3 + 2],
                       status);
  T v[C];
  gather_level<T, C, true>(L, q, v);
  for (int c = 0; c < C; ++c) out[i * C + c] = v[c];
}

extern "C" {

int gsb_grid_sample(int32_t precision, const gsb_level_t* level, const void* feat,
                    const void* points, int64_t n, void* out, int32_t* status, void* stream) {
  if (!level || n < 0) return GSB_E_ARG;
  if (n == 0) return GSB_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  gsb_level_t lv = *level;
  lv.offset = 0;
  size_t esz = precision == 0 ? 4 : 8;
  LevelDev L = level_dev(lv, const_cast<void*>(feat), nullptr, esz);
  int b = (int)((n + 127) / 128);
#define GSB_GS(TT, CC)                                                                        \
  k_grid_sample_twin<TT, CC><<<b, 128, 0, s>>>(L, (const TT*)points, n, (TT*)out, status); \
  break;
  if (precision == 0) {
    switch (level->channels) {
      case 1: GSB_GS(float, 1)
      case 2: GSB_GS(float, 2)
      case 4: GSB_GS(float, 4)
      case 6: GSB_GS(float, 6)
      default: return GSB_E_ARG;
    }
  } else {
    switch (level->channels) {
      case 1: GSB_GS(double, 1)
      case 2: GSB_GS(double, 2)
      case 4: GSB_GS(double, 4)
      case 6: GSB_GS(double, 6)
      default: return GSB_E_ARG;
    }
  }
#undef GSB_GS
  GSB_LAUNCHED();
  return GSB_OK;
}

int gsb_importance_round(int32_t n, int32_t K, int32_t A, int32_t ld, const double* depths,
                         const double* phi, double s, const double* nearv, const double* farv,
                         const double* uniforms, const gsb_pcg64_t* rng, double* depths_out,
                         int32_t* src_out, double* weights_out, void* stream) {
  if (n < 0 || K < 2 || A < 0 || A > GSB_AMAX || K + A > GSB_KMAX || ld < K + A) return GSB_E_ARG;
  if (!uniforms && !rng) return GSB_E_ARG;
  if (n == 0) return GSB_OK;
  gsb_pcg64_t g = {0, 0, 0, 0};
  if (rng) g = *rng;
  const size_t imp_smem = (size_t)kImpRaysPerBlock * imp_row_bytes(K + A, A);
  if (cudaFuncSetAttribute(k_importance_twin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)imp_smem) !=
      cudaSuccess)
    return GSB_E_CUDA;
  k_importance_twin<<<(n + kImpRaysPerBlock - 1) / kImpRaysPerBlock, 128, imp_smem,
                      reinterpret_cast<cudaStream_t>(stream)>>>(
      n, K, A, ld, depths, phi, nullptr, s, nearv, farv, uniforms, g, uniforms ? 0 : 1, depths_out,
      src_out, weights_out);
  GSB_LAUNCHED();
  return GSB_OK;
}

int gsb_importance_refine(int32_t n, int32_t K, int32_t A, int32_t ld, const double* depths,
                          const double* weights, const double* nearv, const double* farv,
                          const double* uniforms, double* depths_out, int32_t* src_out,
                          void* stream) {
  if (n < 0 || K < 2 || A < 0 || A > GSB_AMAX || K + A > GSB_KMAX || ld < K + A || !weights ||
      !uniforms)
    return GSB_E_ARG;
  if (n == 0) return GSB_OK;
  gsb_pcg64_t g = {0, 0, 0, 0};
  const size_t imp_smem = (size_t)kImpRaysPerBlock * imp_row_bytes(K + A, A);
  if (cudaFuncSetAttribute(k_importance_twin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)imp_smem) !=
      cudaSuccess)
    return GSB_E_CUDA;
  k_importance_twin<<<(n + kImpRaysPerBlock - 1) / kImpRaysPerBlock, 128, imp_smem,
                      reinterpret_cast<cudaStream_t>(stream)>>>(
      n, K, A, ld, depths, nullptr, weights, 0.0, nearv, farv, uniforms, g, 0, depths_out,
      src_out, nullptr);
  GSB_LAUNCHED();
  return GSB_OK;
}

}  // extern "C"
