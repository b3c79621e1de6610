// gsb_step_inst.cu -- compiled once per (dtype, grid shape); see build.py.
#include "gsb_step.cuh"

#ifndef GSB_T
#error "define GSB_T, GSB_NL, GSB_CG, GSB_CC, GSB_ENTRY"
#endif

extern "C" int GSB_ENTRY(const gsb_model_t* m, const gsb_dataset_t* d, const gsb_step_t* st,
                         cudaStream_t s) {
  return gsb::host::run_step<GSB_T, gsb::Shape<GSB_NL, GSB_CG, GSB_CC>>(m, d, st, s);
}

#define GSB_CAT2(a, b) a##b
#define GSB_CAT(a, b) GSB_CAT2(a, b)

extern "C" int GSB_CAT(GSB_ENTRY, _sdf_points)(const gsb_model_t* m, const void* pts, int64_t n,
                                               void* phi, void* ws, size_t ws_bytes, cudaStream_t s) {
  return gsb::host::run_sdf_points<GSB_T, gsb::Shape<GSB_NL, GSB_CG, GSB_CC>>(m, pts, n, phi, ws,
                                                                              ws_bytes, s);
}

extern "C" int GSB_CAT(GSB_ENTRY, _sdf_fit)(const gsb_model_t* m, const void* pts, const void* tgt,
                                            int64_t nb, int64_t na, void* ws, size_t ws_bytes,
                                            double* loss, cudaStream_t s) {
  return gsb::host::run_sdf_fit<GSB_T, gsb::Shape<GSB_NL, GSB_CG, GSB_CC>>(m, pts, tgt, nb, na, ws,
                                                                           ws_bytes, loss, s);
}

extern "C" int GSB_CAT(GSB_ENTRY, _sdf_volume)(const gsb_model_t* m, const double* lo, double res,
                                               int64_t nx, int64_t ny, int64_t nz, float* vol, void* ws,
                                               size_t ws_bytes, cudaStream_t s) {
  return gsb::host::run_sdf_volume<GSB_T, gsb::Shape<GSB_NL, GSB_CG, GSB_CC>>(m, lo, res, nx, ny, nz, vol,
                                                                              ws, ws_bytes, s);
}

extern "C" int GSB_CAT(GSB_ENTRY, _pose_grad)(const gsb_model_t* m, const gsb_dataset_t* d, const gsb_step_t* st,
                                              const gsb_pose_t* pose, void* scratch, size_t scratch_bytes,
                                              cudaStream_t s) {
  return gsb::host::run_pose_grad<GSB_T, gsb::Shape<GSB_NL, GSB_CG, GSB_CC>>(m, d, st, pose, scratch,
                                                                             scratch_bytes, s);
}
