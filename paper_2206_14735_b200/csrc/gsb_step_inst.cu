// gsb_step_inst.cu -- compiled once per (dtype, grid shape); see build.py.
#include "gsb_step.cuh"

#ifndef GSB_T
#error "define GSB_T, GSB_NL, GSB_CG, GSB_CC, GSB_ENTRY"
#endif

extern "C" int GSB_ENTRY(const gsb_model_t* m, const gsb_dataset_t* d, const gsb_step_t* st,
                         cudaStream_t s) {
  return gsb::host::run_step<GSB_T, gsb::Shape<GSB_NL, GSB_CG, GSB_CC>>(m, d, st, s);
}
