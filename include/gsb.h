/*
 * gsb.h -- C ABI of the B200 GO-Surf training-step kernels.
 *
 * The reference (gridsurf, /root/reference/pkg/src/gridsurf) is pure Python
 * + numba; its native boundary is the set of numba kernels and the Python
 * step body (gs/optimizer.py:363-373).  This ABI replaces that boundary:
 *
 *   gsb_train_step  <- renderer.train_objective + dc.grad      (gs/renderer.py:279-468,
 *                                                               gs/diffcore.py:1035-1104)
 *   gsb_adam_step   <- optimizer.Adam.step / _adam_kernel       (gs/optimizer.py:38-91)
 *   unit twins of the numba kernels, used by the parity tests:
 *   gsb_gather_weighted   <- diffcore._nb_gather_weighted       (gs/diffcore.py:816-827)
 *   gsb_scatter_weighted  <- diffcore._nb_scatter_weighted      (gs/diffcore.py:830-841)
 *   gsb_grid_sample       <- diffcore.grid_sample (forward)     (gs/diffcore.py:893-920)
 *   gsb_importance_round  <- render_weights_data + importance_refine_with_sources
 *                            (gs/renderer.py:162-173, gs/sampler.py:128-197)
 *   gsb_ray_batch         <- sampler.draw_ray_batch (given drawn ids) (gs/sampler.py:58-88)
 *   gsb_pcg64_random      <- numpy Generator(PCG64).random       (gs/seeds.py:28-30)
 *
 * Conventions: every pointer is a DEVICE pointer unless named *_host; the
 * caller owns all memory (kernels never allocate); every launch is
 * asynchronous on `stream` (a cudaStream_t passed as void*); functions return
 * GSB_OK or a negative status.  Data-dependent errors (a point outside the
 * grid, non-finite values, list overflow) are written to the status words in
 * the step workspace and surface at the caller's next synchronisation.
 */
#ifndef GSB_H
#define GSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSB_OK 0
#define GSB_E_ARG (-1)      /* bad argument / unsupported configuration */
#define GSB_E_CUDA (-2)     /* a CUDA runtime call failed */
#define GSB_E_BOUNDS (-3)   /* GridBoundsError (gs/diffcore.py:738-751) */
#define GSB_E_NONFINITE (-4)

#define GSB_MAX_LEVELS 8
#define GSB_MAX_ROUNDS 8
#define GSB_KMAX 256        /* max samples per ray */
#define GSB_AMAX 32         /* max importance samples added per round */

/* status word indices in the step workspace (int32) */
#define GSB_ST_BOUNDS 0
#define GSB_ST_NONFINITE 1
#define GSB_ST_OVERFLOW 2
#define GSB_ST_VIEWDIR 3
#define GSB_ST_ADAM_BAD 4
#define GSB_ST_DIVERGED 5
#define GSB_N_STATUS 8

/* loss-part slots (double) written by gsb_train_step */
#define GSB_P_TOTAL 0
#define GSB_P_RGB 1
#define GSB_P_DEPTH 2
#define GSB_P_SDF 3
#define GSB_P_FS 4
#define GSB_P_EIK 5
#define GSB_P_SMOOTH 6
#define GSB_P_S 7
#define GSB_N_PARTS 8

/* count slots (int64) */
#define GSB_C_VALID 0
#define GSB_C_TR 1
#define GSB_C_FS 2
#define GSB_C_EIK 3
#define GSB_N_COUNTS 4

/* One dense vertex lattice (diffcore.GridGeom, gs/diffcore.py:704-728) plus
 * where its features live in the parameter arena. */
typedef struct {
  int32_t nx, ny, nz;   /* vertex counts */
  int32_t channels;     /* feature width C */
  double ox, oy, oz;    /* world position of vertex (0,0,0) */
  double voxel;         /* isotropic edge length */
  int64_t offset;       /* element offset of the (V, C) block in the arena */
} gsb_level_t;

/* The model: grids coarse->fine + colour grid, MLP block, log_s
 * (renderer.ModelState, gs/renderer.py:69-105). */
typedef struct {
  int32_t precision;    /* 0: float32 storage/compute, 1: float64 */
  int32_t n_levels;     /* geometry levels */
  gsb_level_t levels[GSB_MAX_LEVELS];
  gsb_level_t color;
  int64_t mlp_offset;   /* geom W0,b0,W1,b1,W2,b2 then colour W0..b2, contiguous */
  int64_t log_s_offset;
  int64_t n_params;     /* arena length in elements */
  double lo_c[3], hi_c[3]; /* box shrunk by half the finest voxel (gs/renderer.py:299-300) */
  void* params;         /* arena (T*) */
  void* grads;          /* gradient arena, same layout (T*) */
} gsb_model_t;

/* Device-resident RGB-D dataset: colours u8 (F,H,W,3) = round(255 c),
 * depths u16 (F,H,W) millimetres = round(1000 z) (gs/scenegen.py:319-320). */
typedef struct {
  const uint8_t* colors;
  const uint16_t* depth_mm;
  int32_t n_frames, height, width;
  double fx, fy, cx, cy;
  const double* poses;  /* (F, 12): R row-major then t, values already rounded to
                           the model dtype (PoseParam stores them in dtype) */
} gsb_dataset_t;

/* Camera poses under refinement (camera.PoseParam, gs/camera.py:53-90): frame f
 * has base rotation R0_f (f64) and, when trainable, nu_f / t_f in the
 * parameter arena (gs/optimizer.py:217-226 names them nu{f}, t{f}). */
typedef struct {
  int32_t n_frames;
  const double* R0;          /* (F, 9) row-major, device */
  const int64_t* nu_offset;  /* (F) element offset of nu_f in the arena, -1: frozen (nu = 0) */
  const int64_t* t_offset;   /* (F) element offset of t_f, -1: frozen (t_fixed) */
  const double* t_fixed;     /* (F, 3) translations of frozen frames (dtype-rounded), device */
} gsb_pose_t;

/* Analytic CSG scene (scenegen.AnalyticScene, gs/scenegen.py:41-155) flattened
 * into a postfix program: op (0 PUSH prim k | 1 NEG | 2 MIN over the top n).
 * prim row: type (0 sphere, 1 box), centre[3], radius | half[3], albedo[3],
 * albedo2[3], checker (m, 0 = solid). */
#define GSB_SCENE_MAX_PRIMS 16
#define GSB_SCENE_MAX_OPS 32
#define GSB_SCENE_MAX_STACK 8
typedef struct {
  int32_t n_prims, n_ops;
  double prim[GSB_SCENE_MAX_PRIMS][16];
  int32_t op[GSB_SCENE_MAX_OPS][2];
  double light[3];       /* unit, from the light toward the scene */
  double background[3];  /* RGB of rays that miss */
} gsb_scene_t;

/* Depth corruptions of scenegen.render_dataset (gs/scenegen.py:328-343). */
typedef struct {
  int32_t rect[4];       /* x0, y0, x1, y1 pixel rectangle zeroed in every frame (x1 <= x0: none) */
  double world_c[3];     /* world-space ball ... */
  double world_r;        /* ... of this radius (<= 0: none) */
  int32_t has_box;       /* world-space box lo..hi */
  double box_lo[3], box_hi[3];
} gsb_render_opts_t;

typedef struct {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;  /* numpy PCG64 bit_generator state */
} gsb_pcg64_t;

typedef struct {
  /* batch (sampler.draw_ray_batch): drawn flat ids into F*H*W */
  const int64_t* ray_ids;
  int32_t n_rays;            /* rays on this rank */
  int32_t ray_base;          /* global row of this rank's first ray (RNG offset) */
  double m_global;           /* global batch size M (loss normaliser) */
  /* sampling (TrainConfig) */
  int32_t n_coarse, n_rounds, n_add;
  int32_t has_fixed_far;
  double near, max_depth, fixed_far;
  gsb_pcg64_t rng_stratify;
  gsb_pcg64_t rng_importance[GSB_MAX_ROUNDS];
  /* LossWeights (gs/renderer.py:46-66) */
  double w_rgb, w_depth, w_sdf, w_fs, w_eik, w_smooth;
  double truncation, fs_alpha;
  /* smoothness points (x then x+eps), (2*n_smooth, 3) model dtype */
  const void* smooth_pts;
  int32_t n_smooth;          /* pairs on this rank */
  double smooth_global;      /* global pair count (normaliser) */
  /* behaviour */
  int32_t exact_gather;      /* reserved (0): the step gathers with FMAs; the per-corner
                                rounding of numba is gsb_gather_weighted (exact twin) */
  int32_t phases;            /* bit0: sampling+counts, bit1: objective+backward+finalize;
                                bit2 / bit3 with bit1: only part A (taped forward, render,
                                geometry backward) / only part B (colour backward, finalize) */
  /* workspace (see gsb_step_workspace_size) */
  void* workspace;
  size_t workspace_bytes;
  /* pose refinement: the gsb_pose_grad scratch (gsb_pose_scratch_size bytes),
   * or NULL.  In float32 mode the step then also leaves each taped sample's
   * dphi/dz and colour-input cotangent there for gsb_pose_grad. */
  void* pose_work;
  size_t pose_work_bytes;
  /* deterministic scatter mode (validation): gsb_det_scratch_size bytes, or
   * NULL.  The grid-gradient scatters then record (row, value) entries that
   * are stably sorted by row and summed in sample order, so the gradients are
   * bit-reproducible run to run (the default mode uses warp-aggregated
   * atomics).  MLP partials are then per-CTA rows reduced in a fixed order. */
  void* det_work;
  size_t det_work_bytes;
} gsb_step_t;

int gsb_version(void);

/* Number of kernels this library has launched in the process (all entry
 * points).  Bench/diagnostic counter; no reference counterpart. */
uint64_t gsb_launch_count(void);

/* Opt-in per-kernel timing for benchmarks: while enabled, gsb_train_step and
 * gsb_adam_step record a CUDA event on their stream after every launch.
 * gsb_timing_collect synchronises, returns per-kernel-name total milliseconds
 * and launch counts (names: max_kernels x 64 chars), and resets the marks. */
int gsb_timing_enable(int32_t on);
int gsb_timing_collect(int32_t max_kernels, char* names, double* total_ms, int64_t* launches,
                       int32_t* n_kernels);

/* Bytes of device workspace gsb_train_step needs. */
int gsb_step_workspace_size(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse,
                            int32_t n_rounds, int32_t n_add, int32_t n_smooth,
                            size_t* bytes);

/* Offsets (bytes) of the externally visible workspace regions:
 * parts (double[GSB_N_PARTS]), counts (int64[GSB_N_COUNTS]), status
 * (int32[GSB_N_STATUS]), final depths (double, [n_rays][ld]), weights (model
 * dtype, [n_rays][ld]), ld. */
int gsb_step_workspace_layout(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse,
                              int32_t n_rounds, int32_t n_add, int32_t n_smooth,
                              int64_t* parts_off, int64_t* counts_off, int64_t* status_off,
                              int64_t* depths_off, int64_t* weights_off, int32_t* ld);

/* Byte offsets of internal workspace arrays (for parity tests / debugging). */
#define GSB_R_PARTS 0    /* double[GSB_N_PARTS] */
#define GSB_R_COUNTS 1   /* int64[GSB_N_COUNTS] */
#define GSB_R_STATUS 2   /* int32[GSB_N_STATUS] */
#define GSB_R_DEPTHS 3   /* double [n_rays][ld] final sample depths */
#define GSB_R_WEIGHTS 4  /* T [n_rays][N] rendering weights */
#define GSB_R_PHI 5      /* T [n_rays*N + 2*n_smooth] */
#define GSB_R_GPHI 6     /* T [.. ][3] */
#define GSB_R_COLOR 7    /* T [n_rays*N][3] */
#define GSB_R_PBAR 8     /* T [n_rays*N + 2*n_smooth]  d total / d phi */
#define GSB_R_UBAR 9     /* T [..][3]                 d total / d grad phi */
#define GSB_R_CBAR 10    /* T [n_rays*N][3]           d total / d colour */
#define GSB_R_RAY_O 11   /* T [n_rays][3] */
#define GSB_R_RAY_R 12   /* T [n_rays][3] */
#define GSB_R_RAY_FAR 13 /* double [n_rays] */
#define GSB_N_REGIONS 14
int gsb_step_workspace_regions(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse,
                               int32_t n_rounds, int32_t n_add, int32_t n_smooth,
                               int64_t* offsets);

/* One training objective + full backward; gradients are ACCUMULATED into
 * model->grads (gsb_adam_step leaves them zeroed). */
int gsb_train_step(const gsb_model_t* model, const gsb_dataset_t* data, const gsb_step_t* step,
                   void* stream);

/* Pose refinement.
 * gsb_pose_table: realised poses of the current parameters: table (F, 12) =
 *   R0c exp_so3(nu) evaluated in the model dtype as the reference's graph does
 *   (PoseParam.rotation, gs/camera.py:68-70, 96-122) and t -- the ray table
 *   gsb_dataset_t.poses expects -- and table_f64 (F, 12) = R0 exp_so3_data(nu)
 *   in float64 (PoseParam.matrix, gs/camera.py:75-80), the smoothness-point table.
 * gsb_pose_grad: after gsb_train_step (same model / data / step arguments),
 *   ACCUMULATES d total / d nu_f and d total / d t_f of every trainable frame
 *   into model->grads: the tracked-point cotangent of each taped sample (phi,
 *   grad-phi Hessian block, colour; gs/diffcore.py:893-991), the clip mask,
 *   x = o + d r, r = R dir_cam per frame, and the exp_so3 adjoint.  Scratch:
 *   gsb_pose_scratch_size bytes. */
int gsb_det_scratch_size(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse, int32_t n_rounds,
                         int32_t n_add, int32_t n_smooth, size_t* bytes);
int gsb_pose_table(const gsb_model_t* model, const gsb_pose_t* pose, double* table, double* table_f64,
                   void* stream);
int gsb_pose_scratch_size(const gsb_model_t* model, int32_t n_rays, int32_t n_coarse, int32_t n_rounds,
                          int32_t n_add, size_t* bytes);
int gsb_pose_grad(const gsb_model_t* model, const gsb_dataset_t* data, const gsb_step_t* step,
                  const gsb_pose_t* pose, void* scratch, size_t scratch_bytes, void* stream);

/* Synthetic RGB-D frames: scenegen._render_frame
 * (gs/scenegen.py:290-325) for n_frames camera-to-world poses (device, (F, 16)
 * row-major f64), one thread per pixel: pixel rays, sphere tracing (tol 1e-6,
 * 256 steps, max_t), Lambert shading, optional Gaussian depth noise
 * sigma0 z^2 with the caller's standard normals (device (F, H, W) f64, drawn
 * from seeds.substream(seed, DEPTH_NOISE, f) on the host) and dropouts;
 * writes u8 colours (F, H, W, 3) = round(255 c) and u16 depth (F, H, W) =
 * round(1000 z) straight into the device dataset layout. */
int gsb_render_frames(const gsb_scene_t* scene, const double* poses, int32_t n_frames, int32_t height,
                      int32_t width, double fx, double fy, double cx, double cy, double max_t,
                      const double* noise, double sigma0, const gsb_render_opts_t* opts, uint8_t* colors,
                      uint16_t* depth_mm, void* stream);

/* Dense Adam over the whole arena (gs/optimizer.py:38-55, replaces
 * Adam.step / _adam_kernel): per segment learning rate (n_seg <= 32 runs
 * starting at seg_begin_host[i]); float64 register math; grads zeroed
 * afterwards.  A segment with a negative learning rate is not owned by this
 * launch (a data-parallel rank's foreign shards): its gradients are zeroed
 * and p / m / v are untouched.  The update is skipped, and
 * status[GSB_ST_DIVERGED] set (which skips every later guarded update), if
 * `guard` is non-null and guard[0] (total loss) is non-finite or
 * > guard_threshold (gs/optimizer.py:368-371), or `guard_status` (the step's
 * status words) is non-null and carries a bounds / overflow / view-direction
 * error (raised inside train_objective by the reference). */
int gsb_adam_step(int32_t precision, void* params, void* grads, void* m, void* v,
                  int64_t n, const int64_t* seg_begin_host, const double* seg_lr_host,
                  int32_t n_seg, double beta1, double beta2, double eps, double c1, double c2,
                  const double* guard, double guard_threshold, const int32_t* guard_status,
                  int32_t* status, void* stream);

/* Smoothness points (renderer.draw_smooth_points, gs/renderer.py:243-276) on
 * the device from the host's RNG draws, in the reference's call order:
 * pick = integers(0, n_valid, count) (index into the valid-depth pixels in
 * np.nonzero order), jitter = uniform(-truncation, truncation, count),
 * normals = normal((count, 8, 3)).  poses: (F, 12) f64 rows of
 * ModelState.pose_matrices() (R row-major, then t); row_cum: (F*H) inclusive
 * prefix counts of valid pixels per image row; valid_u: (F*H, W) int16, row r's
 * valid columns in increasing order in its first row_cum[r]-row_cum[r-1]
 * entries (the per-row compaction of Dataset.valid_pixels, gs/scenegen.py:281-287).
 * out: (2*count, 3) model dtype, x then x + eps, clamped to model->lo_c/hi_c.
 * Bit-exact with the reference. */
int gsb_smooth_points(const gsb_model_t* model, const gsb_dataset_t* data, const double* poses,
                      const int64_t* row_cum, const int16_t* valid_u, const int64_t* pick,
                      const double* jitter, const double* normals, int32_t count, double delta,
                      void* out, void* stream);

/* ---------------- geometry on point lists ---------------- */

/* Bytes of device workspace gsb_sdf_points / gsb_sdf_fit_step need for up to
 * n_points points. */
int gsb_sdf_workspace_size(const gsb_model_t* model, int64_t n_points, size_t* bytes);

/* phi at n points (model dtype, (n, 3) -> (n,)), no grad: the geometry decoder
 * on the multi-level grid (renderer._phi_data / decoders.decode_sdf on
 * feature_grid.sample_multi, gs/renderer.py:236-240, gs/decoders.py:79-83). */
int gsb_sdf_points(const gsb_model_t* model, const void* points, int64_t n, void* phi_out,
                   void* workspace, size_t workspace_bytes, void* stream);

/* One step of the sphere pre-fit (decoders.geometric_init inner loop,
 * gs/decoders.py:160-167): points = n_batch uniform points then n_anchor
 * anchors, targets their SDF (model dtype).  ADDS d/dtheta [mean_batch (phi-t)^2
 * + mean_anchor (phi-t)^2] into the geometry levels' and geometry decoder's
 * gradients (caller zeroes them); colour gradients are untouched.  The loss
 * (double) is written to *loss_out (device pointer, may be NULL). */
int gsb_sdf_fit_step(const gsb_model_t* model, const void* points, const void* targets,
                     int64_t n_batch, int64_t n_anchor, void* workspace, size_t workspace_bytes,
                     double* loss_out, void* stream);

/* ---------------- mesh extraction and metrics (gs/mesher.py) ---------------- */

/* Dense SDF volume (mesher.sdf_volume, gs/mesher.py:114-133): vertex (i,j,k)
 * at lo + (i,j,k) * resolution (f64, then the model dtype), phi stored as
 * float32 in vol[(i * ny + j) * nz + k]. */
int gsb_sdf_volume_workspace_size(const gsb_model_t* model, size_t* bytes);
int gsb_sdf_volume(const gsb_model_t* model, const double* lo_host, double resolution, int64_t nx,
                   int64_t ny, int64_t nz, float* vol, void* workspace, size_t workspace_bytes,
                   void* stream);

/* Marching cubes (mesher.mesh_from_sdf, gs/mesher.py:136-146) with the
 * generated 256-case table (mc_table.py; table = packed int8 ntri[256] |
 * tri[256][16] | edge corners[12][2], device).  gsb_mc_count writes the
 * triangle total (int64) and the volume min/max (2 floats) to device memory;
 * gsb_mc_emit then writes 3 f64 vertices per triangle (verts: 9 * total)
 * and, if `keys` is non-null, each vertex's lattice-edge key (3 * total
 * int64: ((i ny + j) nz + k) 3 + axis of the edge's lower end point); equal
 * keys are bit-identical vertices, which the caller welds. */
int gsb_mc_workspace_size(int64_t nx, int64_t ny, int64_t nz, size_t* bytes);
int gsb_mc_count(const float* vol, int64_t nx, int64_t ny, int64_t nz, float level, const int8_t* table,
                 void* workspace, size_t workspace_bytes, int64_t* total, float* minmax, void* stream);
int gsb_mc_emit(const float* vol, int64_t nx, int64_t ny, int64_t nz, float level, double ox, double oy,
                double oz, double resolution, const int8_t* table, void* workspace,
                size_t workspace_bytes, double* verts, int64_t* keys, void* stream);

/* Exact nearest neighbour from each query into ref (mesher.nearest_neighbors,
 * gs/mesher.py:302-363): the same cell hash (lo, cell, dims computed by the
 * caller as the reference does), ring order and early-out, so distances and
 * tie-broken indices equal the reference's. */
int gsb_nn_workspace_size(int64_t n_ref, int64_t nx, int64_t ny, int64_t nz, size_t* bytes);
int gsb_nearest_neighbors(const double* query, int64_t nq, const double* ref, int64_t nr,
                          const double* lo_host, double cell, int64_t nx, int64_t ny, int64_t nz,
                          void* workspace, size_t workspace_bytes, double* out_d, int64_t* out_i,
                          void* stream);

/* Min-z buffer of a mesh in one camera (mesher._raster_zbuffer,
 * gs/mesher.py:198-229): u, v, z per vertex (f64, device), faces (F, 3) int64;
 * zbuf (height, width) f64 = +inf where nothing is drawn. */
int gsb_raster_zbuffer(const double* u, const double* v, const double* z, const int64_t* faces,
                       int64_t n_faces, int32_t height, int32_t width, double* zbuf, void* stream);

/* ---------------- unit twins (parity tests) ---------------- */

int gsb_pcg64_random(const gsb_pcg64_t* rng, int64_t offset, int64_t n, double* out,
                     void* stream);

/* out (n, 12) f64: frame, u, v, r, g, b, depth_ray, valid, dir x, y, z, scale */
int gsb_ray_batch(const gsb_dataset_t* data, const int64_t* ray_ids, int32_t n, double* out,
                  void* stream);

int gsb_gather_weighted(int32_t precision, const void* feat, int32_t channels,
                        const int64_t* idx8, const double* w8, int64_t n, void* out,
                        void* stream);

int gsb_scatter_weighted(int32_t precision, const int64_t* idx8, const double* w8,
                         const void* g, int32_t channels, int64_t n, void* out, void* stream);

/* points (n,3) model dtype -> features (n,C); exact locate + numba rounding */
int gsb_grid_sample(int32_t precision, const gsb_level_t* level, const void* feat,
                    const void* points, int64_t n, void* out, int32_t* status, void* stream);

/* One importance round for n rays with K current samples (row stride ld):
 * weights from phi (render_weights_data), inverse-CDF draws from `uniforms`
 * (n, A) or, if null, from `rng`, stable merge, separation, provenance. */
int gsb_importance_round(int32_t n, int32_t K, int32_t A, int32_t ld, const double* depths,
                         const double* phi, double s, const double* near, const double* far,
                         const double* uniforms, const gsb_pcg64_t* rng, double* depths_out,
                         int32_t* src_out, double* weights_out, void* stream);

/* sampler.importance_refine_with_sources (gs/sampler.py:128-169) exactly as
 * the reference defines it: given depths (n,K), weights (n,K) and uniforms
 * (n,A) -> merged depths (n,K+A) and provenance (-1 = new/moved). */
int gsb_importance_refine(int32_t n, int32_t K, int32_t A, int32_t ld, const double* depths,
                          const double* weights, const double* near, const double* far,
                          const double* uniforms, double* depths_out, int32_t* src_out,
                          void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GSB_H */
