/*
 * nirc_b200.h — C ABI of the B200 (sm_100a) Neural Incident Radiance Cache
 * hot path.  Every entry point is `extern "C"`, takes plain pointers and
 * sizes, returns an int status and is stream-ordered on the `cudaStream_t`
 * passed last (as `void*`, so the header needs no CUDA include).  All data
 * pointers are DEVICE pointers unless a parameter name ends in `_host`.
 *
 * The reference (`nirclab`, pure Python + numba) has no FFI; the boundary
 * it replaces is its Python module API and the `jit_kernel` backend seam
 * (pkg/src/nirclab/backend.py:27-49).  Each entry point below names the
 * reference function it stands in for.  The Python shim in
 * `paper_2412_04634_b200/` binds these with ctypes and keeps the
 * reference's signatures; INTEGRATION.md shows the binding.
 *
 * Ownership: the caller (torch) owns every buffer.  The library keeps no
 * global state except per-device cached weight images.
 */
#ifndef NIRC_B200_H
#define NIRC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NIRC_MAX_LAYERS 9
#define NIRC_MAX_LEVELS 16
#define NIRC_MAX_BANDS 8

/* Status codes.  The shim maps them onto the reference's exceptions
 * (pkg/src/nirclab/errors.py:8-33): CONFIG -> ConfigError,
 * DIVERGENCE -> DivergenceError, BAD_PDF -> InvalidSampleError. */
enum {
  NIRC_OK = 0,
  NIRC_E_CONFIG = 2,
  NIRC_E_DIVERGENCE = 3,
  NIRC_E_BAD_PDF = 4,
  NIRC_E_CUDA = 5,
  NIRC_E_UNSUPPORTED = 6
};

/* Bits of the device-side status word (`int32_t* status_flags`) that the
 * asynchronous entries set instead of returning; the shim reads it with the
 * call's results and raises the matching exception. */
#define NIRC_FLAG_BAD_PDF 1     /* InvalidSampleError (losses.py:18-20) */
#define NIRC_FLAG_DIVERGED 2    /* DivergenceError: non-finite loss or theta (mlp.py:104-105) */
#define NIRC_FLAG_BAD_INDEX 4   /* ConfigError: dir_to_surf index outside [0, n_surf) */

/* Network layout; mirrors NetSpec (pkg/src/nirclab/mlp.py:26-62).
 * theta = [hash tables (levels*2^table_log2*feats)] ++ per layer W (dout x din,
 * row-major) ++ b.  sh_k[l*8+m] holds NORM[l,0] for m == 0 and
 * sqrt(2)*NORM[l,m] for m > 0 (pkg/src/nirclab/sh.py:21-33), computed on
 * the host with the reference's expression order. */
typedef struct nirc_spec {
  int32_t levels, table_log2, feats, bands, in_dim, n_layers, out_act, pad0;
  int32_t dims[NIRC_MAX_LAYERS + 1];
  int32_t pad1[2];
  int64_t w_off[NIRC_MAX_LAYERS];
  int64_t b_off[NIRC_MAX_LAYERS];
  int32_t res[NIRC_MAX_LEVELS];
  double bb_min[3];
  double bb_inv[3];
  int64_t grid_len, theta_len;
  double sh_k[64];
} nirc_spec_t;

/* Flat scene, mirrors ScnPack (pkg/src/nirclab/scene.py:42-53).  All arrays
 * are device pointers, f64 unless noted; vectors are (n,3) row-major. */
typedef struct nirc_scene {
  int32_t n_tri, n_sph, n_mat, n_light, n_bvh, env_kind, env_h, env_w;
  const double *tri_v0, *tri_e1, *tri_e2, *tri_ng, *tri_area, *tri_lq;
  const int32_t *tri_mat;
  const double *sph_c, *sph_r, *sph_lq;
  const int32_t *sph_mat;
  const int32_t *mat_kind;
  const double *mat_albedo, *mat_rough, *mat_emit;
  const int32_t *lt_kind, *lt_prim;
  const double *lt_cdf, *lt_q;
  const double *env_img;             /* (env_h, env_w, 3) */
  double env_c0[3], env_c1[3], env_c2[3];
  double env_q, eps, diag;
  double bbox_min[3], bbox_inv_ext[3];
  const double *bvh_lo, *bvh_hi;
  const int32_t *bvh_a, *bvh_b, *bvh_prim;
  const float* tri_f32;  /* kernel-private scratch (the staged fp32 triangle
                            filter table); callers pass NULL */
  /* Optional traversal image from nirc_pack_scene (NULL: the kernels walk
   * the bvh_* arrays directly).  Scenes past the warp-uniform scan size
   * traverse it front to back. */
  const void* bvh_packed;
  const void* prim_packed;
  /* Optional fp32 pre-test items for the warp-uniform scan of small
   * triangle-only scenes (NULL: one item per triangle, built in-kernel):
   * n_filter rows of 16 floats -- (v0.xyz, |e1|_1), (e1.xyz, |e2|_1),
   * (e2.xyz, |v0|_1), (cu, slack, mask_lo, mask_hi) -- the 64-bit mask of
   * the scan positions the item covers, as two u32 bit patterns:
   * a triangle (cu = 1) or a parallelogram covering two scan-order
   * triangles that share v0 and their diagonal (cu = 0). */
  const float* filter_items;
  int32_t n_filter;
  int32_t pad_filter;
} nirc_scene_t;

/* Two-level estimator knobs; mirrors EstimatorConfig
 * (pkg/src/nirclab/estimators.py:49-84) as consumed by render_kernel
 * (pkg/src/nirclab/kernels.py:723-759). */
typedef struct nirc_render_cfg {
  int32_t mode;          /* 0 = pt, 1 = two-level, 2 = biased-nirc-bth,
                            3 = biased-nirc-sph, 4 = biased-nrc-sph
                            (kernels.py:37-41) */
  int32_t spp;
  int32_t cache_on;      /* 0: cache skipped (is_zero and not forced) */
  int32_t max_cv;
  int32_t nc[8];         /* nc[:max_cv], each 0..28 */
  double rough_cut;
  double rr_survive;     /* 1 - EstimatorConfig.rr */
  uint64_t seed, frame;
  int32_t width, height; /* camera resolution */
  int32_t row0, row1;    /* pixel-row band [row0, row1) rendered by this call */
  int32_t precision;     /* network arithmetic: 0 tcgen05 3xTF32, 1 fp32 SIMT,
                            2 tcgen05 2xFP16 split (default) */
  int32_t nbias;         /* cache directions at a biased stop vertex (1..28) */
  double sph_c;          /* spread threshold of the *_sph / bth stop tests */
  const uint8_t* v1;     /* (height*width) per-pixel first-vertex stop flags of
                            the *_sph modes, or NULL (all zero) */
} nirc_render_cfg_t;

/* ---- library / introspection ------------------------------------------ */
const char* nirc_version(void);
int nirc_last_error(char* buf, int buflen);
int nirc_device_sm_count(void);
/* Measurement (bench.py): with stage timing on, every render records CUDA
 * events on its stream around the tracer, the fused inference (+ fp16
 * fix-up) and the accumulation; nirc_stage_times writes the last timed
 * render's [trace, inference, accumulate] milliseconds (waits for it).
 * Not part of the reference's interface. */
int nirc_stage_timing(int32_t on);
int nirc_stage_times(float* ms, int32_t n);

/* ---- encoding (pkg/src/nirclab/encoding.py) ----------------------------- */
/* encode_batch (encoding.py:111-157): X (n,in_dim) f32, entries (n,levels,8)
 * i64 slots, weights (n,levels,8) f32.  entries/weights may be NULL. */
int nirc_encode(const nirc_spec_t* spec, const float* theta,
                const double* pos, const double* normal, const double* albedo,
                const double* rough, const double* dirs, int64_t n,
                float* X, int64_t* entries, float* weights, void* stream);

/* scatter_grid_grad (encoding.py:160-167): grad[slot*F+f] += w * dX[:, l*F+f]
 * with np.add.at's semantics: each slot sums its contributions in entry order
 * ((row, level, corner) row-major) from its current value -- a stable radix
 * sort of (slot, entry) then one sequential sum per slot.  Deterministic, and
 * bit-identical to the reference for identical weights and dX. */
int nirc_scatter_grid_grad(const nirc_spec_t* spec, float* grad,
                           const int64_t* entries, const float* weights,
                           const float* dX, int64_t n, int64_t dx_stride,
                           void* stream);

/* ---- network (pkg/src/nirclab/mlp.py) ----------------------------------- */
/* mlp_forward (mlp.py:102-122), fp32 SIMT twin.  zs (n, sum(dims[1:])) f32 is
 * the training cache (pre-activations per layer), NULL for inference.
 * finite_flag (i32, may be NULL) is set to 1 when theta holds a non-finite
 * value (DivergenceError in the reference). */
int nirc_mlp_forward(const nirc_spec_t* spec, const float* theta,
                     const float* X, int64_t n, float* Y, float* zs,
                     int32_t* nonfinite_flag, void* stream);

/* mlp_backward (mlp.py:125-154) without the grid scatter: accumulates dW, db
 * into grad (congruent to theta, caller-zeroed) and writes dX (n, in_dim). */
int nirc_mlp_backward(const nirc_spec_t* spec, const float* theta,
                      const float* X, const float* zs, const float* dY,
                      int64_t n, float* grad, float* dX, float* scratch,
                      void* stream);

/* full_forward (mlp.py:216-224) = encode_batch + mlp_forward fused in one
 * persistent sm_100a kernel: hash-grid + SH + aux encoding written straight
 * into the A operand, every layer a tcgen05.mma with the fp32 accumulator in
 * TMEM.  precision: 0 = tcgen05 3xTF32, 1 = fp32 SIMT twin, 2 = tcgen05
 * 2xFP16 split (3 products).  The 2xFP16 path guards the fp16 range: 32-row
 * units holding an input, weight or activation >= 65000 (or NaN) are
 * recomputed by the fp32 twin in a fix-up launch (stream-ordered, no sync).
 * status_flags (nullable): |= NIRC_FLAG_DIVERGED if theta holds a non-finite
 * value (the reference raises DivergenceError, mlp.py:104-105). */
int nirc_full_forward(const nirc_spec_t* spec, const float* theta,
                      const double* pos, const double* normal,
                      const double* albedo, const double* rough,
                      const double* dirs, int64_t n, float* Y,
                      int32_t precision, int32_t* status_flags, void* stream);

/* Cache._query / nirc_query (pkg/src/nirclab/caches.py:211-233), amortised
 * as the reference does it: n_dirs directions, direction i against surface
 * dir_to_surf[i]; each surface's hash block is encoded once, then every
 * direction row adds its SH block and runs the fused tcgen05 network.
 * surf rows (n_surf, 10) = pos.xyz, ns.xyz, albedo.rgb, roughness (device
 * f64); dirs (n_dirs, 3) f64; Y (n_dirs, dout) f32; precision 2 = tcgen05
 * 2xFP16 (range-guarded as nirc_full_forward), otherwise the fp32 twin.
 * Fully asynchronous: an index outside [0, n_surf) sets
 * NIRC_FLAG_BAD_INDEX in status_flags (required) and NaN in its row; a
 * non-finite theta sets NIRC_FLAG_DIVERGED. */
int nirc_query(const nirc_spec_t* spec, const float* theta, const double* surf,
               int64_t n_surf, const double* dirs, const int32_t* dir_to_surf,
               int64_t n_dirs, float* Y, int32_t precision, int32_t* status_flags,
               void* stream);

/* ---- the reference's 64-bit shadow mode -------------------
 * init_theta(dtype=float64) networks: the same entries on f64 theta / rows
 * (fp64 SIMT; every reduction over rows in a fixed order).  encode: X f64
 * (features sum w * theta in f64, SH and aux unrounded), entries/weights as
 * nirc_encode (encoding.py:111-157); forward/backward as mlp.py:102-154
 * (zs, scratch: (n, sum(dims[1:])) f64; grad accumulates); scatter as
 * nirc_scatter_grid_grad (np.add.at order); loss: every operation f64,
 * frozen_denom (n,3, nullable) = loss_relative_l2's frozen denominator
 * (losses.py:33-42); adam: f64 m / v (adam.py:20-33), skip + skipped++ on a
 * non-finite gradient.  scratch: >= 4 bytes of device memory. */
int nirc_encode_f64(const nirc_spec_t* spec, const double* theta,
                    const double* pos, const double* normal,
                    const double* albedo, const double* rough,
                    const double* dirs, int64_t n, double* X, int64_t* entries,
                    float* weights, void* stream);
int nirc_mlp_forward_f64(const nirc_spec_t* spec, const double* theta,
                         const double* X, int64_t n, double* Y, double* zs,
                         int32_t* nonfinite_flag, void* stream);
int nirc_mlp_backward_f64(const nirc_spec_t* spec, const double* theta,
                          const double* X, const double* zs, const double* dY,
                          int64_t n, double* grad, double* dX, double* scratch,
                          void* stream);
int nirc_scatter_grid_grad_f64(const nirc_spec_t* spec, double* grad,
                               const int64_t* entries, const float* weights,
                               const double* dX, int64_t n, int64_t dx_stride,
                               void* stream);
int nirc_loss_f64(int32_t kind, const double* Y, const double* target,
                  const double* pdf, const double* running_mean,
                  const double* frozen_denom, double eps, int64_t n, double* dY,
                  double* loss_out, int32_t* status_flags, void* stream);
int nirc_adam_step_f64(double* theta, double* m, double* v, const double* grad,
                       int64_t n, int64_t* t, int64_t* skipped, double lr,
                       double beta1, double beta2, double eps, int32_t* scratch,
                       void* stream);

/* ---- losses (pkg/src/nirclab/losses.py) --------------------------------- */
/* kind: 0 l2, 1 relative_l2, 2 variance, 3 bce.  Y (n,3) f32, target (n,3)
 * f64, pdf (n,) f64 (unused for bce), running_mean (3,) f64 (variance).
 * dY (n,3) f32 = the reference gradient cast to f32; loss_out (1,) f64 = the
 * mean.  status_flags[0] |= 1 on pdf <= 0 (InvalidSampleError),
 * |= 2 on a non-finite loss (DivergenceError). */
int nirc_loss(int32_t kind, const float* Y, const double* target,
              const double* pdf, const double* running_mean, double eps,
              int64_t n, float* dY, double* loss_out, int32_t* status_flags,
              double* scratch, void* stream);

/* ---- optimizer (pkg/src/nirclab/adam.py:20-33) -------------------------- */
/* Dense Adam over theta_len params.  t (i64) and skipped (i64) live on the
 * device; a non-finite grad skips the step without touching t.  When
 * gate_flags is non-NULL and *gate_flags != 0 the call is a no-op (a prior
 * divergence). */
int nirc_adam_step(float* theta, float* m, float* v, const float* grad,
                   int64_t n, int64_t* t, int64_t* skipped, double lr,
                   double beta1, double beta2, double eps,
                   const int32_t* gate_flags, int32_t* scratch, void* stream);

/* ---- online training (pkg/src/nirclab/caches.py:310-354) ---------------- */
/* One optimizer step of train_frame on device-resident records (SoA f64):
 * batch selection from the splitmix64 shuffle stream
 * (uniform_array(seed, P_SHUFFLE, frame, n, offset=step*n) + stable argsort,
 * caches.py:327-329), encode, forward, loss, backward + hash-grid scatter,
 * dense Adam.  Records: pos, ns, alb (n,3), rough (n,), dirs (n,3),
 * target (n,3), pdf (n,).  loss_out receives the step's loss (f64).
 * status_flags as in nirc_loss; once a divergence flag is set, later steps are
 * no-ops (state equals the reference at the raise). */
typedef struct nirc_records {
  const double *pos, *ns, *alb, *rough, *dirs, *target, *pdf;
  int64_t n;
} nirc_records_t;

/* Optimizer / reproducibility options of the training entries (NULL = the
 * reference defaults: beta1 0.9, beta2 0.99, eps 1e-8 from AdamState,
 * adam.py:8-17; atomic grid scatter).  deterministic != 0: the hash-grid
 * gradient is summed by the ordered scatter (nirc_scatter_grid_grad's
 * np.add.at order) instead of atomics, so repeated runs give bit-identical
 * theta (the reference's test_training_is_bit_reproducible contract). */
typedef struct nirc_train_opts {
  double beta1, beta2, eps;
  int32_t deterministic;
  int32_t reserved;
} nirc_train_opts_t;

int nirc_train_step(const nirc_spec_t* spec, float* theta, float* m, float* v,
                    int64_t* t, int64_t* skipped, const nirc_records_t* rec,
                    uint64_t seed, int64_t frame, int32_t step,
                    int32_t batch_cap, int32_t loss_kind, double loss_eps,
                    double lr, const nirc_train_opts_t* opts,
                    double* running_mean, double* loss_out,
                    int32_t* status_flags, int64_t* batch_idx_out,
                    void* workspace, int64_t workspace_bytes, void* stream);
int64_t nirc_train_workspace_bytes(const nirc_spec_t* spec, int64_t n_records,
                                   int32_t batch_cap);

/* The whole train_frame body (caches.py:310-354 without the frame counter):
 * `steps` optimizer steps on the same records, the batches of all steps
 * selected up front (they do not depend on theta), then per step the fused
 * encode/forward/loss/backward/scatter and dense Adam.  loss_out receives
 * `steps` f64 losses; status_flags as in nirc_train_step (a divergence stops
 * the remaining steps). */
int nirc_train_frame(const nirc_spec_t* spec, float* theta, float* m, float* v,
                     int64_t* t, int64_t* skipped, const nirc_records_t* rec,
                     uint64_t seed, int64_t frame, int32_t steps,
                     int32_t batch_cap, int32_t loss_kind, double loss_eps,
                     double lr, const nirc_train_opts_t* opts,
                     double* running_mean, double* loss_out,
                     int32_t* status_flags, void* workspace,
                     int64_t workspace_bytes, void* stream);
int64_t nirc_train_frame_workspace_bytes(const nirc_spec_t* spec,
                                         int64_t n_records, int32_t batch_cap,
                                         int32_t steps);

/* Multi-GPU split of nirc_train_step (the reference step is
 * caches.py:327-350).  Every rank holds the same records and selects the
 * same batch; rank r runs the fused encode/forward/loss/backward over the
 * 128-row batch tiles [tile_begin, tile_end) of nirc_train_tiles() and writes
 *   grad (theta_len f32, overwritten): its shard's gradient, the loss still
 *        normalised by the GLOBAL batch (losses.py:33-42 divides by B*3);
 *   aux (2 f64): [0] its shard's raw loss sum, [1] 1.0 if a row had pdf <= 0.
 * The caller sums grad and aux over the ranks (ncclAllReduce) and then runs
 * nirc_train_apply, identical on every rank, so replicas stay bit-identical.
 * l2 / relative_l2 losses only (NIRC_E_UNSUPPORTED otherwise). */
int64_t nirc_train_tiles(int64_t n_records, int32_t batch_cap);
int nirc_train_grad(const nirc_spec_t* spec, const float* theta,
                    const nirc_records_t* rec, uint64_t seed, int64_t frame,
                    int32_t step, int32_t batch_cap, int32_t loss_kind,
                    double loss_eps, const nirc_train_opts_t* opts,
                    int64_t tile_begin, int64_t tile_end,
                    float* grad, double* aux, int32_t* status_flags,
                    int64_t* batch_idx_out, void* workspace,
                    int64_t workspace_bytes, void* stream);
/* loss_out = aux[0] / (batch*3) (status bit 2 if non-finite), status bit 1
 * if aux[1] > 0, then the dense Adam step of nirc_adam_step gated by the
 * status flags.  scratch: >= 4 bytes of device memory. */
int nirc_train_apply(const nirc_spec_t* spec, float* theta, float* m, float* v,
                     int64_t* t, int64_t* skipped, const float* grad,
                     const double* aux, int64_t batch, double lr,
                     const nirc_train_opts_t* opts, double* loss_out,
                     int32_t* status_flags, int32_t* scratch, void* stream);

/* ---- rendering (pkg/src/nirclab/kernels.py:451-759) --------------------- */
/* render_kernel for MODE_PT / MODE_TL: per-pixel sums img, img2 (h,w,3) f64
 * and term (h,w) f64 are ACCUMULATED (caller zeroes).  The two-level cache
 * integral + residual is evaluated by the deferred NIRC inference pipeline
 * (trace -> fused encode/tcgen05 MLP/combine -> accumulate).
 * queries_out (i64, may be NULL) receives the executed-query count. */
int nirc_render(const nirc_scene_t* scene, const double* cam,
                const nirc_render_cfg_t* cfg, const nirc_spec_t* spec,
                const float* theta, double* img, double* img2, double* term,
                int64_t* queries_out, void* workspace, int64_t workspace_bytes,
                void* stream);
int64_t nirc_render_workspace_bytes(const nirc_render_cfg_t* cfg);


/* ---- training records (pkg/src/nirclab/kernels.py:85-311,
 *      caches.py:87-131) ------------------------------------------------- */
/* collect_training_records, kind "nirc" (0) or "nirc_full" (1): traces
 * `count` recording paths and writes the records in the reference's row
 * order (path-major, vertex-minor).  out_* hold `cap` rows; n_out (i64,
 * device) receives the record count. */
typedef struct nirc_records_out {
  double *pos, *ns, *alb, *rough, *dirs, *target, *pdf;
  int64_t cap;
} nirc_records_out_t;

int nirc_collect(const nirc_scene_t* scene, const double* cam, uint64_t seed,
                 uint64_t frame, int64_t count, int32_t kind,
                 const nirc_records_out_t* out, int64_t* n_out,
                 void* workspace, int64_t workspace_bytes, void* stream);
int64_t nirc_collect_workspace_bytes(int64_t count);

/* Paths [path0, path0 + count) of collect_training_records (one GPU's shard
 * in the multi-GPU frame): path p keys stream_key(seed, P_TRAIN, frame, p, 0)
 * (kernels.py:298), so the rank-ordered concatenation of the shards' records
 * equals nirc_collect over all paths row for row. */
int nirc_collect_range(const nirc_scene_t* scene, const double* cam,
                       uint64_t seed, uint64_t frame, int64_t path0,
                       int64_t count, int32_t kind,
                       const nirc_records_out_t* out, int64_t* n_out,
                       void* workspace, int64_t workspace_bytes, void* stream);

/* ---- per-interaction helpers of the API --------------------------------- */
/* estimators.py _surface_dirs (used by estimate_Lc / estimate_Lr,
 * estimators.py:260-320): n bsdf_sample draws at one interaction (shading
 * normal ns, outgoing wo, material mat; both 3-vectors on the HOST) from the
 * device uniforms u (2n); delta, pdf <= 0 and below-horizon draws give zero
 * rows.  dirs, f (n,3), pdf, cos (n,) device f64. */
int nirc_surface_samples(const nirc_scene_t* scene, const double* ns_host,
                         const double* wo_host, int32_t mat, const double* u,
                         int32_t n, double* dirs, double* pdf, double* f,
                         double* cosv, void* stream);

/* sample_incident_targets / incident_targets_kernel (caches.py:134-155,
 * kernels.py:315-338): `count` independent walk_record estimates of the
 * incident radiance along one fixed ray (walk i keyed stream_key(seed,
 * P_TRAIN, frame, i, 0)); out / out_full (count,3) device f64 = MIS-weighted /
 * raw emission at the first hit.  origin, dir, prev_ns on the HOST. */
int nirc_incident_targets(const nirc_scene_t* scene, uint64_t seed, uint64_t frame,
                          const double* origin_host, const double* dir_host,
                          double prev_pdf, const double* prev_ns_host,
                          int32_t count, double* out, double* out_full,
                          void* stream);

/* integrand_samples_kernel (kernels.py:342-421), the control-variate
 * baselines' sampler (baselines.py:426-431): per pixel of the camera
 * (width x height from cam[14..15], device f64), the centre ray's primary hit
 * and per_round BSDF draws keyed stream_key(seed, P_BASELINE, frame, p, k),
 * each with one incident-radiance walk.  Output shapes (device):
 * o_dir / o_f / o_frc (P, K, 3) f64, o_pdf (P, K) f64, o_valid (P,) u8,
 * o_spos / o_sns / o_salb (P, 3) f64, o_srough (P,) f64.  Entries the
 * reference leaves untouched (missed / mirror pixels, dead draws' dir / f /
 * frc) are not written. */
int nirc_integrand_samples(const nirc_scene_t* scene, const double* cam, uint64_t seed,
                           uint64_t frame, int32_t per_round, double* o_dir, double* o_f,
                           double* o_frc, double* o_pdf, uint8_t* o_valid, double* o_spos,
                           double* o_sns, double* o_salb, double* o_srough, void* stream);

/* occluded (geometry.py:206-210) for n shadow rays: out[i] = 1 when any
 * primitive is hit with t in (eps, t_max).  origins / dirs (n, 3) device
 * f64, out (n,) device u8.  Used by estimate_env_direct's residual
 * (estimators.py:323-370). */
int nirc_occluded(const nirc_scene_t* scene, const double* origins, const double* dirs,
                  int64_t n, double t_max, uint8_t* out, void* stream);

/* pt_radiance (estimators.py:240-257): sample `sample` of pixel (ix, iy),
 * MODE_PT, seed / frame / width / height from cfg; out (3,) device f64. */
int nirc_pt_radiance(const nirc_scene_t* scene, const double* cam,
                     const nirc_render_cfg_t* cfg, int32_t ix, int32_t iy,
                     int32_t sample, double* out, void* stream);

/* ---- one frame: render + collect ---------------------------------------- */
/* One frame's render (nirc_render) AND training-record collection
 * (nirc_collect_range over paths [path0, path0+count) with seed train_seed,
 * frame train_frame) in one persistent trace launch: the training walks are
 * the first work items of the path tracer, so their long roulette tails
 * overlap the camera paths (render_kernel + collect_paths_kernel,
 * kernels.py:289-311,723-759, in the order experiment.py:153-172 calls
 * them; both read only the scene, neither reads theta's updates). */
int nirc_render_collect(const nirc_scene_t* scene, const double* cam,
                        const nirc_render_cfg_t* cfg, const nirc_spec_t* spec,
                        const float* theta, double* img, double* img2,
                        double* term, int64_t* queries_out, uint64_t train_seed,
                        uint64_t train_frame, int64_t path0, int64_t count,
                        int32_t kind, const nirc_records_out_t* out,
                        int64_t* n_out, void* workspace, int64_t workspace_bytes,
                        void* stream);
int64_t nirc_render_collect_workspace_bytes(const nirc_render_cfg_t* cfg,
                                            int64_t count);

/* ---- scene acceleration (pkg/src/nirclab/geometry.py:213-274) ----------- */
/* build_bvh on the device: the reference's median-split BVH (<= 4 prims per
 * leaf, left child = next node, right child index in a, leaf iff b > 0 with
 * prims prim[a : a+b]), node for node identical to the host build.  Inputs
 * (device f64): tri_v0 / tri_e1 / tri_e2 (n_tri, 3), sph_c (n_sph, 3),
 * sph_r (n_sph,).  Outputs (device): lo / hi (N, 3) f64, a / b (N,) i32,
 * prim (n_tri + n_sph,) i32, N = nirc_bvh_node_count(n_tri + n_sph).
 * Synchronises `stream` before returning. */
int64_t nirc_bvh_node_count(int64_t n_prims);

/* Traversal image of a scene's BVH (kernels-private layout: per internal
 * node both child boxes and child references; primitives in BVH leaf order
 * with their geometry inline).  `out` is a device buffer of
 * nirc_scene_packed_bytes(scene) bytes; on success scene->bvh_packed and
 * scene->prim_packed point into it.  Hit results are the bvh_* traversal's
 * (same nearest hit, same any-hit boolean). */
int64_t nirc_scene_packed_bytes(const nirc_scene_t* scene);
int nirc_pack_scene(nirc_scene_t* scene, void* out, int64_t out_bytes, void* stream);
int nirc_build_bvh(const double* tri_v0, const double* tri_e1, const double* tri_e2,
                   int64_t n_tri, const double* sph_c, const double* sph_r, int64_t n_sph,
                   double* lo, double* hi, int32_t* a, int32_t* b, int32_t* prim,
                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* NIRC_B200_H */
