/* sgm.h — C ABI of the B200-native candidate-view render + scoring path.
 *
 * This is the drop-in boundary for the reference's renderer/scoring API. The
 * reference has no FFI: its boundary is the C++ header API in
 * proj/include/splatmap/splat_render.hpp:78-95 and
 * proj/include/splatmap/explorer.hpp:114-131. Every entry point
 * below names the reference interface it replaces. Plain pointers and sizes only;
 * no CUDA or torch types appear in the signatures (streams are passed as void*).
 *
 * Conventions
 *   - Every call returns an int status (SGM_OK == 0). On failure the message is
 *     available from sgm_last_error(ctx); the C++/Python wrappers rethrow it as
 *     std::runtime_error / RuntimeError, mirroring the reference's exception style.
 *   - One sgm_ctx per GPU. Calls on one ctx are serialised by the caller; distinct
 *     ctxs may be driven concurrently from different host threads (the reference's
 *     "pure given inputs" threading contract).
 *   - Host buffers are caller-owned. All floating-point inputs/outputs are fp64,
 *     in the reference's storage layouts (gaussian_map.hpp:105-113,
 *     splat_render.hpp:51-54).
 *   - There is no CPU fallback: a ctx cannot be created without a CUDA device.
 */
#ifndef SGM_H
#define SGM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGM_ABI_VERSION 1

typedef struct sgm_ctx sgm_ctx; /* per-GPU context: stream, scratch, last-call state */
typedef struct sgm_map sgm_map; /* device-resident, immutable GaussianMap snapshot */

/* CameraModel (proj/include/splatmap/camera.hpp:11-50); FOV fields are unused by render. */
typedef struct {
    int32_t width, height;
    double fx, fy, cx, cy;
} sgm_camera;

/* Pose (proj/include/splatmap/geometry.hpp:18-41): x_world = R x_cam + t. R row-major. */
typedef struct {
    double R[9];
    double t[3];
} sgm_pose;

/* RenderOptions (proj/include/splatmap/splat_render.hpp:22-28). */
typedef struct {
    int32_t early_exit;        /* default 1 */
    double transmittance_eps;  /* default 1e-4 */
    double z_near;             /* default 0.01 */
    double truncation_sigmas;  /* default 3.0 */
    int32_t tile_size;         /* default 8 (bins are built at this size, bit-exact) */
} sgm_options;

/* SplatProjection (splat_render.hpp:32-39). */
typedef struct {
    double mx, my, rad_px, z, alpha;
    uint32_t index;
    uint32_t reserved;
} sgm_projection;

/* CandidatePose geometry (explorer.hpp:93-106); camera_pose() = look_at(p, p + d). */
typedef struct {
    double position[3];
    double direction[3];
} sgm_candidate;

/* RenderChannels (splat_render.hpp:12-20) as bit flags. */
enum {
    SGM_COLOR = 1u,
    SGM_DEPTH = 2u,
    SGM_SEMANTICS = 4u,
    SGM_RETAIN_CONTRIBUTORS = 8u
};

enum {
    SGM_OK = 0,
    SGM_ERR_INVALID = 1,     /* bad argument (reference would throw std::invalid_argument) */
    SGM_ERR_CUDA = 2,        /* CUDA runtime / launch failure */
    SGM_ERR_OOM = 3,         /* device allocation failed */
    SGM_ERR_UNSUPPORTED = 4  /* valid request this build does not serve */
};

/* Per-ctx counters since creation or the last sgm_ctx_reset_stats. */
typedef struct {
    uint64_t kernel_launches;   /* kernels of this library launched */
    uint64_t views;             /* views processed (render + score) */
    uint64_t visible;           /* sum of V (culled-in projections) */
    uint64_t pairs;             /* sum of P ((tile, projection) pairs) */
    uint64_t contributors;      /* sum of K (composited pixel-splat pairs) */
    uint64_t raster_launches;   /* raster kernel launches (timed when profiling is on) */
    double raster_ms;           /* CUDA-event time of raster launches (profiling on) */
    double binning_ms;          /* CUDA-event time of preprocess+binning (profiling on) */
} sgm_stats;

int sgm_abi_version(void);

/* ---- context ---- */
int sgm_ctx_create(int device, sgm_ctx** out);
void sgm_ctx_destroy(sgm_ctx* ctx);
/* Last error of `ctx`; with ctx == NULL, the last error of sgm_ctx_create on this thread. */
const char* sgm_last_error(const sgm_ctx* ctx);
/* The cudaStream_t (as void*) every kernel of this ctx is launched on. */
void* sgm_ctx_stream(sgm_ctx* ctx);
int sgm_ctx_synchronize(sgm_ctx* ctx);
int sgm_ctx_set_profiling(sgm_ctx* ctx, int enabled);
int sgm_ctx_get_stats(const sgm_ctx* ctx, sgm_stats* out);
int sgm_ctx_reset_stats(sgm_ctx* ctx);

/* ---- map ----
 * Replaces passing `const GaussianMap&` (gaussian_map.hpp:61-114) to each render:
 * uploads a read-only snapshot once per map version. Arrays are the GaussianMap
 * spans: centers 3N, log_radii N, opacity_logits N, colors 3N, sem_indices kN,
 * sem_probs kN. Errors as GaussianMap(k, num_classes) (gaussian_map.hpp:63-66) plus
 * sem index < num_classes + 1. Activations exp/sigmoid and the colour clamp are
 * applied on the host with the reference's libm (gaussian_map.hpp:36-37). */
int sgm_map_upload(sgm_ctx* ctx, uint64_t n, int32_t k, int32_t num_classes,
                   const double* centers, const double* log_radii,
                   const double* opacity_logits, const double* colors,
                   const uint16_t* sem_indices, const double* sem_probs, sgm_map** out);
/* The same, returning once the geometry is on its way: the colours and semantic rows are
 * staged by a background thread and copied / class-sorted on the ctx's upload stream while
 * the caller already queues work (preprocess and binning need only the geometry; the raster
 * waits for the rows). The caller keeps the host arrays alive and unchanged until the first
 * compute call on the map returns, or sgm_map_wait / sgm_map_release (sgm_map_upload is
 * sgm_map_upload_async + sgm_map_wait). A semantic index >= num_classes + 1 is reported by
 * sgm_map_wait or the first compute call on the map (sgm_map_upload reports it itself). */
int sgm_map_upload_async(sgm_ctx* ctx, uint64_t n, int32_t k, int32_t num_classes,
                         const double* centers, const double* log_radii,
                         const double* opacity_logits, const double* colors,
                         const uint16_t* sem_indices, const double* sem_probs, sgm_map** out);
/* Waits until every copy of an uploaded map is on the device. */
int sgm_map_wait(sgm_ctx* ctx, sgm_map* map);
void sgm_map_release(sgm_ctx* ctx, sgm_map* map);

/* ---- anisotropic splat mode (NO reference counterpart, parity unpinned) ----
 * Switches an uploaded map to per-Gaussian anisotropic footprints: log_scales 3N (per-axis
 * log sigma), quats 4N ((w, x, y, z), normalised here). World covariance
 * Sigma = R(q) diag(exp(ls))^2 R(q)^T; projection by EWA, Sigma2D = J R_cw Sigma R_cw^T J^T
 * (J: pinhole Jacobian at the camera-space centre, its direction clamped to 1.3x the
 * half field of view as in 3D Gaussian splatting); footprint alpha exp(-q / 2) with
 * q = d^T Sigma2D^-1 d, cut at q > truncation_sigmas^2; tiles from the truncated
 * axis-aligned extent. log_radii are then unused. Both NULL restores the isotropic
 * (reference) footprint. render / score / render_entropy / eval accept such maps;
 * the Fisher and backward entry points return SGM_ERR_UNSUPPORTED for them. */
int sgm_map_set_anisotropic(sgm_ctx* ctx, sgm_map* map, const double* log_scales,
                            const double* quats);

/* ---- device snapshot interchange (SURVEY §8e collective C1: the map broadcast) ----
 * A map's device snapshot (activated geometry, clamped colours, class-sorted rows, the
 * anisotropic covariance) packed into one blob in DEVICE memory, so a map is broadcast
 * device to device (e.g. ncclBroadcast over NVLink, or a peer copy) instead of re-running
 * the host activations on every rank. sgm_map_export writes into `d_blob` (capacity >=
 * sgm_map_export_bytes) on the ctx's device; sgm_map_import builds a map on ctx's device
 * from a blob in any device memory it can read (peer or own). The imported map is
 * bit-identical to the exported one (the Fisher prior is not part of the snapshot). */
/* n, k, num_classes and whether the anisotropic mode is on, of an uploaded or imported map.
 * Any output may be NULL. */
int sgm_map_info(sgm_ctx* ctx, const sgm_map* map, uint64_t* n, int32_t* k, int32_t* num_classes,
                 int32_t* anisotropic);
int sgm_map_export_bytes(sgm_ctx* ctx, const sgm_map* map, uint64_t* bytes);
int sgm_map_export(sgm_ctx* ctx, const sgm_map* map, void* d_blob, uint64_t capacity);
int sgm_map_import(sgm_ctx* ctx, const void* d_blob, uint64_t bytes, sgm_map** out);

/* ---- multi-GPU scoring in one process (refresh_candidate_scores,
 * explorer.cpp:186-205, whose candidate loop "parallelizes over candidates") ----
 * One sgm_ctx per device (devices NULL: 0 .. n_devices-1; n_devices <= 0: every visible
 * device). sgm_multi_map_upload runs the host activations and H2D once (first device) and
 * replicates the snapshot device to device (peer copies over NVLink). Scoring shards the n
 * views contiguously (sizes differ by <= 1) over the devices, one host thread each, and
 * writes every view's result to its own slot: per-view results are bit-identical to
 * sgm_score_views on one device. Errors: status + sgm_multi_last_error; a failing
 * sgm_multi_create reports through sgm_last_error(NULL). */
typedef struct sgm_multi sgm_multi;
typedef struct sgm_multi_map sgm_multi_map;
int sgm_multi_create(int32_t n_devices, const int32_t* devices, sgm_multi** out);
void sgm_multi_destroy(sgm_multi* mg);
const char* sgm_multi_last_error(const sgm_multi* mg);
int32_t sgm_multi_device_count(const sgm_multi* mg);
/* The i-th device's ctx (owned by mg), for single-device calls (render, ...). */
sgm_ctx* sgm_multi_ctx(sgm_multi* mg, int32_t i);
int sgm_multi_map_upload(sgm_multi* mg, uint64_t n, int32_t k, int32_t num_classes,
                         const double* centers, const double* log_radii,
                         const double* opacity_logits, const double* colors,
                         const uint16_t* sem_indices, const double* sem_probs,
                         sgm_multi_map** out);
void sgm_multi_map_release(sgm_multi* mg, sgm_multi_map* map);
int sgm_multi_score_views(sgm_multi* mg, const sgm_multi_map* map, const sgm_camera* cam,
                          uint64_t n, const sgm_pose* poses, const sgm_options* opt,
                          double* n_missing, double* entropy_sum);
int sgm_multi_score_candidates(sgm_multi* mg, const sgm_multi_map* map, const sgm_camera* cam,
                               uint64_t n, const sgm_candidate* cands, const sgm_options* opt,
                               double* n_missing, double* entropy_sum);

/* ---- render (splat_render.hpp:78-80, render()) ----
 * Host output planes in the reference layout; NULL for channels not requested.
 * silhouette (px) is always written. color px*3, depth px, sem px*(num_classes+1).
 * *n_projections receives V. */
int sgm_render(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam, const sgm_pose* pose,
               uint32_t channels, const sgm_options* opt, double* color, double* depth,
               double* silhouette, double* sem, uint64_t* n_projections);
/* Same, but planes are written to caller-provided DEVICE buffers on the ctx stream. */
int sgm_render_device(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam,
                      const sgm_pose* pose, uint32_t channels, const sgm_options* opt,
                      double* d_color, double* d_depth, double* d_silhouette, double* d_sem,
                      uint64_t* n_projections);
/* ---- render_reference (splat_render.hpp:82-86, splat_render.cpp:330-358) ----
 * The reference's plain per-pixel compositor: default RenderOptions with early_exit = false,
 * and composite_pixel's footprint form f = min(alpha exp(-d2 / (2 r^2)), kMaxFootprint)
 * with f <= 0 skipped (:86-92; no contributor entry, T unchanged). Outputs as sgm_render;
 * contributor lists (SGM_RETAIN_CONTRIBUTORS) then exclude alpha == 0 splats, as the
 * reference's do. */
int sgm_render_reference(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam,
                         const sgm_pose* pose, uint32_t channels, double* color, double* depth,
                         double* silhouette, double* sem, uint64_t* n_projections);
/* RenderOutput.projections of the last sgm_render* call (depth-sorted, culled). */
int sgm_last_projections(sgm_ctx* ctx, sgm_projection* out, uint64_t capacity);
/* The tile bins of the last sgm_render* call at RenderOptions::tile_size
 * (splat_render.cpp:188-213, local to render() in the reference): tile_offsets has
 * tiles+1 entries, ids are projection ids in bin order, probe3 the float Probe
 * fields (mx, my, cutoff_d2). Any pointer may be NULL; *n_pairs receives P. */
int sgm_last_bins(sgm_ctx* ctx, uint32_t* tile_offsets, uint32_t* ids, float* probe3,
                  uint64_t capacity, uint64_t* n_pairs);
/* RenderOutput.contrib / contrib_offset of the last render with
 * SGM_RETAIN_CONTRIBUTORS (splat_render.cpp:125-137). offsets has px+1 entries. */
int sgm_last_contributors(sgm_ctx* ctx, uint32_t* offsets, uint32_t* contrib,
                          uint64_t capacity, uint64_t* n_contrib);

/* ---- entropy (splat_render.hpp:86-91) ---- */
double sgm_clipped_entropy(const double* probs, uint64_t n);
int sgm_render_entropy(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam,
                       const sgm_pose* pose, const sgm_options* opt, double* entropy);

/* ---- candidate scoring (explorer.hpp:114-121) ----
 * refresh_candidate_scores for n views given as poses: per view the exact-zero
 * silhouette count (n_missing) and the summed clipped entropy. Batched on the
 * GPU; per-view results are deterministic and independent of batching/sharding. */
int sgm_score_views(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam, uint64_t n,
                    const sgm_pose* poses, const sgm_options* opt, double* n_missing,
                    double* entropy_sum);
/* Same for CandidatePose geometry (camera_pose() computed on the host). */
int sgm_score_candidates(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam, uint64_t n,
                         const sgm_candidate* cands, const sgm_options* opt,
                         double* n_missing, double* entropy_sum);
/* ---- Fisher-information gain (extension; no reference counterpart) ----
 * Diagonal Fisher information of the rendered colour and depth with respect to each
 * Gaussian's theta = (mu_x, mu_y, mu_z, log_radius, opacity_logit, c_r, c_g, c_b): the
 * per-pixel Jacobian of the analytic chain in proj/src/losses.cpp:242-335, chained to world
 * space per pixel and squared, summed over pixels and the R, G, B, depth channels.
 * sgm_fisher_prior: H_prior = sum over the n past poses (kept with the map); optional host
 * copy H_out [N][8]. sgm_score_views_fisher: per view n_missing, entropy_sum and the
 * FisherRF-style gain  sum_{i,theta} H_view / (H_prior + lambda)  (deterministic). */
int sgm_fisher_prior(sgm_ctx* ctx, sgm_map* map, const sgm_camera* cam, uint64_t n,
                     const sgm_pose* poses, const sgm_options* opt, double lambda, double* H_out);
/* Sets the map's Fisher prior from a host H (N x 8, the layout sgm_fisher_prior returns), e.g.
 * the sum of per-rank sgm_fisher_prior results over sharded past poses (SURVEY §8e collective
 * C2: all-reduce of H_prior), then 1 / (H + lambda) on the device as sgm_fisher_prior does. */
int sgm_fisher_set_prior(sgm_ctx* ctx, sgm_map* map, const double* H, double lambda);
int sgm_score_views_fisher(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam, uint64_t n,
                           const sgm_pose* poses, const sgm_options* opt, double* n_missing,
                           double* entropy_sum, double* fisher_gain);

/* ---- mapping step: losses + analytic backward ----
 * Renders the map at `pose` (render(..., RenderChannels::all(true)), splat_render.cpp:170),
 * then mapping_loss + semantic_loss (losses.cpp:40-160) against the frame planes (rgb px*3,
 * depth px, sem px*(num_classes+1), float, Frame layout, frame.hpp:12-65) and backward
 * (losses.cpp:162-362). weights = {lambda_hd, lambda_cos, mask_k, use_hd, use_cos, use_kl,
 * kl_clip_norm} (LossWeights, losses.hpp:9-17); report = {photometric, depth, semantic,
 * photometric_px, depth_px, semantic_px, uncovered_px} (LossReport). Gradient arrays are the
 * ParamGradients spans (center 3N, log_radius N, opacity_logit N, color 3N, sem kN) and may
 * be NULL. A non-finite gradient fails like the reference's throw. */
int sgm_backward(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam, const sgm_pose* pose,
                 const sgm_options* opt, const float* rgb, const float* depth, const float* sem,
                 const double weights[7], int include_mapping, int include_semantic,
                 double report[7], double* g_center, double* g_log_radius,
                 double* g_opacity_logit, double* g_color, double* g_sem);

/* ---- on-device map optimisation: optimize_map (mapper.cpp:241-283) ----
 * A frame uploaded once (Frame, frame.hpp:12-65: rgb px*3, depth px, sem px*(C) floats, with
 * its pose) and a trainer holding the map parameters plus the Adam moments in HBM. */
typedef struct sgm_frame sgm_frame;
typedef struct sgm_trainer sgm_trainer;

/* AdamParams, optimizer.hpp:8-21. */
typedef struct {
    double lr_center, lr_radius, lr_opacity, lr_color, lr_sem;
    double beta1, beta2, eps, eps_sem;
} sgm_adam_params;

/* The MapperConfig fields optimize_map reads (mapper.hpp:18-33). */
typedef struct {
    int32_t prune_every;
    double prune_opacity;
    double divergence_factor;
    int32_t divergence_window;
} sgm_optimize_config;

int sgm_frame_upload(sgm_ctx* ctx, int32_t width, int32_t height, int32_t num_classes,
                     const sgm_pose* pose, const float* rgb, const float* depth, const float* sem,
                     sgm_frame** out);
void sgm_frame_release(sgm_ctx* ctx, sgm_frame* frame);

/* GaussianMap spans as in sgm_map_upload, plus the AdamState (mapper.hpp / optimizer.hpp:24-60):
 * adam_mv = {m, v} each laid out center 3N | log_radius N | opacity_logit N | color 3N |
 * sem kN (2 * (8 + k) * N doubles; NULL = zero moments) and its step count. */
int sgm_trainer_create(sgm_ctx* ctx, uint64_t n, int32_t k, int32_t num_classes,
                       const double* centers, const double* log_radii, const double* opacity_logits,
                       const double* colors, const uint16_t* sem_indices, const double* sem_probs,
                       const double* adam_mv, int64_t step_count, sgm_trainer** out);
void sgm_trainer_destroy(sgm_ctx* ctx, sgm_trainer* tr);
int sgm_trainer_size(sgm_ctx* ctx, const sgm_trainer* tr, uint64_t* n, int64_t* step_count);
/* Copies the current parameters (and, if adam_mv != NULL, the moments) back to the host. */
int sgm_trainer_download(sgm_ctx* ctx, const sgm_trainer* tr, double* centers, double* log_radii,
                         double* opacity_logits, double* colors, uint16_t* sem_indices,
                         double* sem_probs, double* adam_mv);
/* The creation-time row of each current Gaussian (prune_by_opacity's `kept`, composed over
 * every prune since sgm_trainer_create): n uint32. */
int sgm_trainer_rows(sgm_ctx* ctx, const sgm_trainer* tr, uint32_t* rows);
/* optimize_map: `iters` round-robin iterations over `frames` of render(all(true)) ->
 * mapping_loss + semantic_loss -> backward -> Adam step, with opacity pruning on the
 * prune_every cadence and the reference's divergence check. history receives one LossReport
 * (7 doubles, as sgm_backward) per completed iteration; *n_done their count. Errors as the
 * reference: no frames / iters < 1 -> SGM_ERR_INVALID; divergence or a non-finite gradient ->
 * SGM_ERR_INVALID with the iterations done so far in history. */
int sgm_optimize_map(sgm_ctx* ctx, sgm_trainer* tr, const sgm_camera* cam, uint64_t n_frames,
                     sgm_frame* const* frames, const sgm_options* opt,
                     const sgm_adam_params* adam, const double weights[7],
                     const sgm_optimize_config* cfg, int32_t iters, double* history,
                     int32_t* n_done);

/* ---- evaluation on device render planes ----
 * semantic_metrics (evaluator.cpp:93-238) + photometric_metrics (:274-297) over views
 * added one at a time: each sgm_eval_add_view renders `map` at the frame's pose
 * (RenderChannels::all()) into HBM and consumes the planes there; only the C x C confusion
 * counts and a few sums per view leave the device. */
typedef struct sgm_evaluator sgm_evaluator;

int sgm_eval_create(sgm_ctx* ctx, int32_t num_classes, sgm_evaluator** out);
void sgm_eval_destroy(sgm_ctx* ctx, sgm_evaluator* ev);
/* Frame size must match cam and channels num_classes + 1 ("resolution mismatch"). */
int sgm_eval_add_view(sgm_ctx* ctx, sgm_evaluator* ev, const sgm_map* map, const sgm_camera* cam,
                      const sgm_options* opt, const sgm_frame* frame);
/* MetricReport (evaluator.hpp:20-42). summary = {miou_pct, top1_pct, top3_pct, map_pct,
 * f1_pct, psnr_db, depth_l1_cm}; per_view_miou / per_view_psnr: one per added view;
 * per_class: rows {class_id, iou_pct, ap_pct, f1_pct, gt_pixels} sorted by class_id
 * (at most num_classes rows), *n_per_class their count. No views -> SGM_ERR_INVALID
 * ("view count mismatch"). Any output may be NULL. */
int sgm_eval_report(sgm_ctx* ctx, sgm_evaluator* ev, double summary[7], double* per_view_miou,
                    double* per_view_psnr, double* per_class, uint64_t* n_per_class);

/* combine_scores (explorer.cpp:225-248) on host fp64: returns 1 if any i_total > 0,
 * 0 if the pool is exhausted (or n == 0), negative on invalid arguments. */
int sgm_combine_scores(uint64_t n, const double* n_missing, const double* entropy_sum,
                       const double* positions3, const double current[3], double* i_geo,
                       double* i_sem, double* i_total);
/* The Fisher extension's combined scalar gain and its ranking criterion (the
 * slot of combine_scores, explorer.cpp:225-248, followed by the sort at episode.cpp:410-414):
 *   gain_v   = fisher_gain_v + w_sem * entropy_sum_v    (FisherRF gain + semantic entropy)
 *   i_total_v = (n == 1 ? 1 : 1 - softmax(|pos_v - current|)_v) * softmax(ln gain_v)_v
 * Rank by i_total descending, id ascending. Returns 1 if any i_total > 0, 0 if none or n == 0,
 * negative on invalid arguments (null pointers, w_sem < 0 or not finite). */
int sgm_combine_scores_fisher(uint64_t n, const double* fisher_gain, const double* entropy_sum,
                              const double* positions3, const double current[3], double w_sem,
                              double* gain, double* i_total);
/* look_at(p, p + d) (geometry.hpp:44-56) with Eigen's evaluation order. */
void sgm_candidate_pose(const double position[3], const double direction[3], sgm_pose* out);
void sgm_look_at(const double position[3], const double target[3], sgm_pose* out);

/* ---- exploration map + candidate sampling ----
 * Replaces splatmap::ExplorationMap (explorer.hpp:11-83, explorer.cpp:11-139) with a
 * device-resident u8 grid (0 unknown, 1 free, 2 occupied; linear id (iz*dy + iy)*dx + ix)
 * and a device changelog. Results are bit-identical to the reference: the same voxel
 * states, counts and changelog order. */
typedef struct sgm_emap sgm_emap;

/* Aabb (geometry.hpp:58-67). */
typedef struct {
    double min[3];
    double max[3];
} sgm_aabb;

/* ExplorationMap(bounds, voxel_size) (explorer.cpp:11-20): origin = bounds.min,
 * dims = max(ceil(extent / voxel), 1). voxel_size <= 0 -> SGM_ERR_INVALID. */
int sgm_emap_create(sgm_ctx* ctx, const sgm_aabb* bounds, double voxel_size, sgm_emap** out);
void sgm_emap_destroy(sgm_ctx* ctx, sgm_emap* emap);
/* origin(), voxel_size(), dims(), free_count(), occupied_count(), changelog_size(). Any
 * output may be NULL. */
int sgm_emap_info(sgm_ctx* ctx, const sgm_emap* emap, double origin[3], double* voxel_size,
                  int32_t dims[3], uint64_t* free_count, uint64_t* occupied_count,
                  uint64_t* changelog_size);
/* integrate_frame (explorer.cpp:53-110): the Amanatides-Woo walk of every stride-th depth
 * pixel. depth is the Frame depth plane (cam->width * cam->height floats, 0 = invalid),
 * host memory for sgm_emap_integrate and device memory for the _device variant.
 * *newly_freed receives the number of voxels this frame appended to the changelog. */
int sgm_emap_integrate(sgm_ctx* ctx, sgm_emap* emap, const sgm_camera* cam,
                       const sgm_pose* pose, const float* depth, int32_t stride,
                       uint64_t* newly_freed);
int sgm_emap_integrate_device(sgm_ctx* ctx, sgm_emap* emap, const sgm_camera* cam,
                              const sgm_pose* pose, const float* d_depth, int32_t stride,
                              uint64_t* newly_freed);
/* take_changelog (explorer.cpp:112-116): copies min(size, capacity) ids to out, sets *n to
 * the size and clears the changelog. capacity < size -> SGM_ERR_INVALID, nothing cleared. */
int sgm_emap_take_changelog(sgm_ctx* ctx, sgm_emap* emap, int32_t* out, uint64_t capacity,
                            uint64_t* n);
/* reseed_changelog_with_free (explorer.cpp:118-122). */
int sgm_emap_reseed_changelog_with_free(sgm_ctx* ctx, sgm_emap* emap);
/* seed_free_region / seed_occupied_region (explorer.cpp:124-132). */
int sgm_emap_seed_region(sgm_ctx* ctx, sgm_emap* emap, const sgm_aabb* box, int occupied);
/* grid() (explorer.hpp:42): copies voxel_count bytes of state to host `out`. */
int sgm_emap_grid(sgm_ctx* ctx, const sgm_emap* emap, uint8_t* out, uint64_t capacity);
/* sample_candidates (explorer.cpp:157-184): consumes the changelog and writes one
 * (position, direction) per free, freshly logged lattice point x fibonacci direction, in
 * the reference's order. heights: n_heights values; v1 > 0 lattice spacing; v2 >= 1
 * directions (max elevation 45 deg). capacity too small -> SGM_ERR_INVALID with *n_out =
 * the count needed and the changelog left untouched. */
int sgm_sample_candidates(sgm_ctx* ctx, sgm_emap* emap, double v1, int32_t v2,
                          const double* heights, int32_t n_heights, sgm_candidate* out,
                          uint64_t capacity, uint64_t* n_out);
/* fibonacci_directions (explorer.cpp:142-155), host fp64: count x 3 doubles. */
void sgm_fibonacci_directions(int32_t count, double max_elevation_deg, double* out3);

#ifdef __cplusplus
}
#endif
#endif /* SGM_H */
