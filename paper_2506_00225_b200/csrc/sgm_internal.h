// Internal types shared by the kernels (sgm_kernels.cu) and the host pipeline
// (sgm_capi.cu). Device layout of one map snapshot and one batch of views.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/sgm.h"

namespace sgm {

constexpr double kMaxFootprint = 0.999999;  // splat_render.hpp:41
constexpr int kTile = 8;                    // raster tile edge (== reference tile_size)
constexpr int kTilePx = kTile * kTile;      // pixels (threads) per raster CTA

// Map snapshot in HBM. Geometry stays fp64 because the depth order and tile
// rectangles must be bit-identical to the reference; radius and
// opacity are activated on the host with the reference's libm.
struct DevMap {
    uint64_t n = 0;
    int k = 0;            // sparse entries per Gaussian
    int kpad = 0;         // row stride of sem_idx / sem_prob (k rounded up to 8)
    int C = 0;            // semantic channels = num_classes + 1
    const double* cx = nullptr;  // centres, SoA
    const double* cy = nullptr;
    const double* cz = nullptr;
    const double* rad = nullptr;    // exp(log_radius)
    const double* alpha = nullptr;  // sigmoid(opacity_logit)
    const double* color4 = nullptr; // clamp(colour, 0, 1), [n][4] (4th unused)
    // Sparse rows sorted by class id at upload (per-class addition order is
    // unchanged: a Gaussian lists a class once, or duplicates keep their order).
    // Rows padded to kpad with (0xffff, 0.0) so every row is 16-byte aligned.
    const uint16_t* sem_idx = nullptr;  // [n][kpad]
    const double* sem_prob = nullptr;   // [n][kpad]
    const uint16_t* sem_perm = nullptr; // [n][kpad] original entry index of each sorted slot
    int dup_idx = 0;  // some Gaussian lists a class twice: serialise its RMWs
    // Anisotropic splat mode (no reference counterpart): the world
    // covariance replaces rad; projections use the EWA footprint (sgm_kernels.cu).
    int aniso = 0;
    const double* cov = nullptr;  // [6][n] SoA: xx, xy, xz, yy, yz, zz
    // per Gaussian: the ends of its class-sorted row's 8 raster channel groups (u16 each),
    // computed once per map (launch_group_bounds); the raster stages them with the rows
    const uint4* gbounds = nullptr;
    // the class-sorted rows as 16-byte records {prob (lo, hi words), class, 0}, [n][kpad]:
    // one shared-memory load per (entry, class) in the score raster's scatter. Built from
    // sem_idx / sem_prob before a score pass (launch_sem_records; map_records)
    const uint4* sem_rec = nullptr;
};

struct CamParams {
    int W, H;
    double fx, fy, cx, cy;
};

// Camera-from-world rotation, row-major (Rcw[3i+k] = R(k,i)), and centre.
struct PoseParams {
    double Rcw[9];
    double t[3];
};

struct OptParams {
    int early_exit;
    double eps;
    double z_near;
    double trunc;   // truncation_sigmas
    double cut_sq;  // trunc * trunc (splat_render.cpp:180)
    int ts;         // reference tile_size (binning)
    int tiles_x, tiles_y;
    // render_reference's footprint form (splat_render.cpp:91-92): exp(-d2 / (2 r^2)) with the
    // division, and f <= 0 skipped (not a contributor). k_pack then stores 2 r^2 in the
    // inv_two_r2 slot. Render launches only.
    int ref_div = 0;
};

// One culled-in projection in depth-rank order: the reference's PackedSplat
// (splat_render.cpp:158-166) plus its float Probe (:184-187). 64 bytes.
struct __align__(16) PackedSplat {
    double mx, my;
    double inv_two_r2;
    double cutoff_d2;
    double alpha;
    double z;
    float pmx, pmy, pcut;
    uint32_t aux;  // depth rank (projection id) of this record
};
static_assert(sizeof(PackedSplat) == 64, "PackedSplat must stay 64 B");

// The same record in the anisotropic mode: the conic (inverse 2D covariance) takes
// the slots of inv_two_r2, cutoff_d2 and the float probe (the cut is the constant
// Mahalanobis trunc^2); alpha, z and aux keep their offsets.
struct __align__(16) PackedSplatA {
    double mx, my;
    double qa, qb;
    double alpha;
    double z;
    double qc;
    uint32_t pad;
    uint32_t aux;
};
static_assert(sizeof(PackedSplatA) == 64, "PackedSplatA must stay 64 B");
static_assert(offsetof(PackedSplatA, alpha) == offsetof(PackedSplat, alpha) &&
                  offsetof(PackedSplatA, z) == offsetof(PackedSplat, z) &&
                  offsetof(PackedSplatA, aux) == offsetof(PackedSplat, aux),
              "PackedSplatA must share alpha / z / aux with PackedSplat");

// Channel groups: the C semantic channels are split into P groups of Cg; each
// group is accumulated by its own CTA of a (P,1,1) thread-block cluster.
struct GroupParams {
    int P;
    int Cg;
};

// Fisher extension (sgm_fisher.cu)
struct FisherParams {
    double* H;           // [N][8] prior accumulation (prior mode)
    const double* invp;  // [N][8] 1 / (H_prior + lambda) (gain mode)
};

// Backward pass (sgm_backward.cu): mapping / semantic losses and their gradients.
struct BackwardParams {
    int W, H, C;
    const double* color;     // rendered planes (device, reference layout)
    const double* depth;
    const double* sil;
    const double* sem;
    const uint32_t* ccount;  // contributors per pixel
    const float* rgb;        // frame planes (device): px*3, px, px*C
    const float* fdepth;
    const float* fsem;
    uint8_t* flags;          // per pixel: bit0 photometric mask, bit1 semantic mask
    double tau;              // ln(mask_k)
    double lambda_hd, lambda_cos;
    int use_hd, use_cos, use_kl;
    int include_mapping, include_semantic;
    const double* totals;    // device [8] (k_loss_pixels)
    double* gproj;           // [V][5] projection-space (alpha, mx, my, rad, z)
    double* gcenter;         // [N][3]
    double* glogr;           // [N]
    double* glogit;          // [N]
    double* gcolor;          // [N][3]
    double* gsem;            // [N][k] (original entry order)
    const uint16_t* sem_perm;
};

// Per view of a raster batch.
struct ViewDesc {
    const uint32_t* order;      // [V] depth rank -> map index
    const PoseParams* pose;     // device pose of this view
    double* fis_partial;        // [tiles] per-tile Fisher gain (gain mode)
    const uint2* ranges;        // [tiles] (begin, end) into list
    const uint32_t* list;       // depth ranks grouped by tile, rank order inside a tile
    const PackedSplat* packed;  // [V] by rank
    const uint4* bounds;        // [V] by rank: raster channel-group bounds (8 x u16)
    double* ent_partial;        // [tiles] per-tile entropy sum (score mode)
    uint32_t* miss_partial;     // [tiles] per-tile exact-zero silhouette count
    // render mode planes (device, reference layout); null when not requested
    double* color;
    double* depth;
    double* sil;
    double* sem;
    unsigned long long* contributors;  // K counter
    // retain_contributors (render mode): pass 1 counts per pixel into contrib_count
    // (contrib_offset == null); pass 2 writes depth ranks at contrib_offset[pixel]
    uint32_t* contrib;
    uint32_t* contrib_count;
    const unsigned long long* contrib_offset;
    // score mode with the Fisher gain: [px][4] rendered (R, G, B, depth), written by the
    // score raster and read by k_fisher in place of its pass 0
    double* rc4;
};

struct RasterParams {
    DevMap map;
    CamParams cam;
    OptParams opt;
    const ViewDesc* views;
    int tiles_per_view;  // raster tiles (8x8) per view
    int raster_tiles_x;
    uint32_t channels;   // SGM_COLOR | SGM_DEPTH | SGM_SEMANTICS
    GroupParams groups;
    int want_rc;         // score mode: also write vd.rc4 (colour / depth per pixel)
    int n_items;         // raster: (view, block) items of the launch (set by the launcher)
    int items_per_cta;   // raster: consecutive items per CTA (set by the launcher)
    int tm_first;        // raster (tensor-memory variant): first channel group held in TMEM
    // optional explicit (view, raster tile) items (the redo pass of depth-prefix binning);
    // null: every tile of every view of the launch
    const uint2* item_list;
    int n_item_list;
    // depth-prefix binning, per view v of the launch: trunc[v * bins + bin] = 1 when the bin's
    // list holds only its first entries; a block that exhausts such a list with pixels still
    // open appends its raster tile to incomplete[v * tiles_per_view ..] (count
    // n_incomplete[v]) to be redone from the full list. Null: every list is complete.
    const uint8_t* trunc;
    uint32_t* incomplete;
    uint32_t* n_incomplete;
};

// ---- launchers (sgm_kernels.cu) ----
void launch_preprocess(const DevMap& m, const PoseParams* d_poses, const CamParams& cam,
                       const OptParams& o, int n_views, uint32_t* keys, uint32_t* vals,
                       size_t stride, uint32_t* vcount, unsigned long long* pcount,
                       unsigned long long* rcount, cudaStream_t s);
void launch_tiefix(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                   const OptParams& o, const uint32_t* key, uint32_t* idx, uint32_t V,
                   cudaStream_t s);
void launch_pack(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                 const OptParams& o, const GroupParams& gp, const uint32_t* idx, uint32_t V,
                 PackedSplat* packed, unsigned long long* counts, int4* rects, uint4* bounds,
                 cudaStream_t s);
void launch_ranges(const uint32_t* sorted_tiles, uint64_t P, uint2* ranges, cudaStream_t s);
// row-bucketed binning (sgm_kernels.cu): tile ranges from a 2D difference array, each
// row's ranks in rank order, then a per-row ordered scatter into the tile lists
void launch_bin_hist_prefix(const int4* rects, uint32_t V, int tiles_x, int tiles_y, uint32_t cap, int nc,
                            int* diffc, int* sat, int* diff, unsigned long long* rows, cudaStream_t s);
void launch_bin_hist(const int4* rects, uint32_t V, int tiles_x, int* diff,
                     unsigned long long* rows, cudaStream_t s);
// mask: bins outside it get empty lists; total: the pairs allocated; cap: a bin keeps its
// first `cap` entries (depth-prefix binning), trunc[bin] = 1 when that drops some
void launch_bin_scan(int* diff, int tiles_x, int tiles_y, uint2* ranges, cudaStream_t s,
                     const uint8_t* mask = nullptr, unsigned long long* total = nullptr,
                     uint32_t cap = 0xffffffffu, uint8_t* trunc = nullptr);
// depth-prefix binning of dense views (sgm_pipeline.cu): the redo items / bin mask from a
// view's incomplete raster tiles
void launch_redo_items(const uint32_t* incomplete, uint32_t n, uint32_t view, int raster_tiles_x,
                       int per_bin, int tiles_x, uint2* items, uint8_t* mask, cudaStream_t s);
void launch_emit_rows(const unsigned long long* offsets, const int4* rects, uint32_t V,
                      unsigned long long R, uint32_t* row_keys, unsigned long long* row_vals,
                      cudaStream_t s);
void launch_row_scatter(const unsigned long long* row_list, const uint2* row_ranges,
                        const uint2* tile_ranges, int tiles_x, int tiles_y, uint64_t R, uint4* segs,
                        uint32_t* nseg, uint32_t* cnt, uint32_t* list, cudaStream_t s,
                        const uint8_t* mask = nullptr, bool part = false, bool cols = false);
uint64_t row_scatter_segments(uint64_t R, int tiles_y);  // upper bound on segments
void launch_seg_pass(const unsigned long long* row_list, const uint2* tile_ranges, int tiles_x,
                     uint64_t G, const uint4* segs, const uint32_t* nseg, const uint32_t* cnt,
                     uint32_t* list, const uint8_t* mask, cudaStream_t s, bool cols = false);
void launch_raster_score(const RasterParams& p, int n_views, cudaStream_t s);
void launch_raster_render(const RasterParams& p, int n_views, cudaStream_t s);
void launch_reduce_scores(const ViewDesc* views, int n_views, int tiles, double* out_missing,
                          double* out_entropy, double* out_fisher, cudaStream_t s);
void launch_fisher_prior(const RasterParams& p, const FisherParams& fp, int n_views, cudaStream_t s);
void launch_fisher_gain(const RasterParams& p, const FisherParams& fp, int n_views, cudaStream_t s);
void launch_fisher_invp(const double* H, double lambda, size_t n, double* invp, cudaStream_t s);
void launch_debug_projections(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                              const OptParams& o, const uint32_t* idx, uint32_t V,
                              double* out6, cudaStream_t s);
void launch_bins_to_ids(const uint32_t* list, uint64_t P, const PackedSplat* packed, int aniso,
                        double cut_sq, uint32_t* ids, float* probe3, cudaStream_t s);

void launch_sort_rows(const uint16_t* idx, const double* prob, uint64_t n, int k, int kpad,
                      uint16_t* out_idx, double* out_prob, uint16_t* out_perm, cudaStream_t s);
void launch_group_bounds(const DevMap& m, const GroupParams& gp, uint4* out, cudaStream_t s);
void launch_sem_records(const DevMap& m, uint4* out, cudaStream_t s);
// sgm_backward.cu
size_t backward_loss_blocks(int W, int H);
void launch_loss_pixels(const BackwardParams& b, double* part, double* totals, cudaStream_t s);
void launch_backward(const RasterParams& p, const BackwardParams& b, cudaStream_t s);
size_t backward_smem_bytes(int C, int kpad);
void launch_chain(const DevMap& m, const PoseParams* d_pose, const CamParams& cam, const OptParams& o,
                  const uint32_t* order, uint32_t V, const double* gproj, const BackwardParams& b,
                  cudaStream_t s);
void launch_kl_clip(double* gsem, uint64_t n, int k, double clip, cudaStream_t s);
void launch_finite(const double* v, uint64_t len, unsigned long long* bad, cudaStream_t s);

// sgm_emap.cu (exploration map, explorer.cpp:11-184)
struct EmapParams {
    double origin[3];
    double voxel;
    int dims[3];
    uint64_t nvox;
};
// Camera-to-world pose as the reference stores it (R row-major, t).
struct WorldPose {
    double R[9];
    double t[3];
};
void launch_emap_rays(const EmapParams& e, const CamParams& cam, const WorldPose& P,
                      const float* depth, int stride, const uint8_t* grid,
                      unsigned long long* first_free, uint32_t* first_hit, cudaStream_t s);
void launch_emap_seed(const EmapParams& e, const sgm_aabb& box, int occupied, const uint8_t* grid,
                      unsigned long long* first_free, uint32_t* first_hit, cudaStream_t s);
void launch_emap_resolve(const EmapParams& e, uint8_t* grid, unsigned long long* first_free,
                         uint32_t* first_hit, unsigned long long* log_keys, int32_t* log_ids,
                         unsigned long long* counters, cudaStream_t s);
void launch_emap_lattice(const EmapParams& e, const double* pos, int n, const uint8_t* grid,
                         const uint8_t* fresh, uint8_t* ok, cudaStream_t s);
void launch_emap_mark(const int32_t* ids, uint64_t n, uint8_t* flags, uint8_t value,
                      cudaStream_t s);
void launch_emap_free_ids(const EmapParams& e, const uint8_t* grid, unsigned long long* log_keys,
                          int32_t* log_ids, unsigned long long* counter, cudaStream_t s);

// sgm_optim.cu (AdamState::step, prune, snapshot re-derivation)
struct AdamHyper {
    double lr_center, lr_radius, lr_opacity, lr_color, lr_sem, beta1, beta2, eps, eps_sem;
};
void launch_adam(double* P, const double* G, double* M, double* V, uint64_t n, int k,
                 const AdamHyper& h, double bc1, double bc2, cudaStream_t s);
void launch_derive(const double* P, uint64_t n, int k, int kpad, const uint16_t* perm, double* geo,
                   double* color4, double* sprob, cudaStream_t s);
void launch_keep_flags(const double* logit, uint64_t n, double thr, uint8_t* keep, cudaStream_t s);
void launch_gather_f64(const double* src, double* dst, const uint32_t* kept, uint64_t m, int stride,
                       cudaStream_t s);
void launch_gather_u16(const uint16_t* src, uint16_t* dst, const uint32_t* kept, uint64_t m,
                       int stride, cudaStream_t s);

// sgm_eval.cu (semantic_metrics / photometric_metrics on device planes)
size_t eval_view_smem(int C);
void launch_eval_view(const double* sem, const double* sil, const float* fsem, int px, int C,
                      unsigned long long* confusion, unsigned long long* counters, uint16_t* label,
                      float* scores, cudaStream_t s);
int eval_photo_blocks(int px);
void launch_eval_photo(const double* color, const double* depth, const float* rgb,
                       const float* gdepth, int px, double* part, double* out, cudaStream_t s);
void launch_eval_keys(const float* scores, const uint16_t* label, uint32_t T, int c, uint32_t* keys,
                      uint32_t* pos, cudaStream_t s);
void launch_eval_ap_terms(const uint32_t* pos, const uint32_t* tp, uint32_t T, double P,
                          double* terms, cudaStream_t s);

// sgm_sort.cu: hand-written stable LSD radix sort (8-bit digits) of (u32 key, value) pairs over
// nseg segments (segment s at keys + s * stride, d_n[s] elements on the device, at most
// max_len), bits [0, end_bit). Returns true when the result is in the *_alt buffers.
size_t radix_sort_scratch_bytes(uint64_t max_len, int nseg);
template <typename V, typename N>
bool radix_sort_pairs(uint32_t* keys, V* vals, uint32_t* keys_alt, V* vals_alt, size_t stride,
                      const N* d_n, uint64_t max_len, int nseg, int end_bit, uint32_t* scratch,
                      cudaStream_t s);
int radix_sort_launches(int end_bit, uint64_t max_len);
int exclusive_scan_launches(uint64_t n);
// exclusive scan of n counts (u32 or u64) into u64 offsets
size_t exclusive_scan_scratch_bytes(uint64_t n);
template <typename C>
void exclusive_scan_u64(const C* in, uint64_t n, unsigned long long* out, unsigned long long* scratch,
                        cudaStream_t s);

// sgm_raster.cu
GroupParams choose_groups(int C, int k);
size_t raster_smem_bytes(const DevMap& m, const GroupParams& gp, bool render);
// the score raster runs 4 CTAs per SM, staging DevMap::sem_rec (needs map_records)
bool raster_score_records(const DevMap& m);

}  // namespace sgm
