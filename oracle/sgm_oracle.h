/* CPU restatement of the reference's candidate-view render + scoring path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker that tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg compare the CUDA product against; the product
 * (paper_2506_00225_b200) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks this restatement bit-for-bit against the
 * reference's own code compiled unmodified into oracle/_ref/libsgm_ref.so (projections,
 * planes, n_missing, entropy_sum, combine_scores) and against the reference tests'
 * known-answer values (proj/tests/test_splat_render.cpp:24-265,
 * proj/tests/test_explorer.cpp:183-378) stored in tests/golden/.
 *
 * Every function cites the reference lines it restates. Arithmetic is fp64 with no
 * FMA contraction (built with -ffp-contract=off), libm exp/log, and Eigen 3.3+
 * evaluation order for the 3x3 mat-vec: pc_i = a0 + (a1 + a2) (redux halving).
 */
#ifndef SGM_ORACLE_H
#define SGM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t width, height;
    double fx, fy, cx, cy;
} orc_camera; /* CameraModel, proj/include/splatmap/camera.hpp:11-50 */

typedef struct {
    double R[9]; /* cam->world rotation, row-major */
    double t[3];
} orc_pose; /* Pose, proj/include/splatmap/geometry.hpp:18-41 */

typedef struct {
    int32_t early_exit;
    double transmittance_eps, z_near, truncation_sigmas;
    int32_t tile_size;
} orc_options; /* RenderOptions, proj/include/splatmap/splat_render.hpp:22-28 */

typedef struct {
    uint64_t n;
    int32_t k, num_classes;
    const double *centers, *log_radii, *opacity_logits, *colors;
    const uint16_t* sem_idx;
    const double* sem_probs;
    /* Anisotropic splat mode (NO reference counterpart, parity unpinned):
     * when both are non-NULL, log_scales (3N, per-axis log sigma) and quats (4N, (w, x, y, z),
     * normalised here) replace log_radii. See orc_cov3 / orc_project below. */
    const double *log_scales, *quats;
} orc_map; /* GaussianMap SoA, proj/include/splatmap/gaussian_map.hpp:105-113 */

typedef struct {
    double mx, my, rad_px, z, alpha;
    uint32_t index;
    /* binning reach (x, y) in pixels and, anisotropic mode only, the conic (inverse 2D
     * covariance) qa, qb, qc. Isotropic: rx = ry = truncation_sigmas * rad_px (:205). */
    double rx, ry, qa, qb, qc;
} orc_proj; /* SplatProjection, splat_render.hpp:32-39 (+ mode fields) */

typedef struct {
    uint64_t visible;      /* V: culled-in projections */
    uint64_t pairs;        /* P: (tile, projection) pairs */
    uint64_t probe_tests;  /* float prefilter evaluations */
    uint64_t exact_tests;  /* fp64 d2 tests (prefilter survivors) */
    uint64_t contributors; /* K: composited (pixel, splat) pairs */
} orc_stats;

enum { ORC_COLOR = 1, ORC_DEPTH = 2, ORC_SEM = 4 };

/* World covariance of one anisotropic Gaussian, Sigma = R(q) diag(exp(2 ls)) R(q)^T, as
 * (xx, xy, xz, yy, yz, zz); evaluation order as documented in sgm_oracle.c. */
void orc_cov3(const double log_scale[3], const double quat[4], double out6[6]);

/* project_splats, proj/src/splat_render.cpp:15-47. Returns V; out holds >= map->n.
 * Anisotropic mode (EWA, Zwicker et al. 2001 as used by 3D Gaussian splatting):
 * Sigma2D = J R_cw Sigma R_cw^T J^T with J the pinhole Jacobian at the camera-space
 * centre, its direction x/z, y/z clamped to 1.3 (W/2)/fx, 1.3 (H/2)/fy; culled when det(Sigma2D) <= 0 or the truncated axis-aligned extent
 * (trunc sqrt(Sigma2D_xx), trunc sqrt(Sigma2D_yy)) misses the image (:34-37 analogue);
 * rad_px = sqrt(largest eigenvalue) (informational). The footprint is
 * alpha exp(-q / 2), q = d^T Sigma2D^-1 d, cut at q > trunc^2 (the isotropic d2 > 9 r^2). */
uint64_t orc_project(const orc_map* map, const orc_camera* cam, const orc_pose* pose,
                     const orc_options* opt, orc_proj* out);

/* Binning, proj/src/splat_render.cpp:189-213, over orc_project's output.
 * tile_offsets[tiles+1]; ids[P] (projection ids in bin order); probe3[3P] (float mx,
 * my, cutoff_d2). Returns P; if P > cap only the offsets are filled. */
uint64_t orc_bins(const orc_proj* proj, uint64_t v, const orc_camera* cam,
                  const orc_options* opt, uint32_t* tile_offsets, uint32_t* ids, float* probe3,
                  uint64_t cap);

/* render, proj/src/splat_render.cpp:170-328. Planes in the reference layout
 * (color px*3, depth px, silhouette px, sem px*C); NULL planes are skipped. */
int orc_render(const orc_map* map, const orc_camera* cam, const orc_pose* pose,
               uint32_t channels, const orc_options* opt, double* color, double* depth,
               double* silhouette, double* sem, orc_stats* stats);

/* clipped_entropy, proj/src/splat_render.cpp:360-369. */
double orc_clipped_entropy(const double* p, int n);

/* refresh_candidate_scores, proj/src/explorer.cpp:186-205, over explicit poses, with
 * `threads` pthreads over views (each view's sum is sequential row-major as in
 * the reference, so results do not depend on the thread count). */
int orc_score_views(const orc_map* map, const orc_camera* cam, uint64_t n_views,
                    const orc_pose* poses, const orc_options* opt, int threads,
                    double* n_missing, double* entropy_sum, orc_stats* stats);

/* Per-pixel clipped entropy image, render_entropy (splat_render.cpp:378-390). */
int orc_render_entropy(const orc_map* map, const orc_camera* cam, const orc_pose* pose,
                       const orc_options* opt, double* entropy);

/* combine_scores + stable_softmax, proj/src/explorer.cpp:209-248. Returns 1 if any > 0. */
int orc_combine_scores(uint64_t n, const double* n_missing, const double* entropy_sum,
                       const double* pos3, const double cur[3], double* i_geo, double* i_sem,
                       double* i_total);

/* Fisher-information extension (no reference counterpart). Parameters per
 * Gaussian, theta = (mu_x, mu_y, mu_z, log_radius, opacity_logit, c_r, c_g, c_b). Rendered
 * channels ch = (R, G, B, depth). The per-pixel Jacobian dR_ch/dtheta restates the analytic
 * chain of proj/src/losses.cpp:242-335 with unit seeds per channel (suffix sums formed as
 * S_j = R - P_j from the inclusive prefix P_j), chained to world space per pixel BEFORE squaring:
 *   H[8 i + theta] += sum_px sum_ch (dR_ch(px) / dtheta_i)^2
 * orc_fisher_accumulate adds the diagonal of all n poses into H (8 N doubles).
 * orc_fisher_gain returns per view  sum_{px,i,theta} J^2 / (H_prior[8 i + theta] + lambda). */
int orc_fisher_accumulate(const orc_map* map, const orc_camera* cam, uint64_t n_views,
                          const orc_pose* poses, const orc_options* opt, double* H);
int orc_fisher_gain(const orc_map* map, const orc_camera* cam, uint64_t n_views,
                    const orc_pose* poses, const orc_options* opt, const double* H_prior,
                    double lambda, double* gain);

/* CandidatePose::camera_pose() = look_at(p, p + d), explorer.hpp:105 + geometry.hpp:44-56. */
/* ExplorationMap, proj/include/splatmap/explorer.hpp:11-83 (grid states 0/1/2, changelog). */
typedef struct {
    double origin[3];
    double voxel;
    int32_t dims[3];
    uint64_t nvox;
    uint8_t* grid;
    int32_t* log;
    uint64_t log_n, free_count, occupied_count;
} orc_emap;

/* ExplorationMap ctor (explorer.cpp:11-20); returns 0, or -1 for voxel <= 0 / no memory. */
int orc_emap_init(orc_emap* e, const double bmin[3], const double bmax[3], double voxel);
void orc_emap_free(orc_emap* e);
/* integrate_frame (explorer.cpp:53-110), sequential; returns the newly logged count. */
uint64_t orc_emap_integrate(orc_emap* e, const orc_camera* cam, const orc_pose* pose,
                            const float* depth, int stride);
/* seed_free_region / seed_occupied_region (explorer.cpp:124-132). */
void orc_emap_seed(orc_emap* e, const double bmin[3], const double bmax[3], int occupied);
/* reseed_changelog_with_free (explorer.cpp:118-122). */
void orc_emap_reseed(orc_emap* e);
/* fibonacci_directions (explorer.cpp:142-155). */
void orc_fibonacci_directions(int count, double max_elev_deg, double* out3);
/* sample_candidates (explorer.cpp:157-184): consumes the changelog; writes up to capacity
 * (position, direction) 6-tuples and returns the total count. */
uint64_t orc_sample_candidates(orc_emap* e, double v1, int v2, const double* heights, int nh,
                               double* out6, uint64_t capacity);

void orc_candidate_pose(const double pos[3], const double dir[3], orc_pose* out);
void orc_look_at(const double pos[3], const double target[3], orc_pose* out);

#ifdef __cplusplus
}
#endif
#endif
