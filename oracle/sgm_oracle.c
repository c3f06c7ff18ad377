/* CPU restatement of the reference render + candidate scoring path.
 * TEST INFRASTRUCTURE ONLY (see sgm_oracle.h for the pinning story).
 * Build: gcc -O3 -std=c11 -ffp-contract=off -pthread (oracle/Makefile).
 */
#include "sgm_oracle.h"

#include <limits.h>
#include <pthread.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define K_MAX_FOOTPRINT 0.999999 /* kMaxFootprint, splat_render.hpp:41 */

/* x86-64 cvttsd2si semantics of static_cast<int>(double) as the reference build
 * executes it: out-of-range and NaN give INT_MIN. */
static int to_int_x86(double v) {
    if (!(v > -2147483649.0 && v < 2147483648.0)) return INT_MIN;
    return (int)v;
}

static double clampd(double v, double lo, double hi) {
    /* std::clamp(v, lo, hi): (v < lo) ? lo : (hi < v) ? hi : v */
    return v < lo ? lo : (hi < v ? hi : v);
}

/* ---- project_splats: splat_render.cpp:15-47 ---- */
static int proj_less(const orc_proj* a, const orc_proj* b) {
    if (a->z != b->z) return a->z < b->z;
    if (a->mx != b->mx) return a->mx < b->mx;
    if (a->my != b->my) return a->my < b->my;
    if (a->alpha != b->alpha) return a->alpha < b->alpha;
    /* Exact 4-key ties are unspecified in the reference (std::sort is not
     * stable); the restatement breaks them by map index. */
    return a->index < b->index;
}
static int proj_cmp(const void* pa, const void* pb) {
    const orc_proj* a = (const orc_proj*)pa;
    const orc_proj* b = (const orc_proj*)pb;
    if (proj_less(a, b)) return -1;
    if (proj_less(b, a)) return 1;
    return 0;
}

/* ---- anisotropic mode (f4, no reference): covariance and EWA projection ----
 * Every expression is evaluated left to right with one rounding per operation
 * (-ffp-contract=off); the CUDA product uses the same order, so projections and bins
 * are bit-identical between the two. */
void orc_cov3(const double ls[3], const double q4[4], double S[6]) {
    const double nrm = sqrt(((q4[0] * q4[0] + q4[1] * q4[1]) + q4[2] * q4[2]) + q4[3] * q4[3]);
    const double w = q4[0] / nrm, x = q4[1] / nrm, y = q4[2] / nrm, z = q4[3] / nrm;
    double R[9];
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - w * z);
    R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y);
    R[7] = 2.0 * (y * z + w * x);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
    const double s0 = exp(ls[0]), s1 = exp(ls[1]), s2 = exp(ls[2]);
    const double v0 = s0 * s0, v1 = s1 * s1, v2 = s2 * s2;
    static const int I[6] = {0, 0, 0, 1, 1, 2}, J[6] = {0, 1, 2, 1, 2, 2};
    for (int e = 0; e < 6; ++e) {
        const double* a = R + 3 * I[e];
        const double* b = R + 3 * J[e];
        S[e] = ((a[0] * b[0]) * v0 + (a[1] * b[1]) * v1) + (a[2] * b[2]) * v2;
    }
}

/* Sigma2D and the cull of one anisotropic Gaussian at camera-space (pcx, pcy, pcz). */
static int ewa_project(const double S[6], const double* R, const orc_camera* cam,
                       const orc_options* opt, double pcx, double pcy, double pcz, orc_proj* p) {
    /* the Jacobian is taken at the view direction clamped to 1.3x the half field of view
     * (as 3D Gaussian splatting does): the linearisation is meaningless for centres far
     * outside the frustum, where the unclamped -f x / z^2 term explodes near z_near */
    const double limx = 1.3 * ((0.5 * cam->width) / cam->fx);
    const double limy = 1.3 * ((0.5 * cam->height) / cam->fy);
    const double txz = clampd(pcx / pcz, -limx, limx), tyz = clampd(pcy / pcz, -limy, limy);
    const double tx = txz * pcz, ty = tyz * pcz;
    const double zz = pcz * pcz;
    const double j00 = cam->fx / pcz, j02 = -(cam->fx * tx) / zz;
    const double j11 = cam->fy / pcz, j12 = -(cam->fy * ty) / zz;
    /* M = J R_cw; R_cw(i, k) = R[3 k + i] */
    const double a0 = j00 * R[0] + j02 * R[2], a1 = j00 * R[3] + j02 * R[5],
                 a2 = j00 * R[6] + j02 * R[8];
    const double b0 = j11 * R[1] + j12 * R[2], b1 = j11 * R[4] + j12 * R[5],
                 b2 = j11 * R[7] + j12 * R[8];
    const double ta0 = (S[0] * a0 + S[1] * a1) + S[2] * a2;
    const double ta1 = (S[1] * a0 + S[3] * a1) + S[4] * a2;
    const double ta2 = (S[2] * a0 + S[4] * a1) + S[5] * a2;
    const double tb0 = (S[0] * b0 + S[1] * b1) + S[2] * b2;
    const double tb1 = (S[1] * b0 + S[3] * b1) + S[4] * b2;
    const double tb2 = (S[2] * b0 + S[4] * b1) + S[5] * b2;
    const double va = (a0 * ta0 + a1 * ta1) + a2 * ta2;
    const double vb = (b0 * ta0 + b1 * ta1) + b2 * ta2;
    const double vc = (b0 * tb0 + b1 * tb1) + b2 * tb2;
    const double det = va * vc - vb * vb;
    if (!(det > 0.0)) return 0;
    p->rx = opt->truncation_sigmas * sqrt(va);
    p->ry = opt->truncation_sigmas * sqrt(vc);
    if (p->mx + p->rx < 0 || p->mx - p->rx > cam->width || p->my + p->ry < 0 ||
        p->my - p->ry > cam->height)
        return 0;
    p->qa = vc / det;
    p->qb = -vb / det;
    p->qc = va / det;
    const double hm = 0.5 * (va + vc), hd = 0.5 * (va - vc);
    p->rad_px = sqrt(hm + sqrt(hd * hd + vb * vb));
    return 1;
}

uint64_t orc_project(const orc_map* map, const orc_camera* cam, const orc_pose* pose,
                     const orc_options* opt, orc_proj* out) {
    const double* R = pose->R; /* R_cw(i,j) = R(j,i) (splat_render.cpp:19) */
    const int aniso = map->log_scales && map->quats;
    uint64_t v = 0;
    for (uint64_t i = 0; i < map->n; ++i) {
        const double d0 = map->centers[3 * i] - pose->t[0];
        const double d1 = map->centers[3 * i + 1] - pose->t[1];
        const double d2 = map->centers[3 * i + 2] - pose->t[2];
        /* Eigen lazy product row i: x0 + (x1 + x2) (splat_render.cpp:25) */
        const double pcx = R[0] * d0 + (R[3] * d1 + R[6] * d2);
        const double pcy = R[1] * d0 + (R[4] * d1 + R[7] * d2);
        const double pcz = R[2] * d0 + (R[5] * d1 + R[8] * d2);
        if (pcz <= opt->z_near) continue; /* :26 */
        orc_proj p;
        memset(&p, 0, sizeof(p));
        p.z = pcz;
        p.mx = cam->fx * pcx / pcz + cam->cx; /* :29 */
        p.my = cam->fy * pcy / pcz + cam->cy; /* :30 */
        p.alpha = 1.0 / (1.0 + exp(-map->opacity_logits[i])); /* sigmoid, geometry.hpp:84 */
        p.index = (uint32_t)i;
        if (aniso) {
            double S[6];
            orc_cov3(&map->log_scales[3 * i], &map->quats[4 * i], S);
            if (!ewa_project(S, R, cam, opt, pcx, pcy, pcz, &p)) continue;
            out[v++] = p;
            continue;
        }
        p.rad_px = exp(map->log_radii[i]) * cam->fy / pcz; /* :31 */
        const double reach = opt->truncation_sigmas * p.rad_px; /* :34 */
        p.rx = p.ry = reach;
        if (p.mx + reach < 0 || p.mx - reach > cam->width || p.my + reach < 0 ||
            p.my - reach > cam->height)
            continue; /* :35-37 */
        out[v++] = p;
    }
    qsort(out, v, sizeof(orc_proj), proj_cmp); /* :40-45 */
    return v;
}

/* ---- binning: splat_render.cpp:189-213 ---- */
typedef struct {
    int tx0, tx1, ty0, ty1;
} rect_t;

static rect_t tile_rect(const orc_proj* p, const orc_camera* cam, const orc_options* opt) {
    const int ts = opt->tile_size;
    const int tiles_x = (cam->width + ts - 1) / ts;
    const int tiles_y = (cam->height + ts - 1) / ts;
    /* reach = truncation_sigmas * rad_px (:205); per axis in the anisotropic mode */
    rect_t r;
    int a;
    a = to_int_x86((p->mx - p->rx) / ts);
    r.tx0 = a > 0 ? a : 0; /* :206 */
    a = to_int_x86((p->mx + p->rx) / ts);
    r.tx1 = a < tiles_x - 1 ? a : tiles_x - 1; /* :207 */
    a = to_int_x86((p->my - p->ry) / ts);
    r.ty0 = a > 0 ? a : 0; /* :208 */
    a = to_int_x86((p->my + p->ry) / ts);
    r.ty1 = a < tiles_y - 1 ? a : tiles_y - 1; /* :209 */
    return r;
}

static float probe_cutoff(double rad_px, double trunc) {
    const double cut_sq = trunc * trunc;              /* :180 */
    const double cutoff_d2 = cut_sq * rad_px * rad_px; /* :195 */
    return (float)(cutoff_d2 * (1.0 + 1e-5)) + 1e-6f;  /* :203 */
}

uint64_t orc_bins(const orc_proj* proj, uint64_t v, const orc_camera* cam,
                  const orc_options* opt, uint32_t* tile_offsets, uint32_t* ids, float* probe3,
                  uint64_t cap) {
    const int ts = opt->tile_size;
    const int tiles_x = (cam->width + ts - 1) / ts;
    const int tiles_y = (cam->height + ts - 1) / ts;
    const uint64_t ntiles = (uint64_t)tiles_x * tiles_y;
    memset(tile_offsets, 0, (ntiles + 1) * sizeof(uint32_t));
    uint64_t total = 0;
    for (uint64_t pi = 0; pi < v; ++pi) {
        rect_t r = tile_rect(&proj[pi], cam, opt);
        for (int ty = r.ty0; ty <= r.ty1; ++ty)
            for (int tx = r.tx0; tx <= r.tx1; ++tx) {
                tile_offsets[(uint64_t)ty * tiles_x + tx + 1]++;
                ++total;
            }
    }
    for (uint64_t t = 0; t < ntiles; ++t) tile_offsets[t + 1] += tile_offsets[t];
    if (total > cap || !ids) return total;
    uint32_t* cursor = (uint32_t*)malloc(ntiles * sizeof(uint32_t));
    memcpy(cursor, tile_offsets, ntiles * sizeof(uint32_t));
    for (uint64_t pi = 0; pi < v; ++pi) { /* depth order => each bin in depth order */
        rect_t r = tile_rect(&proj[pi], cam, opt);
        /* anisotropic entries (qa > 0) carry the Mahalanobis cut trunc^2 instead */
        const float cut = proj[pi].qa > 0.0
                              ? (float)(opt->truncation_sigmas * opt->truncation_sigmas)
                              : probe_cutoff(proj[pi].rad_px, opt->truncation_sigmas);
        for (int ty = r.ty0; ty <= r.ty1; ++ty)
            for (int tx = r.tx0; tx <= r.tx1; ++tx) {
                const uint32_t at = cursor[(uint64_t)ty * tiles_x + tx]++;
                ids[at] = (uint32_t)pi;
                if (probe3) {
                    probe3[3 * (uint64_t)at] = (float)proj[pi].mx;
                    probe3[3 * (uint64_t)at + 1] = (float)proj[pi].my;
                    probe3[3 * (uint64_t)at + 2] = cut;
                }
            }
    }
    free(cursor);
    return total;
}

/* ---- per-view prepared state ---- */
typedef struct {
    orc_proj* proj;
    uint64_t v, pairs;
    double *inv_two_r2, *cutoff_d2; /* PackedSplat, :191-199 */
    float* probe3;
    uint32_t *offsets, *ids;
    int tiles_x, tiles_y;
} view_t;

static int view_prepare(view_t* s, const orc_map* map, const orc_camera* cam,
                        const orc_pose* pose, const orc_options* opt) {
    memset(s, 0, sizeof(*s));
    const int ts = opt->tile_size;
    s->tiles_x = (cam->width + ts - 1) / ts;
    s->tiles_y = (cam->height + ts - 1) / ts;
    const uint64_t ntiles = (uint64_t)s->tiles_x * s->tiles_y;
    s->proj = (orc_proj*)malloc((map->n ? map->n : 1) * sizeof(orc_proj));
    s->offsets = (uint32_t*)malloc((ntiles + 1) * sizeof(uint32_t));
    if (!s->proj || !s->offsets) return -1;
    s->v = orc_project(map, cam, pose, opt, s->proj);
    s->inv_two_r2 = (double*)malloc((s->v ? s->v : 1) * sizeof(double));
    s->cutoff_d2 = (double*)malloc((s->v ? s->v : 1) * sizeof(double));
    const double cut_sq = opt->truncation_sigmas * opt->truncation_sigmas;
    for (uint64_t i = 0; i < s->v; ++i) {
        const double r = s->proj[i].rad_px;
        s->inv_two_r2[i] = 1.0 / (2.0 * r * r); /* :194 */
        s->cutoff_d2[i] = cut_sq * r * r;       /* :195 */
    }
    s->pairs = orc_bins(s->proj, s->v, cam, opt, s->offsets, NULL, NULL, 0);
    s->ids = (uint32_t*)malloc((s->pairs ? s->pairs : 1) * sizeof(uint32_t));
    s->probe3 = (float*)malloc((s->pairs ? s->pairs : 1) * 3 * sizeof(float));
    if (!s->ids || !s->probe3) return -1;
    orc_bins(s->proj, s->v, cam, opt, s->offsets, s->ids, s->probe3, s->pairs);
    return 0;
}

static void view_free(view_t* s) {
    free(s->proj);
    free(s->inv_two_r2);
    free(s->cutoff_d2);
    free(s->probe3);
    free(s->offsets);
    free(s->ids);
}

/* Composite one pixel over its tile's bin: splat_render.cpp:261-320. Accumulates
 * into sem_px (C doubles, pre-zeroed) and returns transmittance. */
static double composite(const view_t* s, const orc_map* map, const orc_options* opt,
                        uint32_t channels, uint32_t b0, uint32_t b1, int x, int y,
                        double acc_color[3], double* acc_depth, double* sem_px, orc_stats* st) {
    const double px = x + 0.5, py = y + 0.5;
    const float pxf = (float)px, pyf = (float)py;
    const int k = map->k;
    const int aniso = map->log_scales && map->quats;
    const double cut_sq = opt->truncation_sigmas * opt->truncation_sigmas;
    double T = 1.0;
    uint64_t probes = 0, exact = 0, contrib = 0;
    for (uint32_t b = b0; b < b1; ++b) {
        ++probes;
        if (aniso) { /* f4: no float probe; exact Mahalanobis test */
            ++exact;
            const uint32_t pid = s->ids[b];
            const orc_proj* p = &s->proj[pid];
            const double dx = px - p->mx;
            const double dy = py - p->my;
            const double q = (p->qa * (dx * dx) + (2.0 * p->qb) * (dx * dy)) + p->qc * (dy * dy);
            if (q > cut_sq) continue;
            ++contrib;
            double f = p->alpha * exp(-0.5 * q);
            if (f > K_MAX_FOOTPRINT) f = K_MAX_FOOTPRINT;
            const double w = f * T;
            if (channels & ORC_COLOR) {
                const double* c = &map->colors[(uint64_t)p->index * 3];
                acc_color[0] += clampd(c[0], 0.0, 1.0) * w;
                acc_color[1] += clampd(c[1], 0.0, 1.0) * w;
                acc_color[2] += clampd(c[2], 0.0, 1.0) * w;
            }
            if (channels & ORC_DEPTH) *acc_depth += p->z * w;
            if (channels & ORC_SEM) {
                const uint16_t* idx = &map->sem_idx[(uint64_t)p->index * k];
                const double* pr = &map->sem_probs[(uint64_t)p->index * k];
                for (int j = 0; j < k; ++j) sem_px[idx[j]] += pr[j] * w;
            }
            T *= (1.0 - f);
            if (opt->early_exit && T < opt->transmittance_eps) break;
            continue;
        }
        const float fdx = pxf - s->probe3[3 * (uint64_t)b];
        const float fdy = pyf - s->probe3[3 * (uint64_t)b + 1];
        if (fdx * fdx + fdy * fdy > s->probe3[3 * (uint64_t)b + 2]) continue; /* :276-278 */
        ++exact;
        const uint32_t pid = s->ids[b];
        const orc_proj* p = &s->proj[pid];
        const double dx = px - p->mx;
        const double dy = py - p->my;
        const double d2 = dx * dx + dy * dy;
        if (d2 > s->cutoff_d2[pid]) continue; /* :283 */
        ++contrib;
        double f = p->alpha * exp(-d2 * s->inv_two_r2[pid]); /* :284 */
        if (f > K_MAX_FOOTPRINT) f = K_MAX_FOOTPRINT;        /* :285 */
        const double w = f * T;
        if (channels & ORC_COLOR) {
            const double* c = &map->colors[(uint64_t)p->index * 3];
            acc_color[0] += clampd(c[0], 0.0, 1.0) * w;
            acc_color[1] += clampd(c[1], 0.0, 1.0) * w;
            acc_color[2] += clampd(c[2], 0.0, 1.0) * w;
        }
        if (channels & ORC_DEPTH) *acc_depth += p->z * w; /* :293 */
        if (channels & ORC_SEM) {
            const uint16_t* idx = &map->sem_idx[(uint64_t)p->index * k];
            const double* pr = &map->sem_probs[(uint64_t)p->index * k];
            for (int j = 0; j < k; ++j) sem_px[idx[j]] += pr[j] * w; /* :305-307 */
        }
        T *= (1.0 - f);                                                 /* :311 */
        if (opt->early_exit && T < opt->transmittance_eps) break;      /* :312 */
    }
    if (st) {
        st->probe_tests += probes;
        st->exact_tests += exact;
        st->contributors += contrib;
    }
    return T;
}

int orc_render(const orc_map* map, const orc_camera* cam, const orc_pose* pose,
               uint32_t channels, const orc_options* opt, double* color, double* depth,
               double* silhouette, double* sem, orc_stats* stats) {
    view_t s;
    if (view_prepare(&s, map, cam, pose, opt)) {
        view_free(&s);
        return -1;
    }
    const int W = cam->width, H = cam->height, C = map->num_classes + 1;
    const uint64_t px_count = (uint64_t)W * H;
    /* alloc_output zero-fills every plane (:57-63) */
    if (color) memset(color, 0, px_count * 3 * sizeof(double));
    if (depth) memset(depth, 0, px_count * sizeof(double));
    if (silhouette) memset(silhouette, 0, px_count * sizeof(double));
    if (sem) memset(sem, 0, px_count * C * sizeof(double));
    if (!sem) channels &= ~(uint32_t)ORC_SEM;
    double* scratch = (double*)calloc((size_t)C, sizeof(double));
    const int ts = opt->tile_size;
    for (int ty = 0; ty < s.tiles_y; ++ty)
        for (int tx = 0; tx < s.tiles_x; ++tx) {
            const uint64_t tile = (uint64_t)ty * s.tiles_x + tx;
            const uint32_t b0 = s.offsets[tile], b1 = s.offsets[tile + 1];
            if (b0 == b1) continue; /* :257 */
            const int y1 = H < (ty + 1) * ts ? H : (ty + 1) * ts;
            const int x1 = W < (tx + 1) * ts ? W : (tx + 1) * ts;
            for (int y = ty * ts; y < y1; ++y)
                for (int x = tx * ts; x < x1; ++x) {
                    const uint64_t pix = (uint64_t)y * W + x;
                    double ac[3] = {0, 0, 0}, ad = 0.0;
                    double* sp = (channels & ORC_SEM) ? &sem[pix * C] : scratch;
                    double T = composite(&s, map, opt, channels, b0, b1, x, y, ac, &ad, sp, stats);
                    if (silhouette) silhouette[pix] = 1.0 - T; /* :314 */
                    if (color && (channels & ORC_COLOR)) {
                        color[pix * 3] = ac[0];
                        color[pix * 3 + 1] = ac[1];
                        color[pix * 3 + 2] = ac[2];
                    }
                    if (depth && (channels & ORC_DEPTH)) depth[pix] = ad;
                }
        }
    if (stats) {
        stats->visible += s.v;
        stats->pairs += s.pairs;
    }
    free(scratch);
    view_free(&s);
    return 0;
}

double orc_clipped_entropy(const double* p, int n) {
    double total = 0.0;
    for (int i = 0; i < n; ++i) total += clampd(p[i], 0.001, 1.0); /* :362 */
    double h = 0.0;
    for (int i = 0; i < n; ++i) {
        const double q = clampd(p[i], 0.001, 1.0) / total; /* :365 */
        h -= q * log(q);                                   /* :366 */
    }
    return h;
}

/* Sem-only render of one view with per-pixel entropy and exact-zero silhouette
 * flags; the sem plane is kept one pixel at a time (pixels are independent). */
static int score_one(const orc_map* map, const orc_camera* cam, const orc_pose* pose,
                     const orc_options* opt, double* ent_px, double* n_missing,
                     double* entropy_sum, orc_stats* st) {
    view_t s;
    if (view_prepare(&s, map, cam, pose, opt)) {
        view_free(&s);
        return -1;
    }
    const int W = cam->width, H = cam->height, C = map->num_classes + 1;
    const uint64_t px_count = (uint64_t)W * H;
    double* sem_px = (double*)malloc((size_t)C * sizeof(double));
    double* zero = (double*)calloc((size_t)C, sizeof(double));
    const double h_empty = orc_clipped_entropy(zero, C);
    unsigned char* covered = (unsigned char*)calloc(px_count, 1);
    double* sil = (double*)calloc(px_count, sizeof(double));
    for (uint64_t i = 0; i < px_count; ++i) ent_px[i] = h_empty;
    const int ts = opt->tile_size;
    for (int ty = 0; ty < s.tiles_y; ++ty)
        for (int tx = 0; tx < s.tiles_x; ++tx) {
            const uint64_t tile = (uint64_t)ty * s.tiles_x + tx;
            const uint32_t b0 = s.offsets[tile], b1 = s.offsets[tile + 1];
            if (b0 == b1) continue;
            const int y1 = H < (ty + 1) * ts ? H : (ty + 1) * ts;
            const int x1 = W < (tx + 1) * ts ? W : (tx + 1) * ts;
            for (int y = ty * ts; y < y1; ++y)
                for (int x = tx * ts; x < x1; ++x) {
                    const uint64_t pix = (uint64_t)y * W + x;
                    memset(sem_px, 0, (size_t)C * sizeof(double));
                    double ac[3], ad;
                    const double T = composite(&s, map, opt, ORC_SEM, b0, b1, x, y, ac, &ad,
                                               sem_px, st);
                    sil[pix] = 1.0 - T;
                    covered[pix] = 1;
                    ent_px[pix] = orc_clipped_entropy(sem_px, C);
                }
        }
    /* explorer.cpp:195-203: sequential row-major sums */
    uint64_t missing = 0;
    double entropy = 0.0;
    for (uint64_t i = 0; i < px_count; ++i) {
        if (sil[i] == 0.0) ++missing;
        entropy += ent_px[i];
    }
    *n_missing = (double)missing;
    *entropy_sum = entropy;
    if (st) {
        st->visible += s.v;
        st->pairs += s.pairs;
    }
    free(sem_px);
    free(zero);
    free(covered);
    free(sil);
    view_free(&s);
    return 0;
}

typedef struct {
    const orc_map* map;
    const orc_camera* cam;
    const orc_pose* poses;
    const orc_options* opt;
    double *n_missing, *entropy_sum;
    uint64_t n_views;
    uint64_t next; /* shared view cursor (guarded by mu) */
    pthread_mutex_t mu;
    orc_stats total;
    int err;
} score_job_t;

static void* score_worker(void* arg) {
    score_job_t* job = (score_job_t*)arg;
    const uint64_t px_count = (uint64_t)job->cam->width * job->cam->height;
    double* ent = (double*)malloc((px_count ? px_count : 1) * sizeof(double));
    for (;;) {
        pthread_mutex_lock(&job->mu);
        const uint64_t v = job->next++;
        pthread_mutex_unlock(&job->mu);
        if (v >= job->n_views) break;
        orc_stats st;
        memset(&st, 0, sizeof(st));
        const int e = score_one(job->map, job->cam, &job->poses[v], job->opt, ent,
                                &job->n_missing[v], &job->entropy_sum[v], &st);
        pthread_mutex_lock(&job->mu);
        job->err |= e;
        job->total.visible += st.visible;
        job->total.pairs += st.pairs;
        job->total.probe_tests += st.probe_tests;
        job->total.exact_tests += st.exact_tests;
        job->total.contributors += st.contributors;
        pthread_mutex_unlock(&job->mu);
    }
    free(ent);
    return NULL;
}

int orc_score_views(const orc_map* map, const orc_camera* cam, uint64_t n_views,
                    const orc_pose* poses, const orc_options* opt, int threads,
                    double* n_missing, double* entropy_sum, orc_stats* stats) {
    score_job_t job;
    memset(&job, 0, sizeof(job));
    job.map = map;
    job.cam = cam;
    job.poses = poses;
    job.opt = opt;
    job.n_missing = n_missing;
    job.entropy_sum = entropy_sum;
    job.n_views = n_views;
    pthread_mutex_init(&job.mu, NULL);
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n_views) threads = n_views ? (int)n_views : 1;
    pthread_t* th = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
    for (int i = 1; i < threads; ++i) pthread_create(&th[i], NULL, score_worker, &job);
    score_worker(&job);
    for (int i = 1; i < threads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&job.mu);
    if (stats) *stats = job.total;
    return job.err ? -1 : 0;
}

int orc_render_entropy(const orc_map* map, const orc_camera* cam, const orc_pose* pose,
                       const orc_options* opt, double* entropy) {
    double nm, es;
    return score_one(map, cam, pose, opt, entropy, &nm, &es, NULL);
}

/* ---- combine_scores: explorer.cpp:209-248 ---- */
static void stable_softmax(const double* v, uint64_t n, double* out) {
    double mx = -INFINITY;
    for (uint64_t i = 0; i < n; ++i) {
        out[i] = 0.0;
        if (isfinite(v[i])) mx = v[i] > mx ? v[i] : mx; /* std::max(mx, x) */
    }
    if (!isfinite(mx)) return;
    double sum = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        out[i] = isfinite(v[i]) ? exp(v[i] - mx) : 0.0;
        sum += out[i];
    }
    for (uint64_t i = 0; i < n; ++i) out[i] /= sum;
}

int orc_combine_scores(uint64_t n, const double* n_missing, const double* entropy_sum,
                       const double* pos3, const double cur[3], double* i_geo, double* i_sem,
                       double* i_total) {
    if (n == 0) return 0;
    double* lm = (double*)malloc(n * sizeof(double));
    double* dist = (double*)malloc(n * sizeof(double));
    double* ds = (double*)malloc(n * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) {
        lm[i] = n_missing[i] > 0.0 ? log(n_missing[i]) : -INFINITY;
        const double a = pos3[3 * i] - cur[0], b = pos3[3 * i + 1] - cur[1],
                     c = pos3[3 * i + 2] - cur[2];
        dist[i] = sqrt(a * a + (b * b + c * c)); /* Eigen norm(): redux halving */
    }
    stable_softmax(lm, n, i_geo);
    stable_softmax(entropy_sum, n, i_sem);
    stable_softmax(dist, n, ds);
    int any = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double dist_factor = n == 1 ? 1.0 : 1.0 - ds[i];
        i_total[i] = dist_factor * i_geo[i] * i_sem[i];
        if (i_total[i] > 0.0) any = 1;
    }
    free(lm);
    free(dist);
    free(ds);
    return any;
}

/* ---- look_at: geometry.hpp:44-56 with Eigen's evaluation order ---- */
static void normalize3(double v[3]) {
    const double z = v[0] * v[0] + (v[1] * v[1] + v[2] * v[2]);
    if (z > 0.0) {
        const double s = sqrt(z);
        v[0] /= s;
        v[1] /= s;
        v[2] /= s;
    }
}
static void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

void orc_look_at(const double pos[3], const double target[3], orc_pose* out) {
    static const double up[3] = {0.0, 1.0, 0.0};
    static const double ux[3] = {1.0, 0.0, 0.0};
    double z[3] = {target[0] - pos[0], target[1] - pos[1], target[2] - pos[2]};
    normalize3(z);
    double x[3], y[3];
    cross3(z, up, x);
    if (sqrt(x[0] * x[0] + (x[1] * x[1] + x[2] * x[2])) < 1e-9) cross3(z, ux, x);
    normalize3(x);
    cross3(z, x, y);
    for (int i = 0; i < 3; ++i) {
        out->R[3 * i + 0] = x[i];
        out->R[3 * i + 1] = y[i];
        out->R[3 * i + 2] = z[i];
        out->t[i] = pos[i];
    }
}

void orc_candidate_pose(const double pos[3], const double dir[3], orc_pose* out) {
    const double target[3] = {pos[0] + dir[0], pos[1] + dir[1], pos[2] + dir[2]};
    orc_look_at(pos, target, out);
}

/* ---- Fisher-information extension ---- */

/* J^2 contributions of every contributor of one pixel, in depth order. `sink(i, th, v)`
 * receives v = sum over the 4 channels of (dR_ch/dtheta_i)^2 for theta = th. */
typedef void (*fisher_sink)(void* ctx, uint32_t map_index, int theta, double v);

static void fisher_pixel(const view_t* s, const orc_map* map, const orc_camera* cam,
                         const orc_pose* pose, const orc_options* opt, uint32_t b0, uint32_t b1,
                         int x, int y, fisher_sink sink, void* sctx, uint32_t* ids, double* fs,
                         double* ts, unsigned char* clamped) {
    const double px = x + 0.5, py = y + 0.5;
    const float pxf = (float)px, pyf = (float)py;
    /* forward: the contributor sequence exactly as composite() (splat_render.cpp:275-313) */
    uint32_t n = 0;
    double T = 1.0, Rc[4] = {0, 0, 0, 0};
    for (uint32_t b = b0; b < b1; ++b) {
        const float fdx = pxf - s->probe3[3 * (uint64_t)b];
        const float fdy = pyf - s->probe3[3 * (uint64_t)b + 1];
        if (fdx * fdx + fdy * fdy > s->probe3[3 * (uint64_t)b + 2]) continue;
        const uint32_t pid = s->ids[b];
        const orc_proj* p = &s->proj[pid];
        const double dx = px - p->mx, dy = py - p->my;
        const double d2 = dx * dx + dy * dy;
        if (d2 > s->cutoff_d2[pid]) continue;
        double f = p->alpha * exp(-d2 * s->inv_two_r2[pid]);
        clamped[n] = f > K_MAX_FOOTPRINT;
        if (f > K_MAX_FOOTPRINT) f = K_MAX_FOOTPRINT;
        const double w = f * T;
        const double* c = &map->colors[(uint64_t)p->index * 3];
        for (int ch = 0; ch < 3; ++ch) Rc[ch] += clampd(c[ch], 0.0, 1.0) * w;
        Rc[3] += p->z * w;
        ids[n] = pid;
        fs[n] = f;
        ts[n] = T;
        ++n;
        T *= (1.0 - f);
        if (opt->early_exit && T < opt->transmittance_eps) break;
    }
    /* per contributor: dR/df with S = R - P (inclusive prefix), losses.cpp:285-288 */
    double P[4] = {0, 0, 0, 0};
    const double* R = pose->R;
    for (uint32_t j = 0; j < n; ++j) {
        const orc_proj* p = &s->proj[ids[j]];
        const double f = fs[j], Tj = ts[j], w = f * Tj;
        const double* craw = &map->colors[(uint64_t)p->index * 3];
        double v[4];
        for (int ch = 0; ch < 3; ++ch) v[ch] = clampd(craw[ch], 0.0, 1.0);
        v[3] = p->z;
        double Jsq[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const double dx = px - p->mx, dy = py - p->my;
        const double r = p->rad_px, r2 = r * r;
        for (int ch = 0; ch < 4; ++ch) {
            P[ch] += v[ch] * w;
            const double S = Rc[ch] - P[ch];
            const double dRdf = v[ch] * Tj - S / (1.0 - f);
            double g_a = 0, g_mx = 0, g_my = 0, g_r = 0;
            if (!clamped[j] && r > 0.0) { /* losses.cpp:297-304 */
                g_a = dRdf * f / p->alpha;
                g_mx = dRdf * f * dx / r2;
                g_my = dRdf * f * dy / r2;
                g_r = dRdf * f * (dx * dx + dy * dy) / (r2 * r);
            }
            const double g_z = ch == 3 ? w : 0.0; /* depth channel: dD/dz = w */
            /* projection -> world, losses.cpp:323-334 */
            const double dX = g_mx * cam->fx / p->z;
            const double dY = g_my * cam->fy / p->z;
            const double dZ = g_z - g_mx * (p->mx - cam->cx) / p->z - g_my * (p->my - cam->cy) / p->z -
                              g_r * r / p->z;
            for (int a = 0; a < 3; ++a) {
                const double dw = R[3 * a] * dX + R[3 * a + 1] * dY + R[3 * a + 2] * dZ;
                Jsq[a] += dw * dw;
            }
            const double jl = g_r * r; /* d/d log_r = g_r * rad_px, :333 */
            const double jo = g_a * p->alpha * (1.0 - p->alpha); /* :334 */
            Jsq[3] += jl * jl;
            Jsq[4] += jo * jo;
            if (ch < 3 && craw[ch] > 0.0 && craw[ch] < 1.0) Jsq[5 + ch] += w * w; /* :291-294 */
        }
        for (int th = 0; th < 8; ++th) sink(sctx, p->index, th, Jsq[th]);
    }
}

typedef struct {
    double* H;
} acc_ctx_t;
static void sink_acc(void* ctx, uint32_t i, int th, double v) {
    ((acc_ctx_t*)ctx)->H[8 * (uint64_t)i + th] += v;
}

typedef struct {
    const double* Hp;
    double lambda;
    double sum;
} gain_ctx_t;
static void sink_gain(void* ctx, uint32_t i, int th, double v) {
    gain_ctx_t* g = (gain_ctx_t*)ctx;
    g->sum += v / (g->Hp[8 * (uint64_t)i + th] + g->lambda);
}

static int fisher_view(const orc_map* map, const orc_camera* cam, const orc_pose* pose,
                       const orc_options* opt, fisher_sink sink, void* sctx) {
    view_t s;
    if (view_prepare(&s, map, cam, pose, opt)) {
        view_free(&s);
        return -1;
    }
    const uint64_t cap = s.v + 1;
    uint32_t* ids = (uint32_t*)malloc(cap * sizeof(uint32_t));
    double* fs = (double*)malloc(cap * sizeof(double));
    double* ts = (double*)malloc(cap * sizeof(double));
    unsigned char* cl = (unsigned char*)malloc(cap);
    const int ts_ = opt->tile_size, W = cam->width, H = cam->height;
    for (int ty = 0; ty < s.tiles_y; ++ty)
        for (int tx = 0; tx < s.tiles_x; ++tx) {
            const uint64_t tile = (uint64_t)ty * s.tiles_x + tx;
            const uint32_t b0 = s.offsets[tile], b1 = s.offsets[tile + 1];
            if (b0 == b1) continue;
            const int y1 = H < (ty + 1) * ts_ ? H : (ty + 1) * ts_;
            const int x1 = W < (tx + 1) * ts_ ? W : (tx + 1) * ts_;
            for (int y = ty * ts_; y < y1; ++y)
                for (int x = tx * ts_; x < x1; ++x)
                    fisher_pixel(&s, map, cam, pose, opt, b0, b1, x, y, sink, sctx, ids, fs, ts, cl);
        }
    free(ids);
    free(fs);
    free(ts);
    free(cl);
    view_free(&s);
    return 0;
}

int orc_fisher_accumulate(const orc_map* map, const orc_camera* cam, uint64_t n_views,
                          const orc_pose* poses, const orc_options* opt, double* H) {
    if (map->log_scales && map->quats) return -1; /* isotropic chain only */
    acc_ctx_t a = {H};
    for (uint64_t v = 0; v < n_views; ++v)
        if (fisher_view(map, cam, &poses[v], opt, sink_acc, &a)) return -1;
    return 0;
}

int orc_fisher_gain(const orc_map* map, const orc_camera* cam, uint64_t n_views,
                    const orc_pose* poses, const orc_options* opt, const double* H_prior,
                    double lambda, double* gain) {
    if (map->log_scales && map->quats) return -1; /* isotropic chain only */
    for (uint64_t v = 0; v < n_views; ++v) {
        gain_ctx_t g = {H_prior, lambda, 0.0};
        if (fisher_view(map, cam, &poses[v], opt, sink_gain, &g)) return -1;
        gain[v] = g.sum;
    }
    return 0;
}

/* ------------------------------------------------------------------ ExplorationMap */

enum { ORC_UNKNOWN = 0, ORC_FREE = 1, ORC_OCCUPIED = 2 };
#define ORC_PI 3.14159265358979323846 /* glibc M_PI */

int orc_emap_init(orc_emap* e, const double bmin[3], const double bmax[3], double voxel) {
    memset(e, 0, sizeof(*e));
    if (voxel <= 0) return -1; /* explorer.cpp:13 */
    e->voxel = voxel;
    e->nvox = 1;
    for (int a = 0; a < 3; ++a) {
        e->origin[a] = bmin[a];
        int d = to_int_x86(ceil((bmax[a] - bmin[a]) / voxel)); /* :14-17 */
        e->dims[a] = d < 1 ? 1 : d;                             /* :18 cwiseMax */
        e->nvox *= (uint64_t)e->dims[a];
    }
    e->grid = (uint8_t*)calloc(e->nvox, 1);
    e->log = (int32_t*)malloc(e->nvox * sizeof(int32_t));
    if (!e->grid || !e->log) {
        orc_emap_free(e);
        return -1;
    }
    return 0;
}

void orc_emap_free(orc_emap* e) {
    free(e->grid);
    free(e->log);
    e->grid = NULL;
    e->log = NULL;
}

static int emap_in_grid(const orc_emap* e, int ix, int iy, int iz) { /* explorer.hpp:28-30 */
    return ix >= 0 && iy >= 0 && iz >= 0 && ix < e->dims[0] && iy < e->dims[1] && iz < e->dims[2];
}

static int emap_linear(const orc_emap* e, int ix, int iy, int iz) { /* explorer.hpp:25-27 */
    return (iz * e->dims[1] + iy) * e->dims[0] + ix;
}

static int emap_voxel_at(const orc_emap* e, const double p[3]) { /* explorer.cpp:22-29 */
    int ix = to_int_x86(floor((p[0] - e->origin[0]) / e->voxel));
    int iy = to_int_x86(floor((p[1] - e->origin[1]) / e->voxel));
    int iz = to_int_x86(floor((p[2] - e->origin[2]) / e->voxel));
    if (!emap_in_grid(e, ix, iy, iz)) return -1;
    return emap_linear(e, ix, iy, iz);
}

static void emap_mark_free(orc_emap* e, int id) { /* explorer.cpp:38-43 */
    if (e->grid[id] != ORC_UNKNOWN) return;
    e->grid[id] = ORC_FREE;
    ++e->free_count;
    e->log[e->log_n++] = id;
}

static void emap_mark_occupied(orc_emap* e, int id) { /* explorer.cpp:45-51 */
    if (e->grid[id] == ORC_OCCUPIED) return;
    if (e->grid[id] == ORC_FREE) --e->free_count;
    e->grid[id] = ORC_OCCUPIED;
    ++e->occupied_count;
}

uint64_t orc_emap_integrate(orc_emap* e, const orc_camera* cam, const orc_pose* pose,
                            const float* depth, int stride) {
    const uint64_t before = e->log_n;
    for (int y = 0; y < cam->height; y += stride) {
        for (int x = 0; x < cam->width; x += stride) {
            float d = depth[(size_t)y * cam->width + x];
            if (d <= 0) continue; /* :58 */
            const double dd = (double)d;
            /* end = R * (pixel_ray(x, y) * d) + t   camera.hpp:45-47, geometry.hpp:22 */
            const double c[3] = {(x + 0.5 - cam->cx) / cam->fx * dd, (y + 0.5 - cam->cy) / cam->fy * dd,
                                 1.0 * dd};
            double start[3], end[3], dir[3];
            int idx[3], step[3];
            double t_max[3], t_delta[3];
            for (int i = 0; i < 3; ++i) {
                start[i] = pose->t[i];
                end[i] = (pose->R[3 * i] * c[0] + (pose->R[3 * i + 1] * c[1] + pose->R[3 * i + 2] * c[2])) +
                         pose->t[i];
            }
            for (int a = 0; a < 3; ++a) idx[a] = to_int_x86(floor((start[a] - e->origin[a]) / e->voxel));
            for (int a = 0; a < 3; ++a) dir[a] = end[a] - start[a];
            const double len = sqrt(dir[0] * dir[0] + (dir[1] * dir[1] + dir[2] * dir[2]));
            if (len < 1e-12) continue; /* :68 */
            for (int a = 0; a < 3; ++a) dir[a] = dir[a] / len;
            const double q[3] = {end[0] - dir[0] * 1e-6, end[1] - dir[1] * 1e-6, end[2] - dir[2] * 1e-6};
            const int hit = emap_voxel_at(e, q); /* :72 */
            for (int a = 0; a < 3; ++a) { /* :77-89 */
                if (fabs(dir[a]) < 1e-12) {
                    step[a] = 0;
                    t_max[a] = 1e300;
                    t_delta[a] = 1e300;
                } else {
                    step[a] = dir[a] > 0 ? 1 : -1;
                    double boundary = e->origin[a] + (idx[a] + (dir[a] > 0 ? 1.0 : 0.0)) * e->voxel;
                    t_max[a] = (boundary - start[a]) / dir[a];
                    t_delta[a] = e->voxel / fabs(dir[a]);
                }
            }
            double t = 0.0;
            int guard = e->dims[0] + e->dims[1] + e->dims[2] + 4;
            while (guard-- > 0 && t <= len) { /* :93-104 */
                if (!emap_in_grid(e, idx[0], idx[1], idx[2])) break;
                int id = emap_linear(e, idx[0], idx[1], idx[2]);
                if (id == hit) break;
                emap_mark_free(e, id);
                int axis = 0;
                if (t_max[1] < t_max[axis]) axis = 1;
                if (t_max[2] < t_max[axis]) axis = 2;
                t = t_max[axis];
                t_max[axis] += t_delta[axis];
                idx[axis] += step[axis];
            }
            if (hit >= 0) emap_mark_occupied(e, hit); /* :105 */
        }
    }
    return e->log_n - before;
}

void orc_emap_seed(orc_emap* e, const double bmin[3], const double bmax[3], int occupied) {
    for (uint64_t i = 0; i < e->nvox; ++i) { /* explorer.cpp:124-132 */
        const int id = (int)i;
        const int ix = id % e->dims[0], iy = (id / e->dims[0]) % e->dims[1],
                  iz = id / (e->dims[0] * e->dims[1]); /* voxel_center, :31-36 */
        const double p[3] = {e->origin[0] + e->voxel * (ix + 0.5), e->origin[1] + e->voxel * (iy + 0.5),
                             e->origin[2] + e->voxel * (iz + 0.5)};
        int in = 1;
        for (int a = 0; a < 3; ++a) in = in && p[a] >= bmin[a] && p[a] <= bmax[a];
        if (!in) continue;
        if (occupied) emap_mark_occupied(e, id);
        else emap_mark_free(e, id);
    }
}

void orc_emap_reseed(orc_emap* e) { /* explorer.cpp:118-122 */
    e->log_n = 0;
    for (uint64_t i = 0; i < e->nvox; ++i)
        if (e->grid[i] == ORC_FREE) e->log[e->log_n++] = (int32_t)i;
}

void orc_fibonacci_directions(int count, double max_elev_deg, double* out3) {
    const double golden_angle = ORC_PI * (3.0 - sqrt(5.0));
    const double s_max = sin(max_elev_deg * ORC_PI / 180.0); /* deg_to_rad, geometry.hpp:86 */
    for (int j = 0; j < count; ++j) {
        double s = count == 1 ? 0.0 : s_max * (1.0 - (2.0 * j + 1.0) / count);
        double r = sqrt(fmax(0.0, 1.0 - s * s));
        double az = golden_angle * j;
        out3[3 * j + 0] = r * cos(az);
        out3[3 * j + 1] = s;
        out3[3 * j + 2] = r * sin(az);
    }
}

uint64_t orc_sample_candidates(orc_emap* e, double v1, int v2, const double* heights, int nh,
                               double* out6, uint64_t capacity) {
    const uint64_t n_fresh = e->log_n; /* take_changelog (:159) */
    e->log_n = 0;
    if (n_fresh == 0) return 0;
    uint8_t* fresh = (uint8_t*)calloc(e->nvox, 1);
    double* dirs = (double*)malloc(sizeof(double) * 3 * (size_t)(v2 > 0 ? v2 : 1));
    if (!fresh || !dirs) {
        free(fresh);
        free(dirs);
        return 0;
    }
    for (uint64_t i = 0; i < n_fresh; ++i) fresh[e->log[i]] = 1;
    orc_fibonacci_directions(v2, 45.0, dirs);
    double top[3];
    for (int a = 0; a < 3; ++a) top[a] = e->origin[a] + (double)e->dims[a] * e->voxel;
    uint64_t n = 0;
    for (int hi = 0; hi < nh; ++hi)
        for (double x = e->origin[0]; x <= top[0] + 1e-9; x += v1)
            for (double z = e->origin[2]; z <= top[2] + 1e-9; z += v1) {
                const double p[3] = {x, heights[hi], z};
                int id = emap_voxel_at(e, p);
                if (id < 0 || e->grid[id] != ORC_FREE || !fresh[id]) continue;
                for (int d = 0; d < v2; ++d, ++n) {
                    if (n >= capacity) continue;
                    for (int a = 0; a < 3; ++a) {
                        out6[6 * n + a] = p[a];
                        out6[6 * n + 3 + a] = dirs[3 * d + a];
                    }
                }
            }
    free(fresh);
    free(dirs);
    return n;
}
