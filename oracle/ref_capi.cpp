// C entry points over the REFERENCE's own render/scoring code, compiled
// unmodified from /root/reference/proj/src (see oracle/Makefile). TEST
// INFRASTRUCTURE ONLY: used by tests/ (as the checker), by tests/golden/make_golden.py
// (fixture generation), and by bench.py's reference arm / cpu_baseline. The
// product (paper_2506_00225_b200) never links this.
//
// Wrapped reference interfaces:
//   render / render_reference / render_entropy / clipped_entropy
//       proj/include/splatmap/splat_render.hpp:78-95
//   refresh_candidate_scores / combine_scores   proj/include/splatmap/explorer.hpp:114-121
//   look_at                                      proj/include/splatmap/geometry.hpp:44-56
//   testutil::random_splat_map                   proj/tests/test_helpers.hpp:46-67
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "splatmap/explorer.hpp"
#include "splatmap/gaussian_map.hpp"
#include "splatmap/splat_render.hpp"
#include "test_helpers.hpp"

using namespace splatmap;

namespace {

struct RefMap {
    GaussianMap map;
    RefMap(int k, int c) : map(k, c) {}
};

CameraModel make_cam(const int32_t wh[2], const double intr[4]) {
    CameraModel c;
    c.width = wh[0];
    c.height = wh[1];
    c.fx = intr[0];
    c.fy = intr[1];
    c.cx = intr[2];
    c.cy = intr[3];
    return c;
}

Pose make_pose(const double R_rowmajor[9], const double t[3]) {
    Pose p;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) p.R(i, j) = R_rowmajor[3 * i + j];
    p.t = Vec3(t[0], t[1], t[2]);
    return p;
}

RenderOptions make_opts(const double o[5]) {
    // o = {early_exit, transmittance_eps, z_near, truncation_sigmas, tile_size}
    RenderOptions r;
    r.early_exit = o[0] != 0.0;
    r.transmittance_eps = o[1];
    r.z_near = o[2];
    r.truncation_sigmas = o[3];
    r.tile_size = static_cast<int>(o[4]);
    return r;
}

void copy_out(const RenderOutput& out, double* color, double* depth, double* sil, double* sem,
              double* proj6, uint64_t* n_proj, uint32_t* contrib_offset, uint32_t* contrib,
              uint64_t contrib_cap, uint64_t* n_contrib) {
    if (color && !out.color.empty()) std::memcpy(color, out.color.data(), out.color.size() * 8);
    if (depth && !out.depth.empty()) std::memcpy(depth, out.depth.data(), out.depth.size() * 8);
    if (sil) std::memcpy(sil, out.silhouette.data(), out.silhouette.size() * 8);
    if (sem && !out.sem.empty()) std::memcpy(sem, out.sem.data(), out.sem.size() * 8);
    if (n_proj) *n_proj = out.projections.size();
    if (proj6) {
        for (size_t i = 0; i < out.projections.size(); ++i) {
            const SplatProjection& p = out.projections[i];
            double* r = proj6 + 6 * i;
            r[0] = p.mx;
            r[1] = p.my;
            r[2] = p.rad_px;
            r[3] = p.z;
            r[4] = p.alpha;
            r[5] = static_cast<double>(p.index);
        }
    }
    if (n_contrib) *n_contrib = out.contrib.size();
    if (contrib_offset && !out.contrib_offset.empty())
        std::memcpy(contrib_offset, out.contrib_offset.data(), out.contrib_offset.size() * 4);
    if (contrib && !out.contrib.empty())
        std::memcpy(contrib, out.contrib.data(), std::min<uint64_t>(contrib_cap, out.contrib.size()) * 4);
}

}  // namespace

extern "C" {

void* ref_map_create(uint64_t n, int k, int num_classes, const double* centers,
                     const double* log_radii, const double* logits, const double* colors,
                     const uint16_t* sem_idx, const double* sem_probs) {
    auto* m = new RefMap(k, num_classes);
    for (uint64_t i = 0; i < n; ++i) {
        SemanticGaussian g;
        g.center = Vec3(centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]);
        g.log_radius = log_radii[i];
        g.opacity_logit = logits[i];
        g.color = Vec3(colors[3 * i], colors[3 * i + 1], colors[3 * i + 2]);
        g.sem.indices.assign(sem_idx + i * k, sem_idx + (i + 1) * k);
        g.sem.probs.assign(sem_probs + i * k, sem_probs + (i + 1) * k);
        m->map.add(g);
    }
    return m;
}

void ref_map_destroy(void* m) { delete static_cast<RefMap*>(m); }

// GaussianMap::load (SGMP v1, proj/src/gaussian_map.cpp:163-189).
void* ref_map_load(const char* path) {
    auto* m = new RefMap(1, 1);
    m->map = GaussianMap::load(path);
    return m;
}
uint64_t ref_map_size(void* m) { return static_cast<RefMap*>(m)->map.size(); }

// Which: 0 = render (tiled, production), 1 = render_reference (untiled oracle).
int ref_render(void* m, int which, const int32_t wh[2], const double intr[4], const double R[9],
               const double t[3], uint32_t channels, const double opts[5], double* color,
               double* depth, double* sil, double* sem, double* proj6, uint64_t* n_proj,
               uint32_t* contrib_offset, uint32_t* contrib, uint64_t contrib_cap,
               uint64_t* n_contrib) {
    const GaussianMap& map = static_cast<RefMap*>(m)->map;
    RenderChannels ch;
    ch.color = channels & 1u;
    ch.depth = channels & 2u;
    ch.semantics = channels & 4u;
    ch.retain_contributors = channels & 8u;
    RenderOutput out = which == 0 ? render(map, make_cam(wh, intr), make_pose(R, t), ch, make_opts(opts))
                                  : render_reference(map, make_cam(wh, intr), make_pose(R, t), ch);
    copy_out(out, color, depth, sil, sem, proj6, n_proj, contrib_offset, contrib, contrib_cap,
             n_contrib);
    return 0;
}

void ref_render_entropy(void* m, const int32_t wh[2], const double intr[4], const double R[9],
                        const double t[3], const double opts[5], double* out) {
    auto h = render_entropy(static_cast<RefMap*>(m)->map, make_cam(wh, intr), make_pose(R, t),
                            make_opts(opts));
    std::memcpy(out, h.data(), h.size() * 8);
}

double ref_clipped_entropy(const double* p, uint64_t n) {
    return clipped_entropy(std::span<const double>(p, n));
}

// refresh_candidate_scores over candidates (position, direction), split into
// `threads` disjoint contiguous spans on the shared const map.
void ref_refresh_scores(void* m, const int32_t wh[2], const double intr[4], uint64_t n,
                        const double* pos3, const double* dir3, int threads, double* n_missing,
                        double* entropy_sum) {
    const GaussianMap& map = static_cast<RefMap*>(m)->map;
    CameraModel cam = make_cam(wh, intr);
    std::vector<CandidatePose> cs(n);
    for (uint64_t i = 0; i < n; ++i) {
        cs[i].position = Vec3(pos3[3 * i], pos3[3 * i + 1], pos3[3 * i + 2]);
        cs[i].direction = Vec3(dir3[3 * i], dir3[3 * i + 1], dir3[3 * i + 2]);
        cs[i].id = static_cast<int>(i);
    }
    threads = std::max(1, std::min<int>(threads, static_cast<int>(n)));
    if (threads == 1) {
        refresh_candidate_scores(cs, map, cam);
    } else {
        std::vector<std::thread> pool;
        const uint64_t per = (n + threads - 1) / threads;
        for (int w = 0; w < threads; ++w) {
            uint64_t a = w * per, b = std::min<uint64_t>(n, a + per);
            if (a >= b) break;
            pool.emplace_back([&, a, b] {
                refresh_candidate_scores(std::span<CandidatePose>(cs.data() + a, b - a), map, cam);
            });
        }
        for (auto& th : pool) th.join();
    }
    for (uint64_t i = 0; i < n; ++i) {
        n_missing[i] = cs[i].n_missing;
        entropy_sum[i] = cs[i].entropy_sum;
    }
}

int ref_combine_scores(uint64_t n, const double* n_missing, const double* entropy_sum,
                       const double* pos3, const double cur[3], double* i_geo, double* i_sem,
                       double* i_total) {
    std::vector<CandidatePose> cs(n);
    for (uint64_t i = 0; i < n; ++i) {
        cs[i].position = Vec3(pos3[3 * i], pos3[3 * i + 1], pos3[3 * i + 2]);
        cs[i].n_missing = n_missing[i];
        cs[i].entropy_sum = entropy_sum[i];
    }
    bool any = combine_scores(cs, Vec3(cur[0], cur[1], cur[2]));
    for (uint64_t i = 0; i < n; ++i) {
        i_geo[i] = cs[i].i_geo;
        i_sem[i] = cs[i].i_sem;
        i_total[i] = cs[i].i_total;
    }
    return any ? 1 : 0;
}

// CandidatePose::camera_pose() = look_at(pos, pos + dir) (explorer.hpp:105).
void ref_candidate_pose(const double pos[3], const double dir[3], double R[9], double t[3]) {
    CandidatePose c;
    c.position = Vec3(pos[0], pos[1], pos[2]);
    c.direction = Vec3(dir[0], dir[1], dir[2]);
    Pose p = c.camera_pose();
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) R[3 * i + j] = p.R(i, j);
    for (int i = 0; i < 3; ++i) t[i] = p.t[i];
}

void ref_look_at(const double pos[3], const double target[3], double R[9], double t[3]) {
    Pose p = look_at(Vec3(pos[0], pos[1], pos[2]), Vec3(target[0], target[1], target[2]));
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) R[3 * i + j] = p.R(i, j);
    for (int i = 0; i < 3; ++i) t[i] = p.t[i];
}

// testutil::random_splat_map (proj/tests/test_helpers.hpp:46-67). prm = {num_splats,
// num_classes, k, min_prob, alpha_logit_min, alpha_logit_max, rad_px_min, rad_px_max}.
// Output arrays must hold num_splats (times 3 / k) entries; k_out receives k.
void ref_random_splat_map(uint64_t seed, const int32_t wh[2], const double intr[4],
                          const double R[9], const double t[3], const double prm[8],
                          double* centers, double* log_radii, double* logits, double* colors,
                          uint16_t* sem_idx, double* sem_probs, int* k_out) {
    testutil::SplatSceneParams p;
    p.num_splats = static_cast<int>(prm[0]);
    p.num_classes = static_cast<int>(prm[1]);
    p.k = static_cast<int>(prm[2]);
    p.min_prob = prm[3];
    p.alpha_logit_min = prm[4];
    p.alpha_logit_max = prm[5];
    p.rad_px_min = prm[6];
    p.rad_px_max = prm[7];
    GaussianMap map = testutil::random_splat_map(seed, make_cam(wh, intr), make_pose(R, t), p);
    const int k = map.k();
    *k_out = k;
    std::memcpy(centers, map.centers().data(), map.size() * 24);
    std::memcpy(log_radii, map.log_radii().data(), map.size() * 8);
    std::memcpy(logits, map.opacity_logits().data(), map.size() * 8);
    std::memcpy(colors, map.colors().data(), map.size() * 24);
    std::memcpy(sem_idx, map.sem_indices().data(), map.size() * k * 2);
    std::memcpy(sem_probs, map.sem_probs().data(), map.size() * k * 8);
}

// Camera intrinsics of CameraModel::from_fov (camera.hpp:18-32): out = {W,H,fx,fy,cx,cy}.
void ref_camera_from_fov(int w, int h, double vfov, double hfov, double out[6]) {
    CameraModel c = CameraModel::from_fov(w, h, vfov, hfov);
    out[0] = c.width;
    out[1] = c.height;
    out[2] = c.fx;
    out[3] = c.fy;
    out[4] = c.cx;
    out[5] = c.cy;
}

}  // extern "C"

// ---- losses + backward (proj/src/losses.cpp) over the reference's own render ----
#include "splatmap/losses.hpp"

extern "C" {

// weights = {lambda_hd, lambda_cos, mask_k, use_hd, use_cos, use_kl, kl_clip_norm};
// report  = {photometric, depth, semantic, photometric_px, depth_px, semantic_px, uncovered_px}
// grads: center 3N, log_radius N, opacity_logit N, color 3N, sem kN. Returns 0, or 1 when the
// reference throws (message copied to err).
int ref_backward(void* m, const int32_t wh[2], const double intr[4], const double R[9],
                 const double t[3], const double opts[5], int num_classes, const float* rgb,
                 const float* depth, const float* sem, const double weights[7],
                 int include_mapping, int include_semantic, double* report, double* g_center,
                 double* g_logr, double* g_logit, double* g_color, double* g_sem, char* err,
                 int err_cap) {
    const GaussianMap& map = static_cast<RefMap*>(m)->map;
    CameraModel cam = make_cam(wh, intr);
    Frame fr;
    fr.width = cam.width;
    fr.height = cam.height;
    fr.num_classes = num_classes;
    fr.pose = make_pose(R, t);
    fr.allocate();
    const size_t px = static_cast<size_t>(cam.width) * cam.height;
    std::memcpy(fr.rgb.data(), rgb, px * 3 * 4);
    std::memcpy(fr.depth.data(), depth, px * 4);
    std::memcpy(fr.sem.data(), sem, px * fr.channels() * 4);
    LossWeights w;
    w.lambda_hd = weights[0];
    w.lambda_cos = weights[1];
    w.mask_k = static_cast<int>(weights[2]);
    w.use_hd = weights[3] != 0.0;
    w.use_cos = weights[4] != 0.0;
    w.use_kl = weights[5] != 0.0;
    w.kl_clip_norm = weights[6];
    try {
        RenderOutput out = render(map, cam, fr.pose, RenderChannels::all(true), make_opts(opts));
        LossReport a = mapping_loss(out, fr);
        LossReport b = semantic_loss(out, fr, w);
        report[0] = a.photometric;
        report[1] = a.depth;
        report[2] = b.semantic;
        report[3] = static_cast<double>(a.photometric_px);
        report[4] = static_cast<double>(a.depth_px);
        report[5] = static_cast<double>(b.semantic_px);
        report[6] = static_cast<double>(b.uncovered_px);
        ParamGradients g = backward(out, fr, map, w, include_mapping != 0, include_semantic != 0);
        std::memcpy(g_center, g.center.data(), g.center.size() * 8);
        std::memcpy(g_logr, g.log_radius.data(), g.log_radius.size() * 8);
        std::memcpy(g_logit, g.opacity_logit.data(), g.opacity_logit.size() * 8);
        std::memcpy(g_color, g.color.data(), g.color.size() * 8);
        std::memcpy(g_sem, g.sem.data(), g.sem.size() * 8);
    } catch (const std::exception& e) {
        if (err && err_cap > 0) {
            std::strncpy(err, e.what(), err_cap - 1);
            err[err_cap - 1] = 0;
        }
        return 1;
    }
    return 0;
}

}  // extern "C"

// ---- ExplorationMap + candidate sampling (proj/src/explorer.cpp:11-184) and the
// reference simulator's depth raycast (proj/src/scene_sim.cpp) for test frames ----
#include "splatmap/scene.hpp"
#include "splatmap/scene_sim.hpp"

extern "C" {

void* ref_emap_create(const double bmin[3], const double bmax[3], double voxel) {
    try {
        Aabb b;
        b.min = Vec3(bmin[0], bmin[1], bmin[2]);
        b.max = Vec3(bmax[0], bmax[1], bmax[2]);
        return new ExplorationMap(b, voxel);
    } catch (...) {
        return nullptr;
    }
}

void ref_emap_destroy(void* h) { delete static_cast<ExplorationMap*>(h); }

// info = {free_count, occupied_count, changelog_size, voxel_count}; dims[3]; origin[3]
void ref_emap_info(void* h, uint64_t info[4], int32_t dims[3], double origin[3]) {
    auto* e = static_cast<ExplorationMap*>(h);
    info[0] = e->free_count();
    info[1] = e->occupied_count();
    info[2] = e->changelog_size();
    info[3] = e->voxel_count();
    for (int a = 0; a < 3; ++a) {
        dims[a] = e->dims()[a];
        origin[a] = e->origin()[a];
    }
}

uint64_t ref_emap_integrate(void* h, const int32_t wh[2], const double intr[4], const double R[9],
                            const double t[3], const float* depth, int stride) {
    Frame f;
    f.width = wh[0];
    f.height = wh[1];
    f.pose = make_pose(R, t);
    f.depth.assign(depth, depth + static_cast<size_t>(wh[0]) * wh[1]);
    return static_cast<ExplorationMap*>(h)->integrate_frame(f, make_cam(wh, intr), stride);
}

void ref_emap_grid(void* h, uint8_t* out) {
    auto g = static_cast<ExplorationMap*>(h)->grid();
    for (size_t i = 0; i < g.size(); ++i) out[i] = static_cast<uint8_t>(g[i]);
}

uint64_t ref_emap_take_changelog(void* h, int32_t* out) {
    std::vector<int> log = static_cast<ExplorationMap*>(h)->take_changelog();
    std::memcpy(out, log.data(), log.size() * 4);
    return log.size();
}

void ref_emap_reseed(void* h) { static_cast<ExplorationMap*>(h)->reseed_changelog_with_free(); }

void ref_emap_seed(void* h, const double bmin[3], const double bmax[3], int occupied) {
    Aabb b;
    b.min = Vec3(bmin[0], bmin[1], bmin[2]);
    b.max = Vec3(bmax[0], bmax[1], bmax[2]);
    auto* e = static_cast<ExplorationMap*>(h);
    if (occupied) e->seed_occupied_region(b);
    else e->seed_free_region(b);
}

// sample_candidates: out6 = {position, direction} per candidate (capacity entries).
uint64_t ref_sample_candidates(void* h, double v1, int v2, const double* heights, int nh,
                               double* out6, uint64_t capacity) {
    SamplingSchedule s;
    s.v1 = v1;
    s.v2 = v2;
    s.heights.assign(heights, heights + nh);
    auto c = sample_candidates(*static_cast<ExplorationMap*>(h), s);
    for (size_t i = 0; i < c.size() && i < capacity; ++i)
        for (int a = 0; a < 3; ++a) {
            out6[6 * i + a] = c[i].position[a];
            out6[6 * i + 3 + a] = c[i].direction[a];
        }
    return c.size();
}

void ref_fibonacci_directions(int count, double max_elev, double* out3) {
    auto d = fibonacci_directions(count, max_elev);
    for (size_t i = 0; i < d.size(); ++i)
        for (int a = 0; a < 3; ++a) out3[3 * i + a] = d[i][a];
}

// raycast_frame depth of a room (bounds) with axis-aligned boxes (min, max) and spheres
// (centre, radius): the reference simulator's own depth (scene_sim.hpp:31).
int ref_raycast_depth(const double bmin[3], const double bmax[3], int n_boxes, const double* boxes6,
                      int n_spheres, const double* spheres4, const int32_t wh[2],
                      const double intr[4], const double R[9], const double t[3], float* depth) {
    try {
        SceneSpec s;
        s.bounds.min = Vec3(bmin[0], bmin[1], bmin[2]);
        s.bounds.max = Vec3(bmax[0], bmax[1], bmax[2]);
        s.num_classes = 6;
        for (int i = 0; i < n_boxes; ++i) {
            ScenePrimitive p;
            p.kind = ScenePrimitive::Kind::Box;
            p.box_min = Vec3(boxes6[6 * i], boxes6[6 * i + 1], boxes6[6 * i + 2]);
            p.box_max = Vec3(boxes6[6 * i + 3], boxes6[6 * i + 4], boxes6[6 * i + 5]);
            p.class_id = 3;
            s.primitives.push_back(p);
        }
        for (int i = 0; i < n_spheres; ++i) {
            ScenePrimitive p;
            p.kind = ScenePrimitive::Kind::Sphere;
            p.center = Vec3(spheres4[4 * i], spheres4[4 * i + 1], spheres4[4 * i + 2]);
            p.radius = spheres4[4 * i + 3];
            p.class_id = 4;
            s.primitives.push_back(p);
        }
        s.validate();
        Frame f = raycast_frame(s, make_cam(wh, intr), make_pose(R, t));
        std::memcpy(depth, f.depth.data(), f.depth.size() * 4);
        return 0;
    } catch (...) {
        return 1;
    }
}

}  // extern "C"

// ---- optimize_map (proj/src/mapper.cpp:241-283) on the reference's own code ----
#include "splatmap/mapper.hpp"

extern "C" {

// frames: n_frames poses (R row-major 9 + t 3 = 12 doubles each) and planes (rgb px*3,
// depth px, sem px*(num_classes+1) floats each, concatenated per frame).
// adam = {lr_center, lr_radius, lr_opacity, lr_color, lr_sem, beta1, beta2, eps, eps_sem};
// cfg = {prune_every, prune_opacity, divergence_factor, divergence_window};
// weights as ref_backward. The map arrays are updated in place (sized for the input n);
// returns the final size, or -1 on a throw (message in err), and fills history (iters x 7).
int64_t ref_optimize_map(uint64_t n, int k, int num_classes, double* centers, double* log_radii,
                         double* logits, double* colors, uint16_t* sem_idx, double* sem_probs,
                         const int32_t wh[2], const double intr[4], int n_frames,
                         const double* poses12, const float* planes, const double adam[9],
                         const double cfg[4], const double weights[7], int iters, double* history,
                         int* n_history, char* err, int err_cap) {
    try {
        GaussianMap map(k, num_classes);
        for (uint64_t i = 0; i < n; ++i) {
            SemanticGaussian g;
            g.center = Vec3(centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]);
            g.log_radius = log_radii[i];
            g.opacity_logit = logits[i];
            g.color = Vec3(colors[3 * i], colors[3 * i + 1], colors[3 * i + 2]);
            g.sem.indices.assign(sem_idx + i * k, sem_idx + (i + 1) * k);
            g.sem.probs.assign(sem_probs + i * k, sem_probs + (i + 1) * k);
            map.add(g);
        }
        CameraModel cam = make_cam(wh, intr);
        const size_t px = static_cast<size_t>(wh[0]) * wh[1];
        const size_t C = static_cast<size_t>(num_classes) + 1;
        std::vector<Frame> fr(static_cast<size_t>(n_frames));
        std::vector<const Frame*> fp;
        for (int f = 0; f < n_frames; ++f) {
            Frame& F = fr[f];
            F.width = wh[0];
            F.height = wh[1];
            F.num_classes = num_classes;
            F.pose = make_pose(poses12 + 12 * f, poses12 + 12 * f + 9);
            const float* base = planes + static_cast<size_t>(f) * px * (4 + C);
            F.rgb.assign(base, base + 3 * px);
            F.depth.assign(base + 3 * px, base + 4 * px);
            F.sem.assign(base + 4 * px, base + 4 * px + C * px);
            fp.push_back(&F);
        }
        MapperConfig mc;
        mc.adam.lr_center = adam[0];
        mc.adam.lr_radius = adam[1];
        mc.adam.lr_opacity = adam[2];
        mc.adam.lr_color = adam[3];
        mc.adam.lr_sem = adam[4];
        mc.adam.beta1 = adam[5];
        mc.adam.beta2 = adam[6];
        mc.adam.eps = adam[7];
        mc.adam.eps_sem = adam[8];
        mc.prune_every = static_cast<int>(cfg[0]);
        mc.prune_opacity = cfg[1];
        mc.divergence_factor = cfg[2];
        mc.divergence_window = static_cast<int>(cfg[3]);
        mc.weights.lambda_hd = weights[0];
        mc.weights.lambda_cos = weights[1];
        mc.weights.mask_k = static_cast<int>(weights[2]);
        mc.weights.use_hd = weights[3] != 0.0;
        mc.weights.use_cos = weights[4] != 0.0;
        mc.weights.use_kl = weights[5] != 0.0;
        mc.weights.kl_clip_norm = weights[6];
        AdamState st;
        auto hist = optimize_map(map, st, fp, cam, mc, iters);
        *n_history = static_cast<int>(hist.size());
        for (size_t i = 0; i < hist.size(); ++i) {
            const LossReport& r = hist[i];
            double* h = history + 7 * i;
            h[0] = r.photometric;
            h[1] = r.depth;
            h[2] = r.semantic;
            h[3] = static_cast<double>(r.photometric_px);
            h[4] = static_cast<double>(r.depth_px);
            h[5] = static_cast<double>(r.semantic_px);
            h[6] = static_cast<double>(r.uncovered_px);
        }
        const size_t m = map.size();
        std::memcpy(centers, map.centers().data(), m * 24);
        std::memcpy(log_radii, map.log_radii().data(), m * 8);
        std::memcpy(logits, map.opacity_logits().data(), m * 8);
        std::memcpy(colors, map.colors().data(), m * 24);
        std::memcpy(sem_idx, map.sem_indices().data(), m * k * 2);
        std::memcpy(sem_probs, map.sem_probs().data(), m * k * 8);
        return static_cast<int64_t>(m);
    } catch (const std::exception& e) {
        if (err && err_cap > 0) {
            std::strncpy(err, e.what(), static_cast<size_t>(err_cap) - 1);
            err[err_cap - 1] = 0;
        }
        return -1;
    }
}

}  // extern "C"

// ---- semantic_metrics + photometric_metrics (proj/src/evaluator.cpp:93-297) over the
// reference's own render(map, camera, pose, RenderChannels::all()) of each frame ----
#include "splatmap/evaluator.hpp"

extern "C" {

// frames as ref_optimize_map (poses12, planes). summary = {miou, top1, top3, map, f1, psnr,
// depth_l1}; per_class rows {class_id, iou, ap, f1, gt_pixels} (capacity num_classes).
int ref_eval(void* m, const int32_t wh[2], const double intr[4], int num_classes, int n_frames,
             const double* poses12, const float* planes, double summary[7], double* per_view_miou,
             double* per_view_psnr, double* per_class, uint64_t* n_per_class, char* err,
             int err_cap) {
    try {
        const GaussianMap& map = static_cast<RefMap*>(m)->map;
        CameraModel cam = make_cam(wh, intr);
        const size_t px = static_cast<size_t>(wh[0]) * wh[1];
        const size_t C = static_cast<size_t>(num_classes) + 1;
        std::vector<Frame> fr(static_cast<size_t>(n_frames));
        std::vector<RenderOutput> rs;
        for (int f = 0; f < n_frames; ++f) {
            Frame& F = fr[f];
            F.width = wh[0];
            F.height = wh[1];
            F.num_classes = num_classes;
            F.pose = make_pose(poses12 + 12 * f, poses12 + 12 * f + 9);
            const float* base = planes + static_cast<size_t>(f) * px * (4 + C);
            F.rgb.assign(base, base + 3 * px);
            F.depth.assign(base + 3 * px, base + 4 * px);
            F.sem.assign(base + 4 * px, base + 4 * px + C * px);
            rs.push_back(render(map, cam, F.pose, RenderChannels::all()));
        }
        MetricReport sem = semantic_metrics(rs, fr);
        MetricReport pho = photometric_metrics(rs, fr);
        summary[0] = sem.miou_pct;
        summary[1] = sem.top1_pct;
        summary[2] = sem.top3_pct;
        summary[3] = sem.map_pct;
        summary[4] = sem.f1_pct;
        summary[5] = pho.psnr_db;
        summary[6] = pho.depth_l1_cm;
        for (size_t i = 0; i < sem.per_view_miou.size(); ++i) per_view_miou[i] = sem.per_view_miou[i];
        for (size_t i = 0; i < pho.per_view_psnr.size(); ++i) per_view_psnr[i] = pho.per_view_psnr[i];
        *n_per_class = sem.per_class.size();
        for (size_t i = 0; i < sem.per_class.size(); ++i) {
            const PerClassMetric& pc = sem.per_class[i];
            double* r = per_class + 5 * i;
            r[0] = pc.class_id;
            r[1] = pc.iou_pct;
            r[2] = pc.ap_pct;
            r[3] = pc.f1_pct;
            r[4] = static_cast<double>(pc.gt_pixels);
        }
        return 0;
    } catch (const std::exception& e) {
        if (err && err_cap > 0) {
            std::strncpy(err, e.what(), static_cast<size_t>(err_cap) - 1);
            err[err_cap - 1] = 0;
        }
        return 1;
    }
}

}  // extern "C"
