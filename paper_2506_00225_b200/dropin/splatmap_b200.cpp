// Drop-in replacement for the reference's GPU-served entry points.
//
// Link this translation unit (plus libsgm_b200.so) into a build of the reference
// library in place of these three definitions:
//   RenderOutput render(...)                proj/src/splat_render.cpp:170-328
//   std::vector<double> render_entropy(...) proj/src/splat_render.cpp:378-390
//   void refresh_candidate_scores(...)      proj/src/explorer.cpp:186-205
// Signatures, argument meaning, outputs (RenderOutput layout, projections, contributor
// lists) and error style (exceptions) are the reference's. Everything else of the
// reference (GaussianMap, combine_scores, render_reference, clipped_entropy, ...) is
// untouched. INTEGRATION.md shows the build wiring; tests/test_dropin.py links the
// reference's own test files against this TU and runs them on the GPU.
//
// Devices: SGM_DEVICES ("0,1,2,3"), else SGM_DEVICE (one device), else every visible GPU;
// one sgm_multi per process. refresh_candidate_scores shards its candidates over all of
// them (sgm_multi: the map uploaded once, replicated device to device over NVLink, one host
// thread per GPU); render / render_entropy run on the first. The map is uploaded on every
// call: GaussianMap is mutable through its spans, so no stale snapshot is ever rendered
// (refresh_candidate_scores uploads once for all its candidates).
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgm.h"
#include "splatmap/explorer.hpp"
#include "splatmap/splat_render.hpp"

namespace splatmap {
namespace {

std::mutex g_mu;  // the C ABI serialises calls per ctx; the reference API is free to call from threads

sgm_multi* multi() {
    static sgm_multi* m = [] {
        std::vector<int32_t> devs;
        if (const char* list = std::getenv("SGM_DEVICES")) {
            for (const char* p = list; *p;) {
                char* end = nullptr;
                const long d = std::strtol(p, &end, 10);
                if (end == p) break;
                devs.push_back(static_cast<int32_t>(d));
                p = (*end == ',') ? end + 1 : end;
            }
        } else if (const char* one = std::getenv("SGM_DEVICE")) {
            devs.push_back(static_cast<int32_t>(std::atoi(one)));
        }
        sgm_multi* h = nullptr;
        const int rc = devs.empty() ? sgm_multi_create(0, nullptr, &h)
                                    : sgm_multi_create(static_cast<int32_t>(devs.size()), devs.data(), &h);
        if (rc != SGM_OK) throw std::runtime_error(std::string("sgm: ") + sgm_last_error(nullptr));
        return h;
    }();
    return m;
}

sgm_ctx* ctx() { return sgm_multi_ctx(multi(), 0); }

void check(int rc) {
    if (rc == SGM_OK) return;
    const std::string msg = std::string("sgm: ") + sgm_last_error(ctx());
    if (rc == SGM_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

struct MapHandle {
    sgm_map* m = nullptr;
    // async upload: the spans stay untouched until the call that made this handle returns
    explicit MapHandle(const GaussianMap& map) {
        check(sgm_map_upload_async(ctx(), map.size(), map.k(), map.num_classes(), map.centers().data(),
                             map.log_radii().data(), map.opacity_logits().data(),
                             map.colors().data(), map.sem_indices().data(), map.sem_probs().data(),
                             &m));
    }
    ~MapHandle() { sgm_map_release(ctx(), m); }
    MapHandle(const MapHandle&) = delete;
    MapHandle& operator=(const MapHandle&) = delete;
};

sgm_camera cam_of(const CameraModel& c) {
    return sgm_camera{c.width, c.height, c.fx, c.fy, c.cx, c.cy};
}

sgm_pose pose_of(const Pose& p) {
    sgm_pose q;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) q.R[3 * i + j] = p.R(i, j);
    for (int i = 0; i < 3; ++i) q.t[i] = p.t[i];
    return q;
}

sgm_options opt_of(const RenderOptions& o) {
    return sgm_options{o.early_exit ? 1 : 0, o.transmittance_eps, o.z_near, o.truncation_sigmas,
                       o.tile_size};
}

}  // namespace

RenderOutput render(const GaussianMap& map, const CameraModel& camera, const Pose& pose,
                    const RenderChannels& channels, const RenderOptions& options,
                    const DenseSemantics* dense) {
    if (dense)  // dead in shipped code; the sparse path is the product
        throw std::invalid_argument("render: DenseSemantics is not served by the B200 path");
    std::lock_guard<std::mutex> lock(g_mu);
    RenderOutput out;
    out.width = camera.width;
    out.height = camera.height;
    out.proj_fx = camera.fx;
    out.proj_fy = camera.fy;
    out.proj_cx = camera.cx;
    out.proj_cy = camera.cy;
    const size_t px = static_cast<size_t>(camera.width) * camera.height;
    out.silhouette.assign(px, 0.0);
    if (channels.color) out.color.assign(px * 3, 0.0);
    if (channels.depth) out.depth.assign(px, 0.0);
    if (channels.semantics) {
        out.channels = map.channels();
        out.sem.assign(px * map.channels(), 0.0);
    }
    MapHandle h(map);
    const sgm_camera cam = cam_of(camera);
    const sgm_pose ps = pose_of(pose);
    const sgm_options op = opt_of(options);
    const uint32_t flags = (channels.color ? SGM_COLOR : 0u) | (channels.depth ? SGM_DEPTH : 0u) |
                           (channels.semantics ? SGM_SEMANTICS : 0u) |
                           (channels.retain_contributors ? SGM_RETAIN_CONTRIBUTORS : 0u);
    uint64_t nproj = 0;
    check(sgm_render(ctx(), h.m, &cam, &ps, flags, &op, channels.color ? out.color.data() : nullptr,
                     channels.depth ? out.depth.data() : nullptr, out.silhouette.data(),
                     channels.semantics ? out.sem.data() : nullptr, &nproj));
    std::vector<sgm_projection> pr(nproj);
    if (nproj) check(sgm_last_projections(ctx(), pr.data(), nproj));
    out.projections.resize(nproj);
    for (uint64_t i = 0; i < nproj; ++i) {
        SplatProjection& s = out.projections[i];
        s.mx = pr[i].mx;
        s.my = pr[i].my;
        s.rad_px = pr[i].rad_px;
        s.z = pr[i].z;
        s.alpha = pr[i].alpha;
        s.index = pr[i].index;
    }
    if (channels.retain_contributors) {
        uint64_t n = 0;
        check(sgm_last_contributors(ctx(), nullptr, nullptr, 0, &n));
        out.contrib_offset.assign(px + 1, 0);
        out.contrib.assign(n, 0);
        check(sgm_last_contributors(ctx(), out.contrib_offset.data(), out.contrib.data(), n, &n));
    }
    return out;
}

std::vector<double> render_entropy(const GaussianMap& map, const CameraModel& camera,
                                   const Pose& pose, const RenderOptions& options) {
    std::lock_guard<std::mutex> lock(g_mu);
    std::vector<double> entropy(static_cast<size_t>(camera.width) * camera.height);
    MapHandle h(map);
    const sgm_camera cam = cam_of(camera);
    const sgm_pose ps = pose_of(pose);
    const sgm_options op = opt_of(options);
    check(sgm_render_entropy(ctx(), h.m, &cam, &ps, &op, entropy.data()));
    return entropy;
}

void refresh_candidate_scores(std::span<CandidatePose> candidates, const GaussianMap& map,
                              const CameraModel& scoring_camera) {
    std::vector<CandidatePose*> active;
    for (auto& c : candidates)
        if (c.state == CandidatePose::State::Active) active.push_back(&c);
    if (active.empty()) return;
    std::lock_guard<std::mutex> lock(g_mu);
    std::vector<sgm_candidate> cs(active.size());
    for (size_t i = 0; i < active.size(); ++i)
        for (int a = 0; a < 3; ++a) {
            cs[i].position[a] = active[i]->position[a];
            cs[i].direction[a] = active[i]->direction[a];
        }
    auto mcheck = [](int rc) {
        if (rc == SGM_OK) return;
        const std::string msg = std::string("sgm: ") + sgm_multi_last_error(multi());
        if (rc == SGM_ERR_INVALID) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    };
    sgm_multi_map* mm = nullptr;
    mcheck(sgm_multi_map_upload(multi(), map.size(), map.k(), map.num_classes(),
                                map.centers().data(), map.log_radii().data(),
                                map.opacity_logits().data(), map.colors().data(),
                                map.sem_indices().data(), map.sem_probs().data(), &mm));
    struct Release {
        sgm_multi_map* m;
        ~Release() { sgm_multi_map_release(multi(), m); }
    } release{mm};
    const sgm_camera cam = cam_of(scoring_camera);
    const RenderOptions defaults;  // the reference scores with default options (explorer.cpp:194)
    const sgm_options op = opt_of(defaults);
    std::vector<double> nm(active.size()), es(active.size());
    // candidates sharded over every device of the process
    mcheck(sgm_multi_score_candidates(multi(), mm, &cam, active.size(), cs.data(), &op, nm.data(),
                                      es.data()));
    for (size_t i = 0; i < active.size(); ++i) {
        active[i]->n_missing = nm[i];
        active[i]->entropy_sum = es[i];
    }
}

}  // namespace splatmap
