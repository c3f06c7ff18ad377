// C ABI (include/sgm.h), part 2: exploration map (f1), on-device optimize_map (f2) and
// evaluation on device planes (f3).
#include "sgm_ctx.h"

struct sgm_frame {
    int W = 0, H = 0, C = 0;
    PoseParams pose{};
    DevBuf planes;  // rgb px*3 | depth px | sem px*C (floats)
};

struct sgm_trainer {
    sgm_map map;       // render snapshot, re-derived after every step
    DevBuf P, M, V;    // parameters and Adam moments (backward_core gradient layout, NS = n)
    DevBuf sidx;       // sem_indices kN (reference order)
    DevBuf rows;       // creation-time row of each current Gaussian (u32)
    DevBuf keep, kept, sel_count, sel_tmp;
    uint64_t n = 0;
    int k = 0, num_classes = 0, dup = 0;
    int64_t t = 0;     // AdamState::step_count
};


namespace {


// (Re)allocates the render snapshot for the current n: class-sorted rows + permutation
// from the master indices, then the activations (k_derive).
void trainer_rebuild(sgm_ctx* ctx, sgm_trainer* tr) {
    cudaStream_t s = ctx->stream;
    const uint64_t n = tr->n;
    const int k = tr->k, C = tr->num_classes + 1, kpad = (k + 7) / 8 * 8;
    const size_t ns = std::max<uint64_t>(n, 1);
    sgm_map& m = tr->map;
    CK(m.geo.reserve(8 * 5 * ns));
    CK(m.color.reserve(8 * 4 * ns));
    CK(m.idx.reserve(2 * ns * kpad));
    CK(m.prob.reserve(8 * ns * kpad));
    CK(m.perm.reserve(2 * ns * kpad));
    const double* P = tr->P.as<double>();
    launch_sort_rows(tr->sidx.as<uint16_t>(), P + 8 * n, n, k, kpad, m.idx.as<uint16_t>(),
                     m.prob.as<double>(), m.perm.as<uint16_t>(), s);
    launch_derive(P, n, k, kpad, m.perm.as<uint16_t>(), m.geo.as<double>(), m.color.as<double>(),
                  m.prob.as<double>(), s);
    ctx->stats.kernel_launches += n ? 2 : 0;
    m.num_classes = tr->num_classes;
    DevMap& d = m.dev;
    d.n = n;
    d.k = k;
    d.kpad = kpad;
    d.C = C;
    const double* g = m.geo.as<double>();
    d.cx = g;
    d.cy = g + ns;
    d.cz = g + 2 * ns;
    d.rad = g + 3 * ns;
    d.alpha = g + 4 * ns;
    d.color4 = m.color.as<double>();
    d.sem_idx = m.idx.as<uint16_t>();
    d.sem_prob = m.prob.as<double>();
    d.sem_perm = m.perm.as<uint16_t>();
    d.dup_idx = tr->dup;
    m.groups = choose_groups(C, k);
    map_group_bounds(ctx, &m, s);
    m.rec_valid = false;
    if (ctx->last_map == &m) ctx->last_valid = false;
}

// GaussianMap::prune_by_opacity + AdamState::compact (gaussian_map.cpp:97-124, mapper.cpp:53-69).
void trainer_prune(sgm_ctx* ctx, sgm_trainer* tr, double thr) {
    cudaStream_t s = ctx->stream;
    const uint64_t n = tr->n;
    if (n == 0) return;
    const int k = tr->k;
    CK(tr->keep.reserve(n));
    CK(tr->kept.reserve(4 * n));
    CK(tr->sel_count.reserve(8));
    launch_keep_flags(tr->P.as<double>() + 4 * n, n, thr, tr->keep.as<uint8_t>(), s);
    size_t tmp = 0;
    thrust::counting_iterator<uint32_t> ids(0);
    CK(cub::DeviceSelect::Flagged(nullptr, tmp, ids, tr->keep.as<uint8_t>(), tr->kept.as<uint32_t>(),
                                  tr->sel_count.as<uint32_t>(), static_cast<int>(n), s));
    CK(tr->sel_tmp.reserve(tmp));
    CK(cub::DeviceSelect::Flagged(tr->sel_tmp.p, tmp, ids, tr->keep.as<uint8_t>(), tr->kept.as<uint32_t>(),
                                  tr->sel_count.as<uint32_t>(), static_cast<int>(n), s));
    ctx->stats.kernel_launches += 2;
    uint32_t m = 0;
    CK(cudaMemcpyAsync(&m, tr->sel_count.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (m == n) return;
    const size_t per = 8 + static_cast<size_t>(k);
    const size_t ms = std::max<uint64_t>(m, 1);
    const uint32_t* kept = tr->kept.as<uint32_t>();
    // segments of the shared layout: (offset in units of n, stride)
    const int seg_off[5] = {0, 3, 4, 5, 8};
    const int seg_w[5] = {3, 1, 1, 3, k};
    for (DevBuf* buf : {&tr->P, &tr->M, &tr->V}) {
        DevBuf next;
        CK(next.reserve(8 * per * ms));
        for (int g = 0; g < 5; ++g)
            launch_gather_f64(buf->as<double>() + seg_off[g] * n, next.as<double>() + seg_off[g] * m, kept,
                              m, seg_w[g], s);
        *buf = std::move(next);
    }
    DevBuf nidx, nrows;
    CK(nidx.reserve(2 * k * ms));
    CK(nrows.reserve(4 * ms));
    launch_gather_u16(tr->sidx.as<uint16_t>(), nidx.as<uint16_t>(), kept, m, k, s);
    launch_gather_u16(tr->rows.as<uint16_t>(), nrows.as<uint16_t>(), kept, m, 2, s);  // u32 as 2 x u16
    tr->sidx = std::move(nidx);
    tr->rows = std::move(nrows);
    ctx->stats.kernel_launches += 16;
    tr->n = m;
    trainer_rebuild(ctx, tr);
}


}  // namespace


struct sgm_evaluator {
    int num_classes = 0, C = 0;
    struct View {
        std::vector<unsigned long long> confusion;  // [C][C]
        unsigned long long top1 = 0, top3 = 0, total = 0;
        double mse_sum = 0, dep_sum = 0, dep_cnt = 0;
        int px = 0;
        uint32_t T = 0;      // pixels (unknown-labelled ones carry label 0xffff)
        DevBuf scores;       // [M][T] float
        DevBuf labels;       // [T] u16
    };
    std::vector<View> views;
    DevBuf conf, counters, photo_part, photo_out;
};


namespace {


void eval_add_view(sgm_ctx* ctx, sgm_evaluator* ev, const sgm_map* map, const CamParams& cam,
                   const OptParams& o, const sgm_frame* fr) {
    cudaStream_t s = ctx->stream;
    const int C = ev->C;
    const size_t px = static_cast<size_t>(cam.W) * cam.H;
    if (px >= (1ull << 31)) fail(SGM_ERR_UNSUPPORTED, "evaluator: more than 2^31-1 pixels");
    // render(map, camera, pose, RenderChannels::all()) into HBM
    CK(ctx->planes.reserve(8 * px * (5 + C)));
    double* d_sil = ctx->planes.as<double>();
    double* d_color = d_sil + px;
    double* d_depth = d_color + 3 * px;
    double* d_sem = d_depth + px;
    RenderTargets rt;
    rt.channels = SGM_COLOR | SGM_DEPTH | SGM_SEMANTICS;
    rt.color = d_color;
    rt.depth = d_depth;
    rt.sil = d_sil;
    rt.sem = d_sem;
    run_views(ctx, map, cam, o, 1, &fr->pose, Mode::Render, rt, nullptr, nullptr);
    const float* f_rgb = fr->planes.as<float>();
    const float* f_depth = f_rgb + 3 * px;
    const float* f_sem = f_depth + px;
    CK(ev->conf.reserve(8ull * C * C));
    CK(ev->counters.reserve(64));
    const int nb = eval_photo_blocks(static_cast<int>(px));
    CK(ev->photo_part.reserve(24ull * nb + 24));
    CK(ev->photo_out.reserve(24));
    auto* conf = ev->conf.as<unsigned long long>();
    auto* cnt = ev->counters.as<unsigned long long>();
    CK(cudaMemsetAsync(conf, 0, 8ull * C * C, s));
    CK(cudaMemsetAsync(cnt, 0, 24, s));
    sgm_evaluator::View v;
    v.px = static_cast<int>(px);
    v.T = static_cast<uint32_t>(px);
    const int M = C - 1;
    CK(v.scores.reserve(4ull * px * std::max(M, 1)));
    CK(v.labels.reserve(2ull * px));
    need_smem(ctx->device, eval_view_smem(C), C, "evaluator");
    launch_eval_view(d_sem, d_sil, f_sem, static_cast<int>(px), C, conf, cnt, v.labels.as<uint16_t>(),
                     v.scores.as<float>(), s);
    launch_eval_photo(d_color, d_depth, f_rgb, f_depth, static_cast<int>(px), ev->photo_part.as<double>(),
                      ev->photo_out.as<double>(), s);
    ctx->stats.kernel_launches += 3;
    v.confusion.resize(static_cast<size_t>(C) * C);
    unsigned long long hc[3];
    double hp[3];
    CK(cudaMemcpyAsync(v.confusion.data(), conf, 8ull * C * C, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hc, cnt, 24, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hp, ev->photo_out.p, 24, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    v.top1 = hc[0];
    v.top3 = hc[1];
    v.total = hc[2];
    v.mse_sum = hp[0];
    v.dep_sum = hp[1];
    v.dep_cnt = hp[2];
    ev->views.push_back(std::move(v));
}

// AP per class (evaluator.cpp:151-188) over all views' pixels in (view, pixel) order; the
// unknown-labelled ones sort after every valid score and are never positive.
// Returns -1 for classes without positives.
std::vector<double> eval_ap(sgm_ctx* ctx, sgm_evaluator* ev, const std::vector<uint64_t>& positives) {
    cudaStream_t s = ctx->stream;
    const int M = ev->C - 1;
    uint64_t T = 0;
    for (auto& v : ev->views) T += v.T;
    std::vector<double> ap(static_cast<size_t>(std::max(M, 0)), -1.0);
    if (T == 0 || M <= 0) return ap;
    if (T >= (1ull << 31)) fail(SGM_ERR_UNSUPPORTED, "evaluator: more than 2^31-1 pixels in total");
    DevBuf sc, lab, keys, keys_alt, pos, pos_alt, tp, terms, sum, tmpb;
    CK(sc.reserve(4 * T));
    CK(lab.reserve(2 * T));
    CK(keys.reserve(4 * T));
    CK(keys_alt.reserve(4 * T));
    CK(pos.reserve(4 * T));
    CK(pos_alt.reserve(4 * T));
    CK(tp.reserve(4 * T));
    CK(terms.reserve(8 * T));
    CK(sum.reserve(8 * static_cast<size_t>(M)));
    uint64_t off = 0;
    for (auto& v : ev->views) {
        if (v.T) CK(cudaMemcpyAsync(lab.as<uint16_t>() + off, v.labels.p, 2ull * v.T, cudaMemcpyDeviceToDevice, s));
        off += v.T;
    }
    const int n = static_cast<int>(T);
    size_t need = 0, t1 = 0, t2 = 0, t3 = 0;
    {
        cub::DoubleBuffer<uint32_t> dk(keys.as<uint32_t>(), keys_alt.as<uint32_t>());
        cub::DoubleBuffer<uint32_t> dv(pos.as<uint32_t>(), pos_alt.as<uint32_t>());
        CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, dk, dv, n, 0, 32, s));
        CK(cub::DeviceScan::InclusiveSum(nullptr, t2, pos.as<uint32_t>(), tp.as<uint32_t>(), n, s));
        CK(cub::DeviceReduce::Sum(nullptr, t3, terms.as<double>(), sum.as<double>(), n, s));
        need = std::max(t1, std::max(t2, t3));
    }
    CK(tmpb.reserve(need));
    for (int c = 0; c < M; ++c) {
        if (positives[static_cast<size_t>(c)] == 0) continue;  // :166
        off = 0;
        for (auto& v : ev->views) {
            if (v.T)
                CK(cudaMemcpyAsync(sc.as<float>() + off, v.scores.as<float>() + static_cast<size_t>(c) * v.T,
                                   4ull * v.T, cudaMemcpyDeviceToDevice, s));
            off += v.T;
        }
        launch_eval_keys(sc.as<float>(), lab.as<uint16_t>(), static_cast<uint32_t>(T), c, keys.as<uint32_t>(),
                         pos.as<uint32_t>(), s);
        cub::DoubleBuffer<uint32_t> dk(keys.as<uint32_t>(), keys_alt.as<uint32_t>());
        cub::DoubleBuffer<uint32_t> dv(pos.as<uint32_t>(), pos_alt.as<uint32_t>());
        size_t t = need;
        CK(cub::DeviceRadixSort::SortPairs(tmpb.p, t, dk, dv, n, 0, 32, s));  // stable
        t = need;
        CK(cub::DeviceScan::InclusiveSum(tmpb.p, t, dv.Current(), tp.as<uint32_t>(), n, s));
        launch_eval_ap_terms(dv.Current(), tp.as<uint32_t>(), static_cast<uint32_t>(T),
                             static_cast<double>(positives[static_cast<size_t>(c)]), terms.as<double>(), s);
        t = need;
        CK(cub::DeviceReduce::Sum(tmpb.p, t, terms.as<double>(), sum.as<double>() + c, n, s));
        ctx->stats.kernel_launches += 5;
    }
    std::vector<double> h(static_cast<size_t>(M));
    CK(cudaMemcpyAsync(h.data(), sum.p, 8ull * M, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int c = 0; c < M; ++c)
        if (positives[static_cast<size_t>(c)]) ap[static_cast<size_t>(c)] = h[static_cast<size_t>(c)];
    return ap;
}


}  // namespace


struct sgm_emap {
    EmapParams p{};
    DevBuf grid, first_free, first_hit, log, keys, keys_alt, ids, ids_alt, fresh, counters, depth,
        lattice, ok, sort_tmp;
    HostBuf h_counters;
    uint64_t log_n = 0, free_count = 0, occupied_count = 0;
};


namespace {


// Sorts the n emitted (key, id) pairs by key and appends the ids to the changelog.
void emap_append_sorted(sgm_ctx* ctx, sgm_emap* em, uint64_t n) {
    if (n == 0) return;
    cudaStream_t s = ctx->stream;
    cub::DoubleBuffer<unsigned long long> dk(em->keys.as<unsigned long long>(),
                                             em->keys_alt.as<unsigned long long>());
    cub::DoubleBuffer<int32_t> dv(em->ids.as<int32_t>(), em->ids_alt.as<int32_t>());
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, static_cast<int>(n), 0, 64, s));
    CK(em->sort_tmp.reserve(tmp));
    CK(cub::DeviceRadixSort::SortPairs(em->sort_tmp.p, tmp, dk, dv, static_cast<int>(n), 0, 64, s));
    ctx->stats.kernel_launches += 1;
    CK(cudaMemcpyAsync(em->log.as<int32_t>() + em->log_n, dv.Current(), 4 * n,
                       cudaMemcpyDeviceToDevice, s));
    em->log_n += n;
}

// Pass 2 + counts + changelog append; returns the number of newly logged voxels.
uint64_t emap_resolve(sgm_ctx* ctx, sgm_emap* em) {
    cudaStream_t s = ctx->stream;
    auto* cnt = em->counters.as<unsigned long long>();
    CK(cudaMemsetAsync(cnt, 0, 3 * sizeof(unsigned long long), s));
    launch_emap_resolve(em->p, em->grid.as<uint8_t>(), em->first_free.as<unsigned long long>(),
                        em->first_hit.as<uint32_t>(), em->keys.as<unsigned long long>(),
                        em->ids.as<int32_t>(), cnt, s);
    ctx->stats.kernel_launches += 1;
    auto* h = em->h_counters.as<unsigned long long>();
    CK(cudaMemcpyAsync(h, cnt, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    em->free_count = h[1];
    em->occupied_count = h[2];
    const uint64_t n = h[0];
    emap_append_sorted(ctx, em, n);
    CK(cudaStreamSynchronize(s));
    return n;
}

uint64_t emap_integrate(sgm_ctx* ctx, sgm_emap* em, const CamParams& cam, const sgm_pose& pose,
                        const float* d_depth, int stride) {
    WorldPose P;
    for (int i = 0; i < 9; ++i) P.R[i] = pose.R[i];
    for (int i = 0; i < 3; ++i) P.t[i] = pose.t[i];
    launch_emap_rays(em->p, cam, P, d_depth, stride, em->grid.as<uint8_t>(),
                     em->first_free.as<unsigned long long>(), em->first_hit.as<uint32_t>(),
                     ctx->stream);
    ctx->stats.kernel_launches += 1;
    return emap_resolve(ctx, em);
}


}  // namespace

extern "C" {

// ---------------------------------------------------------------- exploration map (f1)

int sgm_emap_create(sgm_ctx* ctx, const sgm_aabb* bounds, double voxel_size, sgm_emap** out) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!out || !bounds) fail(SGM_ERR_INVALID, "emap: null argument");
        *out = nullptr;
        if (voxel_size <= 0) fail(SGM_ERR_INVALID, "emap: voxel size must be > 0");  // explorer.cpp:13
        auto em = std::make_unique<sgm_emap>();
        uint64_t nvox = 1;
        for (int a = 0; a < 3; ++a) {
            em->p.origin[a] = bounds->min[a];
            const double e = bounds->max[a] - bounds->min[a];  // Aabb::extent
            em->p.dims[a] = std::max(static_cast<int>(std::ceil(e / voxel_size)), 1);  // :14-18
            nvox *= static_cast<uint64_t>(em->p.dims[a]);
        }
        if (nvox >= (1ull << 31)) fail(SGM_ERR_UNSUPPORTED, "emap: more than 2^31-1 voxels");
        em->p.voxel = voxel_size;
        em->p.nvox = nvox;
        cudaStream_t s = ctx->stream;
        CK(em->grid.reserve(nvox));
        CK(em->first_free.reserve(8 * nvox));
        CK(em->first_hit.reserve(4 * nvox));
        CK(em->log.reserve(4 * nvox));
        CK(em->keys.reserve(8 * nvox));
        CK(em->keys_alt.reserve(8 * nvox));
        CK(em->ids.reserve(4 * nvox));
        CK(em->ids_alt.reserve(4 * nvox));
        CK(em->fresh.reserve(nvox));
        CK(em->counters.reserve(3 * sizeof(unsigned long long)));
        CK(em->h_counters.reserve(3 * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(em->grid.p, 0, nvox, s));  // VoxelState::Unknown
        CK(cudaMemsetAsync(em->first_free.p, 0xff, 8 * nvox, s));
        CK(cudaMemsetAsync(em->first_hit.p, 0xff, 4 * nvox, s));
        CK(cudaMemsetAsync(em->fresh.p, 0, nvox, s));
        CK(cudaStreamSynchronize(s));
        *out = em.release();
    });
}

void sgm_emap_destroy(sgm_ctx* ctx, sgm_emap* emap) {
    if (!emap) return;
    if (ctx) {
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
    }
    delete emap;
}

int sgm_emap_info(sgm_ctx* ctx, const sgm_emap* em, double origin[3], double* voxel_size,
                  int32_t dims[3], uint64_t* free_count, uint64_t* occupied_count,
                  uint64_t* changelog_size) {
    return guard(ctx, [&] {
        if (!em) fail(SGM_ERR_INVALID, "emap is null");
        for (int a = 0; a < 3; ++a) {
            if (origin) origin[a] = em->p.origin[a];
            if (dims) dims[a] = em->p.dims[a];
        }
        if (voxel_size) *voxel_size = em->p.voxel;
        if (free_count) *free_count = em->free_count;
        if (occupied_count) *occupied_count = em->occupied_count;
        if (changelog_size) *changelog_size = em->log_n;
    });
}

int sgm_emap_integrate_device(sgm_ctx* ctx, sgm_emap* em, const sgm_camera* camera,
                              const sgm_pose* pose, const float* d_depth, int32_t stride,
                              uint64_t* newly_freed) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!em || !pose) fail(SGM_ERR_INVALID, "emap: null argument");
        const CamParams cam = to_cam(camera);
        if (stride < 1) fail(SGM_ERR_INVALID, "emap: stride must be >= 1");
        if (!d_depth) fail(SGM_ERR_INVALID, "emap: depth is null");
        const uint64_t n = emap_integrate(ctx, em, cam, *pose, d_depth, stride);
        if (newly_freed) *newly_freed = n;
    });
}

int sgm_emap_integrate(sgm_ctx* ctx, sgm_emap* em, const sgm_camera* camera, const sgm_pose* pose,
                       const float* depth, int32_t stride, uint64_t* newly_freed) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!em || !pose) fail(SGM_ERR_INVALID, "emap: null argument");
        const CamParams cam = to_cam(camera);
        if (stride < 1) fail(SGM_ERR_INVALID, "emap: stride must be >= 1");
        if (!depth) fail(SGM_ERR_INVALID, "emap: depth is null");
        const size_t bytes = 4ull * cam.W * cam.H;
        CK(em->depth.reserve(bytes));
        CK(cudaMemcpyAsync(em->depth.p, depth, bytes, cudaMemcpyHostToDevice, ctx->stream));
        const uint64_t n = emap_integrate(ctx, em, cam, *pose, em->depth.as<float>(), stride);
        if (newly_freed) *newly_freed = n;
    });
}

int sgm_emap_take_changelog(sgm_ctx* ctx, sgm_emap* em, int32_t* out, uint64_t capacity,
                            uint64_t* n) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!em) fail(SGM_ERR_INVALID, "emap is null");
        if (n) *n = em->log_n;
        if (em->log_n == 0) return;
        if (!out || capacity < em->log_n)
            fail(SGM_ERR_INVALID, "take_changelog: capacity %llu < %llu",
                 static_cast<unsigned long long>(capacity), static_cast<unsigned long long>(em->log_n));
        CK(cudaMemcpyAsync(out, em->log.p, 4 * em->log_n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        em->log_n = 0;
    });
}

int sgm_emap_reseed_changelog_with_free(sgm_ctx* ctx, sgm_emap* em) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!em) fail(SGM_ERR_INVALID, "emap is null");
        cudaStream_t s = ctx->stream;
        auto* cnt = em->counters.as<unsigned long long>();
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
        launch_emap_free_ids(em->p, em->grid.as<uint8_t>(), em->keys.as<unsigned long long>(),
                             em->ids.as<int32_t>(), cnt, s);
        ctx->stats.kernel_launches += 1;
        auto* h = em->h_counters.as<unsigned long long>();
        CK(cudaMemcpyAsync(h, cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        em->log_n = 0;  // explorer.cpp:119
        emap_append_sorted(ctx, em, h[0]);
    });
}

int sgm_emap_seed_region(sgm_ctx* ctx, sgm_emap* em, const sgm_aabb* box, int occupied) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!em || !box) fail(SGM_ERR_INVALID, "emap: null argument");
        launch_emap_seed(em->p, *box, occupied ? 1 : 0, em->grid.as<uint8_t>(),
                         em->first_free.as<unsigned long long>(), em->first_hit.as<uint32_t>(),
                         ctx->stream);
        ctx->stats.kernel_launches += 1;
        emap_resolve(ctx, em);
    });
}

int sgm_emap_grid(sgm_ctx* ctx, const sgm_emap* em, uint8_t* out, uint64_t capacity) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!em || !out) fail(SGM_ERR_INVALID, "emap: null argument");
        if (capacity < em->p.nvox) fail(SGM_ERR_INVALID, "emap_grid: capacity < voxel count");
        CK(cudaMemcpyAsync(out, em->grid.p, em->p.nvox, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int sgm_sample_candidates(sgm_ctx* ctx, sgm_emap* em, double v1, int32_t v2, const double* heights,
                          int32_t n_heights, sgm_candidate* out, uint64_t capacity,
                          uint64_t* n_out) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!em) fail(SGM_ERR_INVALID, "emap is null");
        if (!(v1 > 0)) fail(SGM_ERR_INVALID, "sample_candidates: v1 must be > 0");
        if (v2 < 0 || n_heights < 0 || (n_heights > 0 && !heights))
            fail(SGM_ERR_INVALID, "sample_candidates: bad schedule");
        if (n_out) *n_out = 0;
        if (em->log_n == 0) return;  // fresh_set empty (explorer.cpp:161)
        // lattice positions in the reference's loop order (:163-172)
        double top[3];
        for (int a = 0; a < 3; ++a) top[a] = em->p.origin[a] + static_cast<double>(em->p.dims[a]) * em->p.voxel;
        std::vector<double> pos;
        for (int hi = 0; hi < n_heights; ++hi)
            for (double x = em->p.origin[0]; x <= top[0] + 1e-9; x += v1)
                for (double z = em->p.origin[2]; z <= top[2] + 1e-9; z += v1) {
                    pos.push_back(x);
                    pos.push_back(heights[hi]);
                    pos.push_back(z);
                }
        const int np = static_cast<int>(pos.size() / 3);
        std::vector<uint8_t> ok(static_cast<size_t>(np));
        cudaStream_t s = ctx->stream;
        if (np > 0) {
            CK(em->lattice.reserve(8 * pos.size()));
            CK(em->ok.reserve(static_cast<size_t>(np)));
            CK(cudaMemcpyAsync(em->lattice.p, pos.data(), 8 * pos.size(), cudaMemcpyHostToDevice, s));
            launch_emap_mark(em->log.as<int32_t>(), em->log_n, em->fresh.as<uint8_t>(), 1, s);
            launch_emap_lattice(em->p, em->lattice.as<double>(), np, em->grid.as<uint8_t>(),
                                em->fresh.as<uint8_t>(), em->ok.as<uint8_t>(), s);
            launch_emap_mark(em->log.as<int32_t>(), em->log_n, em->fresh.as<uint8_t>(), 0, s);
            ctx->stats.kernel_launches += 3;
            CK(cudaMemcpyAsync(ok.data(), em->ok.p, static_cast<size_t>(np), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        uint64_t hits = 0;
        for (uint8_t f : ok) hits += f;
        const uint64_t need = hits * static_cast<uint64_t>(v2);
        if (n_out) *n_out = need;
        if (need > 0 && (!out || capacity < need))
            fail(SGM_ERR_INVALID, "sample_candidates: capacity %llu < %llu",
                 static_cast<unsigned long long>(capacity), static_cast<unsigned long long>(need));
        std::vector<double> dirs(3 * static_cast<size_t>(v2));
        sgm_fibonacci_directions(v2, 45.0, dirs.data());
        uint64_t w = 0;
        for (int j = 0; j < np; ++j) {
            if (!ok[static_cast<size_t>(j)]) continue;
            for (int d = 0; d < v2; ++d, ++w) {
                for (int a = 0; a < 3; ++a) {
                    out[w].position[a] = pos[3 * static_cast<size_t>(j) + a];
                    out[w].direction[a] = dirs[3 * static_cast<size_t>(d) + a];
                }
            }
        }
        em->log_n = 0;  // the changelog is consumed (:159)
    });
}


// ---------------------------------------------------------------- on-device optimize_map (f2)

int sgm_frame_upload(sgm_ctx* ctx, int32_t width, int32_t height, int32_t num_classes,
                     const sgm_pose* pose, const float* rgb, const float* depth, const float* sem,
                     sgm_frame** out) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!out || !pose || !rgb || !depth || !sem) fail(SGM_ERR_INVALID, "frame: null argument");
        *out = nullptr;
        if (width <= 0 || height <= 0 || num_classes < 0) fail(SGM_ERR_INVALID, "frame: bad size");
        auto f = std::make_unique<sgm_frame>();
        f->W = width;
        f->H = height;
        f->C = num_classes + 1;
        f->pose = to_pose(*pose);
        const size_t px = static_cast<size_t>(width) * height;
        CK(f->planes.reserve(4 * px * (4 + f->C)));
        float* d = f->planes.as<float>();
        CK(cudaMemcpyAsync(d, rgb, 12 * px, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d + 3 * px, depth, 4 * px, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d + 4 * px, sem, 4 * px * f->C, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        *out = f.release();
    });
}

void sgm_frame_release(sgm_ctx* ctx, sgm_frame* frame) {
    if (!frame) return;
    if (ctx) {
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
    }
    delete frame;
}

int sgm_trainer_create(sgm_ctx* ctx, uint64_t n, int32_t k, int32_t num_classes,
                       const double* centers, const double* log_radii, const double* opacity_logits,
                       const double* colors, const uint16_t* sem_indices, const double* sem_probs,
                       const double* adam_mv, int64_t step_count, sgm_trainer** out) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!out) fail(SGM_ERR_INVALID, "out is null");
        *out = nullptr;
        if (k < 1 || k > num_classes + 1) fail(SGM_ERR_INVALID, "map: k must be in [1, num_classes+1]");
        if (n > 0 && (!centers || !log_radii || !opacity_logits || !colors || !sem_indices || !sem_probs))
            fail(SGM_ERR_INVALID, "map: null array with n > 0");
        if (n >= (1ull << 31)) fail(SGM_ERR_UNSUPPORTED, "trainer: more than 2^31-1 Gaussians");
        if (step_count < 0) fail(SGM_ERR_INVALID, "trainer: negative step count");
        const int C = num_classes + 1;
        int dup = 0;
        std::vector<uint32_t> seen(static_cast<size_t>(C), 0xffffffffu);
        for (uint64_t i = 0; i < n; ++i)
            for (int j = 0; j < k; ++j) {
                const uint16_t c = sem_indices[i * k + j];
                if (c >= C) fail(SGM_ERR_INVALID, "map: semantic index >= channels %d", C);
                if (seen[c] == static_cast<uint32_t>(i)) dup = 1;
                seen[c] = static_cast<uint32_t>(i);
            }
        auto tr = std::make_unique<sgm_trainer>();
        tr->n = n;
        tr->k = k;
        tr->num_classes = num_classes;
        tr->t = step_count;
        tr->dup = dup;
        const size_t per = 8 + static_cast<size_t>(k);
        const size_t ns = std::max<uint64_t>(n, 1);
        cudaStream_t s = ctx->stream;
        CK(tr->P.reserve(8 * per * ns));
        CK(tr->M.reserve(8 * per * ns));
        CK(tr->V.reserve(8 * per * ns));
        CK(tr->sidx.reserve(2 * k * ns));
        CK(tr->rows.reserve(4 * ns));
        {
            std::vector<uint32_t> iota(n);
            for (uint64_t i = 0; i < n; ++i) iota[i] = static_cast<uint32_t>(i);
            if (n) CK(cudaMemcpyAsync(tr->rows.p, iota.data(), 4 * n, cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
        }
        double* P = tr->P.as<double>();
        if (n) {
            CK(cudaMemcpyAsync(P, centers, 24 * n, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(P + 3 * n, log_radii, 8 * n, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(P + 4 * n, opacity_logits, 8 * n, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(P + 5 * n, colors, 24 * n, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(P + 8 * n, sem_probs, 8 * k * n, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(tr->sidx.p, sem_indices, 2 * k * n, cudaMemcpyHostToDevice, s));
            if (adam_mv) {
                CK(cudaMemcpyAsync(tr->M.p, adam_mv, 8 * per * n, cudaMemcpyHostToDevice, s));
                CK(cudaMemcpyAsync(tr->V.p, adam_mv + per * n, 8 * per * n, cudaMemcpyHostToDevice, s));
            } else {
                CK(cudaMemsetAsync(tr->M.p, 0, 8 * per * n, s));
                CK(cudaMemsetAsync(tr->V.p, 0, 8 * per * n, s));
            }
        }
        trainer_rebuild(ctx, tr.get());
        CK(cudaStreamSynchronize(s));
        *out = tr.release();
    });
}

void sgm_trainer_destroy(sgm_ctx* ctx, sgm_trainer* tr) {
    if (!tr) return;
    if (ctx) {
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->last_map == &tr->map) ctx->last_valid = false;
    }
    delete tr;
}

int sgm_trainer_size(sgm_ctx* ctx, const sgm_trainer* tr, uint64_t* n, int64_t* step_count) {
    return guard(ctx, [&] {
        if (!tr) fail(SGM_ERR_INVALID, "trainer is null");
        if (n) *n = tr->n;
        if (step_count) *step_count = tr->t;
    });
}

int sgm_trainer_rows(sgm_ctx* ctx, const sgm_trainer* tr, uint32_t* rows) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!tr || (!rows && tr->n)) fail(SGM_ERR_INVALID, "null argument");
        if (tr->n == 0) return;
        CK(cudaMemcpyAsync(rows, tr->rows.p, 4 * tr->n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int sgm_trainer_download(sgm_ctx* ctx, const sgm_trainer* tr, double* centers, double* log_radii,
                         double* opacity_logits, double* colors, uint16_t* sem_indices,
                         double* sem_probs, double* adam_mv) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!tr) fail(SGM_ERR_INVALID, "trainer is null");
        const uint64_t n = tr->n;
        if (n == 0) return;
        const int k = tr->k;
        const size_t per = 8 + static_cast<size_t>(k);
        cudaStream_t s = ctx->stream;
        const double* P = tr->P.as<double>();
        if (centers) CK(cudaMemcpyAsync(centers, P, 24 * n, cudaMemcpyDeviceToHost, s));
        if (log_radii) CK(cudaMemcpyAsync(log_radii, P + 3 * n, 8 * n, cudaMemcpyDeviceToHost, s));
        if (opacity_logits) CK(cudaMemcpyAsync(opacity_logits, P + 4 * n, 8 * n, cudaMemcpyDeviceToHost, s));
        if (colors) CK(cudaMemcpyAsync(colors, P + 5 * n, 24 * n, cudaMemcpyDeviceToHost, s));
        if (sem_probs) CK(cudaMemcpyAsync(sem_probs, P + 8 * n, 8 * k * n, cudaMemcpyDeviceToHost, s));
        if (sem_indices) CK(cudaMemcpyAsync(sem_indices, tr->sidx.p, 2 * k * n, cudaMemcpyDeviceToHost, s));
        if (adam_mv) {
            CK(cudaMemcpyAsync(adam_mv, tr->M.p, 8 * per * n, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(adam_mv + per * n, tr->V.p, 8 * per * n, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
    });
}

int sgm_optimize_map(sgm_ctx* ctx, sgm_trainer* tr, const sgm_camera* camera, uint64_t n_frames,
                     sgm_frame* const* frames, const sgm_options* opt,
                     const sgm_adam_params* adam, const double weights[7],
                     const sgm_optimize_config* cfg, int32_t iters, double* history,
                     int32_t* n_done) {
    if (n_done) *n_done = 0;
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!tr || !adam || !weights || !cfg) fail(SGM_ERR_INVALID, "optimize_map: null argument");
        if (n_frames == 0 || !frames) fail(SGM_ERR_INVALID, "optimize_map: no frames");  // mapper.cpp:244
        if (iters < 1) fail(SGM_ERR_INVALID, "optimize_map: iters must be >= 1");       // :245
        const CamParams cam = to_cam(camera);
        const OptParams o = to_opt(opt, cam);
        for (uint64_t f = 0; f < n_frames; ++f) {
            if (!frames[f]) fail(SGM_ERR_INVALID, "optimize_map: null frame");
            if (frames[f]->W != cam.W || frames[f]->H != cam.H || frames[f]->C != tr->num_classes + 1)
                fail(SGM_ERR_INVALID, "optimize_map: frame %llu does not match the camera / classes",
                     static_cast<unsigned long long>(f));
        }
        const AdamHyper h{adam->lr_center, adam->lr_radius, adam->lr_opacity, adam->lr_color,
                          adam->lr_sem,    adam->beta1,     adam->beta2,      adam->eps,
                          adam->eps_sem};
        cudaStream_t s = ctx->stream;
        double initial_total = -1.0;
        int diverged_streak = 0;
        for (int it = 0; it < iters; ++it) {
            const sgm_frame* kf = frames[static_cast<uint64_t>(it) % n_frames];
            if (tr->n == 0) break;  // :253
            const size_t px = static_cast<size_t>(cam.W) * cam.H;
            const float* fp = kf->planes.as<float>();
            double rep[7];
            backward_core(ctx, &tr->map, cam, o, kf->pose, fp, fp + 3 * px, fp + 4 * px, weights, 1, 1,
                          rep);
            // adam.step (mapper.cpp:10-51)
            ++tr->t;
            const double bc1 = 1.0 - std::pow(h.beta1, static_cast<double>(tr->t));
            const double bc2 = 1.0 - std::pow(h.beta2, static_cast<double>(tr->t));
            launch_adam(tr->P.as<double>(), ctx->bw_grad.as<double>(), tr->M.as<double>(),
                        tr->V.as<double>(), tr->n, tr->k, h, bc1, bc2, s);
            launch_derive(tr->P.as<double>(), tr->n, tr->k, tr->map.dev.kpad, tr->map.dev.sem_perm,
                          tr->map.geo.as<double>(), tr->map.color.as<double>(), tr->map.prob.as<double>(), s);
            tr->map.rec_valid = false;
            ctx->stats.kernel_launches += 3;
            CK(cudaGetLastError());
            if (ctx->last_map == &tr->map) ctx->last_valid = false;
            const double total = (rep[1] + 0.5 * rep[0]) + rep[2];  // LossReport::total (losses.hpp:29-30)
            if (history) std::memcpy(history + 7 * static_cast<size_t>(it), rep, sizeof(rep));
            if (initial_total < 0) initial_total = total;
            if (initial_total > 0 && total > cfg->divergence_factor * initial_total) {
                if (++diverged_streak >= cfg->divergence_window)
                    fail(SGM_ERR_INVALID,
                         "optimize_map: diverged (loss %f vs initial %f for %d iterations)", total,
                         initial_total, diverged_streak);
            } else {
                diverged_streak = 0;
            }
            if (cfg->prune_every > 0 && tr->t % cfg->prune_every == 0) trainer_prune(ctx, tr, cfg->prune_opacity);
            if (n_done) *n_done = it + 1;
        }
        CK(cudaStreamSynchronize(s));
    });
}


// ---------------------------------------------------------------- evaluation (f3)

int sgm_eval_create(sgm_ctx* ctx, int32_t num_classes, sgm_evaluator** out) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!out) fail(SGM_ERR_INVALID, "out is null");
        *out = nullptr;
        if (num_classes < 0 || num_classes > 65534) fail(SGM_ERR_INVALID, "evaluator: bad class count");
        auto ev = std::make_unique<sgm_evaluator>();
        ev->num_classes = num_classes;
        ev->C = num_classes + 1;
        *out = ev.release();
    });
}

void sgm_eval_destroy(sgm_ctx* ctx, sgm_evaluator* ev) {
    if (!ev) return;
    if (ctx) {
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
    }
    delete ev;
}

int sgm_eval_add_view(sgm_ctx* ctx, sgm_evaluator* ev, const sgm_map* map, const sgm_camera* camera,
                      const sgm_options* opt, const sgm_frame* frame) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!ev || !map || !frame) fail(SGM_ERR_INVALID, "evaluator: null argument");
        const CamParams cam = to_cam(camera);
        const OptParams o = to_opt(opt, cam);
        if (frame->W != cam.W || frame->H != cam.H || frame->C != ev->C || map->dev.C != ev->C)
            fail(SGM_ERR_INVALID, "semantic_metrics: resolution mismatch");  // evaluator.cpp:107-108
        eval_add_view(ctx, ev, map, cam, o, frame);
    });
}

int sgm_eval_report(sgm_ctx* ctx, sgm_evaluator* ev, double summary[7], double* per_view_miou,
                    double* per_view_psnr, double* per_class, uint64_t* n_per_class) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!ev) fail(SGM_ERR_INVALID, "evaluator is null");
        if (ev->views.empty()) fail(SGM_ERR_INVALID, "semantic_metrics: view count mismatch");  // :95-96
        const int C = ev->C, M = C - 1;
        const size_t CC = static_cast<size_t>(C) * C;
        std::vector<unsigned long long> pooled(CC, 0);
        unsigned long long top1 = 0, top3 = 0, total = 0;
        std::vector<double> view_miou;
        for (const auto& v : ev->views) {  // :100-148
            top1 += v.top1;
            top3 += v.top3;
            total += v.total;
            for (size_t i = 0; i < CC; ++i) pooled[i] += v.confusion[i];
            double iou_sum = 0;
            int iou_classes = 0;
            for (int c = 0; c < C; ++c) {
                int64_t rowsum = 0;
                for (int m = 0; m < C; ++m) rowsum += static_cast<int64_t>(v.confusion[static_cast<size_t>(c) * C + m]);
                if (rowsum == 0) continue;  // !present[c]
                const int64_t tp = static_cast<int64_t>(v.confusion[static_cast<size_t>(c) * C + c]);
                int64_t fn = 0, fp = 0;
                for (int m = 0; m < C; ++m)
                    if (m != c) {
                        fn += static_cast<int64_t>(v.confusion[static_cast<size_t>(c) * C + m]);
                        fp += static_cast<int64_t>(v.confusion[static_cast<size_t>(m) * C + c]);
                    }
                const int64_t uni = tp + fn + fp;
                if (uni > 0) {
                    iou_sum += static_cast<double>(tp) / uni;
                    ++iou_classes;
                }
            }
            view_miou.push_back(iou_classes ? 100.0 * iou_sum / iou_classes : 0.0);
        }
        double miou = 0.0;  // std::accumulate in order, then / size
        for (double x : view_miou) miou += x;
        miou /= static_cast<double>(view_miou.size());
        const double top1_pct = total ? 100.0 * top1 / total : 0.0;
        const double top3_pct = total ? 100.0 * top3 / total : 0.0;
        // AP (:151-196): positives of class c = its ground-truth pixel count
        std::vector<uint64_t> positives(static_cast<size_t>(std::max(M, 0)), 0);
        for (int c = 0; c < M; ++c)
            for (int m = 0; m < C; ++m) positives[static_cast<size_t>(c)] += pooled[static_cast<size_t>(c) * C + m];
        const std::vector<double> ap = eval_ap(ctx, ev, positives);
        struct PC {
            int id;
            double iou = 0, ap = 0, f1 = 0;
            uint64_t gt = 0;
        };
        std::vector<PC> pcs;
        double ap_sum = 0;
        int ap_classes = 0;
        for (int c = 0; c < M; ++c) {
            if (ap[static_cast<size_t>(c)] < 0) continue;
            ap_sum += ap[static_cast<size_t>(c)];
            ++ap_classes;
            PC pc;
            pc.id = c;
            pc.ap = 100.0 * ap[static_cast<size_t>(c)];
            pc.gt = positives[static_cast<size_t>(c)];
            pcs.push_back(pc);
        }
        const double map_pct = ap_classes ? 100.0 * ap_sum / ap_classes : 0.0;
        double f1_sum = 0;  // macro F1 (:199-232)
        int f1_classes = 0;
        for (int c = 0; c < M; ++c) {
            const int64_t tp = static_cast<int64_t>(pooled[static_cast<size_t>(c) * C + c]);
            int64_t fn = 0, fp = 0;
            for (int m = 0; m < C; ++m)
                if (m != c) {
                    fn += static_cast<int64_t>(pooled[static_cast<size_t>(c) * C + m]);
                    fp += static_cast<int64_t>(pooled[static_cast<size_t>(m) * C + c]);
                }
            if (tp + fn + fp == 0) continue;
            const double f1 = tp > 0 ? 2.0 * tp / (2.0 * tp + fp + fn) : 0.0;
            f1_sum += f1;
            ++f1_classes;
            const double iou = tp + fn + fp > 0 ? static_cast<double>(tp) / (tp + fn + fp) : 0.0;
            bool found = false;
            for (auto& pc : pcs)
                if (pc.id == c) {
                    pc.f1 = 100.0 * f1;
                    pc.iou = 100.0 * iou;
                    found = true;
                }
            if (!found) {
                PC pc;
                pc.id = c;
                pc.f1 = 100.0 * f1;
                pc.iou = 100.0 * iou;
                pcs.push_back(pc);
            }
        }
        const double f1_pct = f1_classes ? 100.0 * f1_sum / f1_classes : 0.0;
        std::sort(pcs.begin(), pcs.end(), [](const PC& a, const PC& b) { return a.id < b.id; });
        // photometric (:274-297)
        std::vector<double> psnr;
        double dep_sum = 0, dep_cnt = 0;
        for (const auto& v : ev->views) {
            double mse = v.mse_sum / static_cast<double>(3ull * v.px);  // mapper.cpp:97-107
            psnr.push_back(mse <= 0.0 ? 100.0 : std::min(100.0, 10.0 * std::log10(1.0 / mse)));
            dep_sum += v.dep_sum;
            dep_cnt += v.dep_cnt;
        }
        double psnr_db = 0.0;
        for (double x : psnr) psnr_db += x;
        psnr_db /= static_cast<double>(psnr.size());
        const double depth_l1 = dep_cnt > 0 ? 100.0 * dep_sum / dep_cnt : 0.0;
        if (summary) {
            summary[0] = miou;
            summary[1] = top1_pct;
            summary[2] = top3_pct;
            summary[3] = map_pct;
            summary[4] = f1_pct;
            summary[5] = psnr_db;
            summary[6] = depth_l1;
        }
        for (size_t i = 0; i < ev->views.size(); ++i) {
            if (per_view_miou) per_view_miou[i] = view_miou[i];
            if (per_view_psnr) per_view_psnr[i] = psnr[i];
        }
        if (per_class)
            for (size_t i = 0; i < pcs.size(); ++i) {
                double* r = per_class + 5 * i;
                r[0] = pcs[i].id;
                r[1] = pcs[i].iou;
                r[2] = pcs[i].ap;
                r[3] = pcs[i].f1;
                r[4] = static_cast<double>(pcs[i].gt);
            }
        if (n_per_class) *n_per_class = pcs.size();
    });
}

}  // extern "C"
