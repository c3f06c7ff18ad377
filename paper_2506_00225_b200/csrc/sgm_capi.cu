// C ABI (include/sgm.h), part 1: context, map, render, scoring, Fisher, backward.
// The view pipeline is in sgm_pipeline.cu; the exploration map, trainer and evaluator
// entry points are in sgm_capi_ext.cu.
#include "sgm_ctx.h"

namespace {
thread_local std::string g_create_error;
}  // namespace


extern "C" {

int sgm_abi_version(void) { return SGM_ABI_VERSION; }

int sgm_ctx_create(int device, sgm_ctx** out) {
    g_create_error.clear();
    if (!out) {
        g_create_error = "out is null";
        return SGM_ERR_INVALID;
    }
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        g_create_error = std::string("no CUDA device available (this library has no CPU path): ") +
                         cudaGetErrorString(e);
        return SGM_ERR_CUDA;
    }
    if (device < 0 || device >= count) {
        g_create_error = "device index out of range";
        return SGM_ERR_INVALID;
    }
    auto* ctx = new (std::nothrow) sgm_ctx();
    if (!ctx) return SGM_ERR_OOM;
    ctx->device = device;
    int rc = guard(ctx, [&] {
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        int prio_low = 0, prio_high = 0;
        CK(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
        // binning kernels are small and latency-bound: give them priority so the
        // block scheduler slots them in as raster CTAs of the previous sub-batch retire
        CK(cudaStreamCreateWithPriority(&ctx->bin_stream, cudaStreamNonBlocking, prio_high));
        CK(cudaStreamCreateWithFlags(&ctx->up_stream, cudaStreamNonBlocking));
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        // tile lists of one group of views: a fifth of the device (36 GB on a B200), at least 8 GB
        ctx->list_budget = std::max<uint64_t>(uint64_t(8) << 30, total_b / 5) / 4;
        for (auto& ev : ctx->ev) CK(cudaEventCreate(&ev));
        CK(cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming));
        for (auto& ev : ctx->ev_binned) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        for (auto& ev : ctx->ev_r) CK(cudaEventCreate(&ev));
    });
    if (rc != SGM_OK) {
        g_create_error = ctx->err;
        delete ctx;
        return rc;
    }
    *out = ctx;
    return SGM_OK;
}

void sgm_ctx_destroy(sgm_ctx* ctx) {
    if (!ctx) return;
    if (ctx->rows_owner && ctx->rows_owner->rows_pending) {  // its staging uses ctx buffers
        ctx->rows_owner->rows_thread.join();
        ctx->rows_owner->rows_pending = false;
    }
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->bin_stream) cudaStreamSynchronize(ctx->bin_stream);
    if (ctx->up_stream) cudaStreamSynchronize(ctx->up_stream);
    if (ctx->ev_hstage) cudaEventDestroy(ctx->ev_hstage);
    if (ctx->ev_hrows) cudaEventDestroy(ctx->ev_hrows);
    for (auto& ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
    for (auto& ev : ctx->ev_binned)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev_r)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev_ring)
        if (ev) cudaEventDestroy(ev);
    cudaStream_t s = ctx->stream, s2 = ctx->bin_stream, s3 = ctx->up_stream;
    delete ctx;
    if (s) cudaStreamDestroy(s);
    if (s2) cudaStreamDestroy(s2);
    if (s3) cudaStreamDestroy(s3);
}

const char* sgm_last_error(const sgm_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

void* sgm_ctx_stream(sgm_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int sgm_ctx_synchronize(sgm_ctx* ctx) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int sgm_ctx_set_profiling(sgm_ctx* ctx, int enabled) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        ctx->profiling = enabled != 0;
    });
}

int sgm_ctx_get_stats(const sgm_ctx* ctx, sgm_stats* out) {
    if (!ctx || !out) return SGM_ERR_INVALID;
    *out = ctx->stats;
    return SGM_OK;
}

int sgm_ctx_reset_stats(sgm_ctx* ctx) {
    if (!ctx) return SGM_ERR_INVALID;
    ctx->stats = sgm_stats{};
    return SGM_OK;
}

// Map upload in two phases (the e2e step's per-step cost: about 112 MB at cfg1, bound by
// host memory bandwidth and the host libm activations):
//   A (this call, a pool of host threads): geometry SoA with the activations radius =
//     exp(log_r), alpha = sigmoid(logit) (reference libm, gaussian_map.hpp:36-37), the
//     semantic-index validation (a failure is reported here) and duplicate-class detection;
//     copied chunk by chunk on the ctx stream. Preprocess and binning need nothing else.
//   B (a staging thread, returning before it ends): clamped colours and the raw rows into
//     pinned memory, copied on the upload stream, then the class sort of the rows and the
//     channel-group bounds there; ev_rows marks the end. The raster waits for it
//     (map_ready), so phase B overlaps the preprocess and the first binning.
int sgm_map_upload_async(sgm_ctx* ctx, uint64_t n, int32_t k, int32_t num_classes,
                         const double* centers, const double* log_radii,
                         const double* opacity_logits, const double* colors,
                         const uint16_t* sem_indices, const double* sem_probs, sgm_map** out) {
    sgm_map* m = nullptr;
    int rc = guard(ctx, [&] {
        need_ctx(ctx);
        if (!out) fail(SGM_ERR_INVALID, "out is null");
        *out = nullptr;
        // GaussianMap(k, num_classes) invariant, gaussian_map.hpp:63-66
        if (k < 1 || k > num_classes + 1)
            fail(SGM_ERR_INVALID, "map: k must be in [1, num_classes+1]");
        if (n > 0 && (!centers || !log_radii || !opacity_logits || !colors || !sem_indices || !sem_probs))
            fail(SGM_ERR_INVALID, "map: null array with n > 0");
        if (n >= (1ull << 32)) fail(SGM_ERR_UNSUPPORTED, "map: more than 2^32-1 Gaussians");
        // the previous upload's staging thread and copies out of the pinned buffers
        if (ctx->rows_owner) map_ready(ctx, ctx->rows_owner);
        if (!ctx->ev_hstage) CK(cudaEventCreateWithFlags(&ctx->ev_hstage, cudaEventDisableTiming));
        if (!ctx->ev_hrows) CK(cudaEventCreateWithFlags(&ctx->ev_hrows, cudaEventDisableTiming));
        CK(cudaEventSynchronize(ctx->ev_hstage));
        CK(cudaEventSynchronize(ctx->ev_hrows));
        const int C = num_classes + 1;
        const int kpad = (k + 7) / 8 * 8;
        m = new sgm_map();
        m->num_classes = num_classes;
        const size_t ns = std::max<uint64_t>(n, 1);
        const size_t geo_b = 8 * 5 * ns, col_b = 8 * 4 * ns, idx_b = 2 * static_cast<size_t>(k) * ns,
                     prob_b = 8 * static_cast<size_t>(k) * ns;
        CK(ctx->h_stage.reserve(geo_b + 64));
        CK(ctx->h_rows.reserve(col_b + prob_b + idx_b + 64));
        double* geo = ctx->h_stage.as<double>();
        char* hr = ctx->h_rows.as<char>();
        double* col = reinterpret_cast<double*>(hr);
        double* rprob = reinterpret_cast<double*>(hr + col_b);
        uint16_t* ridx = reinterpret_cast<uint16_t*>(hr + col_b + prob_b);
        cudaStream_t s = ctx->stream;
        ctx->take(m->geo, geo_b);
        ctx->take(m->color, col_b);
        ctx->take(m->idx, 2 * ns * kpad);
        ctx->take(m->prob, 8 * ns * kpad);
        ctx->take(m->perm, 2 * ns * kpad);
        ctx->take(m->gbnd, 16 * ns);
        ctx->take(m->rec, 16 * ns * kpad);
        CK(m->geo.reserve(geo_b));
        CK(m->color.reserve(col_b));
        CK(m->idx.reserve(2 * ns * kpad));
        CK(m->prob.reserve(8 * ns * kpad));
        CK(m->perm.reserve(2 * ns * kpad));
        CK(m->gbnd.reserve(16 * ns));
        CK(ctx->upload_tmp.reserve(idx_b + prob_b + 64));
        CK(cudaEventCreateWithFlags(&m->ev_rows, cudaEventDisableTiming));
        const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        const unsigned nth = n > 65536 ? hw : 1;
        const unsigned kChunks = n > 65536 ? 8 : 1;
        // phase B's copies start per 1/16 of the rows, so the staging and the H2D copies overlap
        const unsigned kChunksB = n > 65536 ? 16 : 1;
        if (nth > 1 && (!ctx->workers || ctx->workers->size() < nth)) ctx->workers.reset(new HostPool(nth));
        HostPool* pool = nth > 1 ? ctx->workers.get() : nullptr;
        // ---- phase A: geometry + activations, chunk copies on s ----
        std::unique_ptr<std::atomic<unsigned>[]> finished(new std::atomic<unsigned>[kChunks]);
        for (unsigned c = 0; c < kChunks; ++c) finished[c].store(0);
        auto work_a = [&](unsigned w) {
            for (unsigned c = 0; c < kChunks; ++c) {
                const uint64_t ca = n * c / kChunks, cb = n * (c + 1) / kChunks;
                const uint64_t a = ca + (cb - ca) * w / nth, b = ca + (cb - ca) * (w + 1) / nth;
                for (uint64_t i = a; i < b; ++i) {
                    geo[i] = centers[3 * i];
                    geo[ns + i] = centers[3 * i + 1];
                    geo[2 * ns + i] = centers[3 * i + 2];
                    geo[3 * ns + i] = std::exp(log_radii[i]);                      // radius()
                    geo[4 * ns + i] = 1.0 / (1.0 + std::exp(-opacity_logits[i]));  // sigmoid
                }
                finished[c].fetch_add(1, std::memory_order_release);
            }
        };
        {
            if (pool) pool->start(nth, work_a);
            else work_a(0);
            cudaError_t copy_err = cudaSuccess;
            for (unsigned c = 0; c < kChunks; ++c) {
                while (finished[c].load(std::memory_order_acquire) < nth) std::this_thread::yield();
                const uint64_t ca = n * c / kChunks, cb = n * (c + 1) / kChunks;
                if (cb == ca) continue;
                for (int f = 0; f < 5 && copy_err == cudaSuccess; ++f)
                    copy_err = cudaMemcpyAsync(m->geo.as<double>() + f * ns + ca, geo + f * ns + ca,
                                               8 * (cb - ca), cudaMemcpyHostToDevice, s);
            }
            if (pool) pool->wait();
            CK(copy_err);
            CK(cudaEventRecord(ctx->ev_hstage, s));
        }
        DevMap& d = m->dev;
        d.n = n;
        d.k = k;
        d.kpad = kpad;
        d.C = C;
        const double* g = m->geo.as<double>();
        d.cx = g;
        d.cy = g + ns;
        d.cz = g + 2 * ns;
        d.rad = g + 3 * ns;
        d.alpha = g + 4 * ns;
        d.color4 = m->color.as<double>();
        d.sem_idx = m->idx.as<uint16_t>();
        d.sem_prob = m->prob.as<double>();
        d.sem_perm = m->perm.as<uint16_t>();
        d.dup_idx = 0;  // set by map_ready from phase B's scan of the rows
        d.gbounds = m->gbnd.as<uint4>();
        m->groups = choose_groups(C, k);
        ctx->stats.kernel_launches += n ? 2 : 0;  // the row sort and the group bounds (phase B)
        // ---- phase B: colours + rows, staged by a thread, copied / sorted on the upload stream
        char* draw = ctx->upload_tmp.as<char>();
        const int device = ctx->device;
        cudaStream_t us = ctx->up_stream;
        cudaEvent_t ev_hrows = ctx->ev_hrows;
        sgm_map* mm = m;
        m->rows_pending = true;
        m->rows_thread = std::thread([=]() {
            try {
                CK(cudaSetDevice(device));
                const unsigned kChunks = kChunksB;
                std::unique_ptr<std::atomic<unsigned>[]> done(new std::atomic<unsigned>[kChunks]);
                for (unsigned c = 0; c < kChunks; ++c) done[c].store(0);
                std::vector<int> bad(nth, -1), dup(nth, 0);
                auto work_b = [&](unsigned w) {
                    std::vector<uint32_t> seen(static_cast<size_t>(C), 0xffffffffu);
                    for (unsigned c = 0; c < kChunks; ++c) {
                        const uint64_t ca = n * c / kChunks, cb = n * (c + 1) / kChunks;
                        const uint64_t a = ca + (cb - ca) * w / nth, b = ca + (cb - ca) * (w + 1) / nth;
                        for (uint64_t i = a; i < b; ++i) {
                            for (int q = 0; q < 3; ++q) col[4 * i + q] = std::clamp(colors[3 * i + q], 0.0, 1.0);
                            col[4 * i + 3] = 0.0;
                            // index range (gaussian_map.hpp:63-66) and repeated classes
                            for (int j = 0; j < k; ++j) {
                                const uint16_t cl = sem_indices[i * k + j];
                                if (cl >= C) {
                                    if (bad[w] < 0) bad[w] = static_cast<int>(i % 0x7fffffff);
                                    continue;
                                }
                                if (seen[cl] == static_cast<uint32_t>(i)) dup[w] = 1;
                                seen[cl] = static_cast<uint32_t>(i);
                            }
                        }
                        std::memcpy(ridx + a * k, sem_indices + a * k, 2 * (b - a) * k);
                        std::memcpy(rprob + a * k, sem_probs + a * k, 8 * (b - a) * k);
                        done[c].fetch_add(1, std::memory_order_release);
                    }
                };
                if (pool) pool->start(nth, work_b);
                else work_b(0);
                cudaError_t e = cudaSuccess;
                for (unsigned c = 0; c < kChunks; ++c) {
                    while (done[c].load(std::memory_order_acquire) < nth) std::this_thread::yield();
                    const uint64_t ca = n * c / kChunks, cb = n * (c + 1) / kChunks;
                    if (cb == ca) continue;
                    if (e == cudaSuccess)
                        e = cudaMemcpyAsync(mm->color.as<double>() + 4 * ca, col + 4 * ca, 32 * (cb - ca),
                                            cudaMemcpyHostToDevice, us);
                    if (e == cudaSuccess)
                        e = cudaMemcpyAsync(draw + 8 * k * ca, rprob + k * ca, 8 * k * (cb - ca),
                                            cudaMemcpyHostToDevice, us);
                    if (e == cudaSuccess)
                        e = cudaMemcpyAsync(draw + prob_b + 2 * k * ca, ridx + k * ca, 2 * k * (cb - ca),
                                            cudaMemcpyHostToDevice, us);
                }
                if (pool) pool->wait();
                CK(e);
                CK(cudaEventRecord(ev_hrows, us));
                for (unsigned w = 0; w < nth; ++w) {
                    mm->rows_dup |= dup[w];
                    if (bad[w] >= 0)
                        fail(SGM_ERR_INVALID, "map: semantic index >= channels %d (near gaussian %d)", C, bad[w]);
                }
                // rows sorted by class id (stable) and padded to kpad; their group bounds
                launch_sort_rows(reinterpret_cast<const uint16_t*>(draw + prob_b),
                                 reinterpret_cast<const double*>(draw), n, k, kpad,
                                 mm->idx.as<uint16_t>(), mm->prob.as<double>(), mm->perm.as<uint16_t>(), us);
                launch_group_bounds(mm->dev, mm->groups, mm->gbnd.as<uint4>(), us);
                CK(cudaGetLastError());
                CK(cudaEventRecord(mm->ev_rows, us));
            } catch (const SgmError& err) {
                mm->rows_code = err.code;
                mm->rows_msg = err.msg;
            } catch (const std::exception& err) {
                mm->rows_code = SGM_ERR_INVALID;
                mm->rows_msg = err.what();
            }
        });
        ctx->rows_owner = m;
        *out = m;
        m = nullptr;
    });
    delete m;
    return rc;
}

int sgm_map_wait(sgm_ctx* ctx, sgm_map* map) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map) fail(SGM_ERR_INVALID, "map is null");
        map_ready(ctx, map);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int sgm_map_upload(sgm_ctx* ctx, uint64_t n, int32_t k, int32_t num_classes, const double* centers,
                   const double* log_radii, const double* opacity_logits, const double* colors,
                   const uint16_t* sem_indices, const double* sem_probs, sgm_map** out) {
    int rc = sgm_map_upload_async(ctx, n, k, num_classes, centers, log_radii, opacity_logits, colors,
                                  sem_indices, sem_probs, out);
    if (rc != SGM_OK) return rc;
    rc = sgm_map_wait(ctx, *out);  // the host arrays are no longer read after this
    if (rc != SGM_OK) {
        sgm_map_release(ctx, *out);
        *out = nullptr;
    }
    return rc;
}

void sgm_map_release(sgm_ctx* ctx, sgm_map* map) {
    if (!map) return;
    if (map->rows_pending) {
        map->rows_thread.join();
        map->rows_pending = false;
    }
    if (ctx) {
        if (ctx->rows_owner == map) ctx->rows_owner = nullptr;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->bin_stream);
        if (ctx->up_stream) cudaStreamSynchronize(ctx->up_stream);
        if (ctx->last_map == map) ctx->last_valid = false;
        ctx->give(std::move(map->geo));
        ctx->give(std::move(map->color));
        ctx->give(std::move(map->idx));
        ctx->give(std::move(map->prob));
        ctx->give(std::move(map->perm));
        ctx->give(std::move(map->cov));
        ctx->give(std::move(map->gbnd));
        ctx->give(std::move(map->rec));
    }
    if (map->ev_rows) cudaEventDestroy(map->ev_rows);
    delete map;
}

int sgm_map_set_anisotropic(sgm_ctx* ctx, sgm_map* map, const double* log_scales,
                            const double* quats) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map) fail(SGM_ERR_INVALID, "map is null");
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaStreamSynchronize(ctx->bin_stream));
        if (ctx->last_map == map) ctx->last_valid = false;
        DevMap& d = map->dev;
        if (!log_scales && !quats) {  // back to the isotropic (reference) footprint
            d.aniso = 0;
            d.cov = nullptr;
            return;
        }
        const uint64_t n = d.n;
        if (n > 0 && (!log_scales || !quats)) fail(SGM_ERR_INVALID, "anisotropic: null array with n > 0");
        const size_t ns = std::max<uint64_t>(n, 1);
        CK(ctx->h_stage.reserve(8 * 6 * ns));
        double* cov = ctx->h_stage.as<double>();
        std::vector<int> bad(1, -1);
        // Sigma = R(q) diag(exp(ls))^2 R(q)^T, left-to-right evaluation with one rounding
        // per operation (-ffp-contract=off); oracle/sgm_oracle.c orc_cov3 states the same
        // order, so both sides project identical covariances.
        for (uint64_t i = 0; i < n; ++i) {
            const double* q4 = quats + 4 * i;
            const double nrm = std::sqrt(((q4[0] * q4[0] + q4[1] * q4[1]) + q4[2] * q4[2]) + q4[3] * q4[3]);
            if (!(nrm > 0.0) || !std::isfinite(nrm)) {
                bad[0] = static_cast<int>(i % 0x7fffffff);
                break;
            }
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
            const double s0 = std::exp(log_scales[3 * i]), s1 = std::exp(log_scales[3 * i + 1]),
                         s2 = std::exp(log_scales[3 * i + 2]);
            const double v0 = s0 * s0, v1 = s1 * s1, v2 = s2 * s2;
            static const int I[6] = {0, 0, 0, 1, 1, 2}, J[6] = {0, 1, 2, 1, 2, 2};
            for (int e = 0; e < 6; ++e) {
                const double* a = R + 3 * I[e];
                const double* b = R + 3 * J[e];
                cov[e * n + i] = ((a[0] * b[0]) * v0 + (a[1] * b[1]) * v1) + (a[2] * b[2]) * v2;
            }
        }
        if (bad[0] >= 0) fail(SGM_ERR_INVALID, "anisotropic: zero or non-finite quaternion (gaussian %d)", bad[0]);
        ctx->take(map->cov, 8 * 6 * ns);
        CK(map->cov.reserve(8 * 6 * ns));
        CK(cudaMemcpyAsync(map->cov.p, cov, 8 * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        d.cov = map->cov.as<double>();
        d.aniso = 1;
    });
}

int sgm_render_device(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam, const sgm_pose* pose,
                      uint32_t channels, const sgm_options* opt, double* d_color, double* d_depth,
                      double* d_sil, double* d_sem, uint64_t* n_projections) {
    return guard(ctx, [&] {
        if (!d_sil) fail(SGM_ERR_INVALID, "silhouette plane is required");
        do_render(ctx, map, cam, pose, channels, opt, d_color, d_depth, d_sil, d_sem, n_projections);
    });
}


// render() / render_reference() into caller-owned host planes (reference layout)
static int render_to_host(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera,
                          const sgm_pose* pose, uint32_t channels, const sgm_options* opt,
                          double* color, double* depth, double* silhouette, double* sem,
                          uint64_t* n_projections, bool reference_form) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map) fail(SGM_ERR_INVALID, "map is null");
        const CamParams cam = to_cam(camera);
        if (!silhouette) fail(SGM_ERR_INVALID, "silhouette plane is required");
        const size_t px = static_cast<size_t>(cam.W) * cam.H;
        const size_t C = static_cast<size_t>(map->dev.C);
        const bool want_c = (channels & SGM_COLOR) && color;
        const bool want_d = (channels & SGM_DEPTH) && depth;
        const bool want_s = (channels & SGM_SEMANTICS) && sem;
        const size_t need = px * (1 + (want_c ? 3 : 0) + (want_d ? 1 : 0) + (want_s ? C : 0));
        CK(ctx->planes.reserve(8 * need));
        double* base = ctx->planes.as<double>();
        double* d_sil = base;
        double* d_color = want_c ? d_sil + px : nullptr;
        double* d_depth = want_d ? (want_c ? d_color + 3 * px : d_sil + px) : nullptr;
        double* d_sem = want_s ? base + px * (1 + (want_c ? 3 : 0) + (want_d ? 1 : 0)) : nullptr;
        uint32_t ch = (want_c ? SGM_COLOR : 0u) | (want_d ? SGM_DEPTH : 0u) |
                      (want_s ? SGM_SEMANTICS : 0u) | (channels & SGM_RETAIN_CONTRIBUTORS);
        do_render(ctx, map, camera, pose, ch, opt, d_color, d_depth, d_sil, d_sem, n_projections,
                  reference_form);
        std::vector<CopyOut> segs{{silhouette, d_sil, 8 * px}};
        if (want_c) segs.push_back({color, d_color, 24 * px});
        if (want_d) segs.push_back({depth, d_depth, 8 * px});
        if (want_s) segs.push_back({sem, d_sem, 8 * px * C});
        copy_out(ctx, segs);
        // Unrequested-but-provided planes: the reference leaves them empty; zero them.
        if ((channels & SGM_COLOR) == 0 && color) std::memset(color, 0, 24 * px);
        if ((channels & SGM_DEPTH) == 0 && depth) std::memset(depth, 0, 8 * px);
    });
}

int sgm_render(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera, const sgm_pose* pose,
               uint32_t channels, const sgm_options* opt, double* color, double* depth,
               double* silhouette, double* sem, uint64_t* n_projections) {
    return render_to_host(ctx, map, camera, pose, channels, opt, color, depth, silhouette, sem,
                          n_projections, false);
}

// render_reference (splat_render.cpp:330-358): default RenderOptions with early_exit = false,
// every projection composited in depth order with composite_pixel's footprint (:86-92).
int sgm_render_reference(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera,
                         const sgm_pose* pose, uint32_t channels, double* color, double* depth,
                         double* silhouette, double* sem, uint64_t* n_projections) {
    const sgm_options o{0, 1e-4, 0.01, 3.0, 8};  // RenderOptions{} with early_exit = false (:333-334)
    return render_to_host(ctx, map, camera, pose, channels, &o, color, depth, silhouette, sem,
                          n_projections, true);
}

int sgm_last_projections(sgm_ctx* ctx, sgm_projection* out, uint64_t capacity) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!ctx->last_valid) fail(SGM_ERR_INVALID, "no render state (call sgm_render first)");
        const uint32_t V = ctx->last_V;
        if (capacity < V) fail(SGM_ERR_INVALID, "capacity %llu < %u projections",
                               static_cast<unsigned long long>(capacity), V);
        if (V == 0) return;
        CK(ctx->dbg.reserve(48ull * V + 96));
        PoseParams* dpose = reinterpret_cast<PoseParams*>(ctx->dbg.as<char>() + 48ull * V);
        CK(cudaMemcpyAsync(dpose, &ctx->last_pose, sizeof(PoseParams), cudaMemcpyHostToDevice, ctx->stream));
        launch_debug_projections(ctx->last_map->dev, dpose, ctx->last_cam, ctx->last_opt,
                                 ctx->vals.as<uint32_t>(), V, ctx->dbg.as<double>(), ctx->stream);
        std::vector<double> h(6ull * V);
        CK(cudaMemcpyAsync(h.data(), ctx->dbg.p, 48ull * V, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (uint32_t r = 0; r < V; ++r) {
            out[r].mx = h[6 * r];
            out[r].my = h[6 * r + 1];
            out[r].rad_px = h[6 * r + 2];
            out[r].z = h[6 * r + 3];
            out[r].alpha = h[6 * r + 4];
            out[r].index = static_cast<uint32_t>(h[6 * r + 5]);
            out[r].reserved = 0;
        }
    });
}

int sgm_last_bins(sgm_ctx* ctx, uint32_t* tile_offsets, uint32_t* ids, float* probe3,
                  uint64_t capacity, uint64_t* n_pairs) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!ctx->last_valid) fail(SGM_ERR_INVALID, "no render state (call sgm_render first)");
        const uint64_t P = ctx->last_P;
        if (n_pairs) *n_pairs = P;
        const int tiles = ctx->last_bin_tiles;
        if (tile_offsets) {
            std::vector<uint2> r(tiles);
            CK(cudaMemcpy(r.data(), ctx->ranges.p, sizeof(uint2) * tiles, cudaMemcpyDeviceToHost));
            uint64_t acc = 0;
            for (int t = 0; t < tiles; ++t) {
                tile_offsets[t] = static_cast<uint32_t>(acc);
                acc += r[t].y - r[t].x;
            }
            tile_offsets[tiles] = static_cast<uint32_t>(acc);
        }
        if ((ids || probe3) && P) {
            if (capacity < P) fail(SGM_ERR_INVALID, "capacity < %llu pairs", static_cast<unsigned long long>(P));
            CK(ctx->dbg.reserve(16 * P));
            uint32_t* d_ids = ctx->dbg.as<uint32_t>();
            float* d_probe = reinterpret_cast<float*>(ctx->dbg.as<char>() + 4 * P);
            launch_bins_to_ids(ctx->tvals.as<uint32_t>(), P, ctx->packed.as<PackedSplat>(),
                               ctx->last_map->dev.aniso, ctx->last_opt.cut_sq, d_ids, d_probe,
                               ctx->stream);
            if (ids) CK(cudaMemcpyAsync(ids, d_ids, 4 * P, cudaMemcpyDeviceToHost, ctx->stream));
            if (probe3) CK(cudaMemcpyAsync(probe3, d_probe, 12 * P, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
    });
}

int sgm_last_contributors(sgm_ctx* ctx, uint32_t* offsets, uint32_t* contrib, uint64_t capacity,
                          uint64_t* n_contrib) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!ctx->last_valid || !ctx->last_has_contrib)
            fail(SGM_ERR_INVALID, "no retained contributors (render with SGM_RETAIN_CONTRIBUTORS)");
        const uint64_t total = ctx->last_ncontrib;
        if (n_contrib) *n_contrib = total;
        const size_t px = static_cast<size_t>(ctx->last_px);
        if (offsets) {
            std::vector<unsigned long long> off(px + 1);
            CK(cudaMemcpyAsync(off.data(), ctx->coffset.p, 8 * (px + 1), cudaMemcpyDeviceToHost,
                               ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            for (size_t i = 0; i <= px; ++i) offsets[i] = static_cast<uint32_t>(off[i]);
        }
        if (contrib && total) {
            if (capacity < total) fail(SGM_ERR_INVALID, "capacity < %llu contributors",
                                       static_cast<unsigned long long>(total));
            CK(cudaMemcpyAsync(contrib, ctx->contrib.p, 4 * total, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
    });
}

int sgm_render_entropy(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera,
                       const sgm_pose* pose, const sgm_options* opt, double* entropy) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map || !entropy) fail(SGM_ERR_INVALID, "null argument");
        const CamParams cam = to_cam(camera);
        const size_t px = static_cast<size_t>(cam.W) * cam.H;
        const size_t C = static_cast<size_t>(map->dev.C);
        std::vector<double> sil(px), sem(px * C);
        uint64_t nproj = 0;
        int rc = sgm_render(ctx, map, camera, pose, SGM_SEMANTICS, opt, nullptr, nullptr, sil.data(),
                            sem.data(), &nproj);
        if (rc != SGM_OK) fail(rc, "%s", ctx->err.c_str());
        for (size_t i = 0; i < px; ++i) entropy[i] = sgm_clipped_entropy(&sem[i * C], C);
    });
}

int sgm_score_views(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera, uint64_t n,
                    const sgm_pose* poses, const sgm_options* opt, double* n_missing,
                    double* entropy_sum) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map) fail(SGM_ERR_INVALID, "map is null");
        if (n == 0) return;
        if (!poses || !n_missing || !entropy_sum) fail(SGM_ERR_INVALID, "null argument");
        const CamParams cam = to_cam(camera);
        const OptParams o = to_opt(opt, cam);
        std::vector<PoseParams> pp(n);
        for (uint64_t i = 0; i < n; ++i) pp[i] = to_pose(poses[i]);
        run_views(ctx, map, cam, o, n, pp.data(), Mode::Score, RenderTargets{}, n_missing,
                  entropy_sum);
    });
}

int sgm_fisher_prior(sgm_ctx* ctx, sgm_map* map, const sgm_camera* camera, uint64_t n,
                     const sgm_pose* poses, const sgm_options* opt, double lambda, double* H_out) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map) fail(SGM_ERR_INVALID, "map is null");
        if (map->dev.aniso)
            fail(SGM_ERR_UNSUPPORTED, "the Fisher / backward chain is isotropic only (anisotropic map)");
        if (n > 0 && !poses) fail(SGM_ERR_INVALID, "poses are null");
        if (!(lambda > 0.0)) fail(SGM_ERR_INVALID, "lambda must be > 0");
        const CamParams cam = to_cam(camera);
        const OptParams o = to_opt(opt, cam);
        const size_t nh = 8 * std::max<uint64_t>(map->dev.n, 1);
        CK(map->fisher_H.reserve(8 * nh));
        CK(map->fisher_invp.reserve(8 * nh));
        CK(cudaMemsetAsync(map->fisher_H.p, 0, 8 * nh, ctx->stream));
        std::vector<PoseParams> pp(n);
        for (uint64_t i = 0; i < n; ++i) pp[i] = to_pose(poses[i]);
        if (n) run_views(ctx, map, cam, o, n, pp.data(), Mode::Score, RenderTargets{}, nullptr, nullptr,
                         Fisher::Prior, nullptr, map->fisher_H.as<double>());
        launch_fisher_invp(map->fisher_H.as<double>(), lambda, 8 * map->dev.n, map->fisher_invp.as<double>(),
                           ctx->stream);
        ctx->stats.kernel_launches += 1;
        if (H_out && map->dev.n)
            CK(cudaMemcpyAsync(H_out, map->fisher_H.p, 64 * map->dev.n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        map->has_prior = true;
    });
}

int sgm_fisher_set_prior(sgm_ctx* ctx, sgm_map* map, const double* H, double lambda) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map) fail(SGM_ERR_INVALID, "map is null");
        if (map->dev.aniso)
            fail(SGM_ERR_UNSUPPORTED, "the Fisher / backward chain is isotropic only (anisotropic map)");
        if (map->dev.n > 0 && !H) fail(SGM_ERR_INVALID, "H is null");
        if (!(lambda > 0.0)) fail(SGM_ERR_INVALID, "lambda must be > 0");
        const size_t nh = 8 * std::max<uint64_t>(map->dev.n, 1);
        CK(map->fisher_H.reserve(8 * nh));
        CK(map->fisher_invp.reserve(8 * nh));
        if (map->dev.n)
            CK(cudaMemcpyAsync(map->fisher_H.p, H, 64 * map->dev.n, cudaMemcpyHostToDevice, ctx->stream));
        launch_fisher_invp(map->fisher_H.as<double>(), lambda, 8 * map->dev.n,
                           map->fisher_invp.as<double>(), ctx->stream);
        ctx->stats.kernel_launches += 1;
        CK(cudaStreamSynchronize(ctx->stream));
        map->has_prior = true;
    });
}

int sgm_score_views_fisher(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera, uint64_t n,
                           const sgm_pose* poses, const sgm_options* opt, double* n_missing,
                           double* entropy_sum, double* fisher_gain) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map) fail(SGM_ERR_INVALID, "map is null");
        if (map->dev.aniso)
            fail(SGM_ERR_UNSUPPORTED, "the Fisher / backward chain is isotropic only (anisotropic map)");
        if (!map->has_prior) fail(SGM_ERR_INVALID, "no Fisher prior (call sgm_fisher_prior first)");
        if (n == 0) return;
        if (!poses || !n_missing || !entropy_sum || !fisher_gain) fail(SGM_ERR_INVALID, "null argument");
        const CamParams cam = to_cam(camera);
        const OptParams o = to_opt(opt, cam);
        std::vector<PoseParams> pp(n);
        for (uint64_t i = 0; i < n; ++i) pp[i] = to_pose(poses[i]);
        run_views(ctx, map, cam, o, n, pp.data(), Mode::Score, RenderTargets{}, n_missing, entropy_sum,
                  Fisher::Gain, fisher_gain, nullptr);
    });
}

int sgm_backward(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera, const sgm_pose* pose,
                 const sgm_options* opt, const float* rgb, const float* depth, const float* sem,
                 const double weights[7], int include_mapping, int include_semantic,
                 double report[7], double* g_center, double* g_log_radius,
                 double* g_opacity_logit, double* g_color, double* g_sem) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map || !pose || !rgb || !depth || !sem || !weights || !report)
            fail(SGM_ERR_INVALID, "null argument");
        if (map->dev.aniso)
            fail(SGM_ERR_UNSUPPORTED, "the Fisher / backward chain is isotropic only (anisotropic map)");
        const CamParams cam = to_cam(camera);
        const OptParams o = to_opt(opt, cam);
        const PoseParams p = to_pose(*pose);
        cudaStream_t s = ctx->stream;
        const size_t px = static_cast<size_t>(cam.W) * cam.H;
        const int C = map->dev.C, k = map->dev.k;
        const uint64_t N = map->dev.n;
        const size_t NS = std::max<uint64_t>(N, 1);
        CK(ctx->bw_frame.reserve(4 * px * (4 + C) + 16));
        float* f_rgb = ctx->bw_frame.as<float>();
        float* f_depth = f_rgb + 3 * px;
        float* f_sem = f_depth + px;
        CK(cudaMemcpyAsync(f_rgb, rgb, 12 * px, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(f_depth, depth, 4 * px, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(f_sem, sem, 4 * px * C, cudaMemcpyHostToDevice, s));
        backward_core(ctx, map, cam, o, p, f_rgb, f_depth, f_sem, weights, include_mapping,
                      include_semantic, report);
        const double* g = ctx->bw_grad.as<double>();
        if (N) {
            if (g_center) CK(cudaMemcpyAsync(g_center, g, 24 * N, cudaMemcpyDeviceToHost, s));
            if (g_log_radius) CK(cudaMemcpyAsync(g_log_radius, g + 3 * NS, 8 * N, cudaMemcpyDeviceToHost, s));
            if (g_opacity_logit) CK(cudaMemcpyAsync(g_opacity_logit, g + 4 * NS, 8 * N, cudaMemcpyDeviceToHost, s));
            if (g_color) CK(cudaMemcpyAsync(g_color, g + 5 * NS, 24 * N, cudaMemcpyDeviceToHost, s));
            if (g_sem) CK(cudaMemcpyAsync(g_sem, g + 8 * NS, 8 * N * k, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    });
}

int sgm_score_candidates(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* cam, uint64_t n,
                         const sgm_candidate* cands, const sgm_options* opt, double* n_missing,
                         double* entropy_sum) {
    if (n > 0 && !cands) {
        if (ctx) ctx->err = "candidates are null";
        return SGM_ERR_INVALID;
    }
    std::vector<sgm_pose> poses(n);
    for (uint64_t i = 0; i < n; ++i) sgm_candidate_pose(cands[i].position, cands[i].direction, &poses[i]);
    return sgm_score_views(ctx, map, cam, n, poses.data(), opt, n_missing, entropy_sum);
}

}  // extern "C"
