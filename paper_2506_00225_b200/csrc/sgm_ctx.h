// Host-side internals shared by the C-ABI translation units (sgm_capi.cu, sgm_capi_ext.cu)
// and the view pipeline (sgm_pipeline.cu): device / pinned buffers, the error plumbing
// behind the status codes, the opaque sgm_map / sgm_ctx, and the pipeline entry points.
#pragma once

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sgm.h"
#include "sgm_internal.h"

namespace sgm {


// Persistent host workers for the map upload's staging (spawning 16 threads per upload cost
// about 0.3 ms per phase on the bench host). start(n, fn) runs fn(0) .. fn(n - 1) on n
// workers and returns at once; wait() blocks until they are done. One job at a time.
class HostPool {
public:
    explicit HostPool(unsigned n) {
        for (unsigned w = 0; w < n; ++w) th_.emplace_back([this, w] { loop(w); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    unsigned size() const { return static_cast<unsigned>(th_.size()); }
    void start(unsigned n, std::function<void(unsigned)> fn) {
        {
            std::lock_guard<std::mutex> g(mu_);
            fn_ = std::move(fn);
            active_ = std::min<unsigned>(n, size());
            left_ = active_;
            ++gen_;
        }
        cv_.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> g(mu_);
        done_cv_.wait(g, [this] { return left_ == 0; });
    }

private:
    void loop(unsigned w) {
        uint64_t seen = 0;
        for (;;) {
            std::function<void(unsigned)> fn;
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                if (w >= active_) continue;
                fn = fn_;
            }
            fn(w);
            std::lock_guard<std::mutex> g(mu_);
            if (--left_ == 0) done_cv_.notify_all();
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::function<void(unsigned)> fn_;
    unsigned active_ = 0, left_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
        o.p = nullptr;
        o.bytes = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            if (p) cudaFree(p);
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    // Grows (never shrinks); contents are not preserved.
    cudaError_t reserve(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        // 1/8 headroom: per-view sizes vary, so exact-size growth would reallocate often
        const size_t b = std::max<size_t>(want + want / 8, 256);
        cudaError_t e = cudaMalloc(&p, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    cudaError_t reserve(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMallocHost(&p, std::max<size_t>(want, 256));
        if (e == cudaSuccess) bytes = std::max<size_t>(want, 256);
        return e;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct SgmError {
    int code;
    std::string msg;
};

[[noreturn]] inline void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    throw SgmError{code, buf};
}

// Fails with SGM_ERR_UNSUPPORTED when a kernel's shared-memory layout (which grows with the
// channel count: the per-block fp64 accumulator) exceeds the device's per-block limit.
inline void need_smem(int device, size_t bytes, int channels, const char* what) {
    int lim = 0;
    cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (lim > 0 && bytes > static_cast<size_t>(lim))
        fail(SGM_ERR_UNSUPPORTED, "%s: %d semantic channels need %zu B of shared memory per block "
             "(device limit %d B)", what, channels, bytes, lim);
}

#define CK(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            fail(e_ == cudaErrorMemoryAllocation ? SGM_ERR_OOM : SGM_ERR_CUDA,         \
                 "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,     \
                 __LINE__);                                                            \
    } while (0)


}  // namespace sgm

using namespace sgm;

struct sgm_map {
    DevMap dev;
    GroupParams groups{1, 1};
    int num_classes = 0;
    DevBuf fisher_H, fisher_invp;  // Fisher prior (sgm_fisher_prior)
    bool has_prior = false;
    DevBuf geo;    // cx, cy, cz, rad, alpha (5 x n doubles)
    DevBuf color;  // [n][4]
    DevBuf idx;    // [n][kpad] u16 (class-sorted)
    DevBuf prob;   // [n][kpad] f64
    DevBuf perm;   // [n][kpad] u16 original entry index
    DevBuf cov;    // anisotropic mode: [6][n] world covariance (sgm_map_set_anisotropic)
    DevBuf gbnd;   // [n] uint4: class-sorted rows' channel-group bounds (DevMap::gbounds)
    DevBuf rec;    // [n][kpad] uint4: DevMap::sem_rec (map_records), valid while rec_valid
    bool rec_valid = false;  // cleared wherever sem_prob / sem_idx change
    // Upload split in two (sgm_map_upload): the geometry is staged and copied on the ctx
    // stream before the call returns; the colours and semantic rows are staged by
    // rows_thread and copied / sorted on the ctx's upload stream, ending at ev_rows. The
    // first use of the rows (the raster) waits for both (map_ready).
    std::thread rows_thread;
    bool rows_pending = false;
    int rows_code = 0;
    int rows_dup = 0;  // phase B found a Gaussian listing a class twice (DevMap::dup_idx)
    std::string rows_msg;
    cudaEvent_t ev_rows = nullptr;
};

struct sgm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    sgm_stats stats{};
    bool profiling = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaStream_t bin_stream = nullptr;  // binning of the next sub-batch overlaps the raster
    cudaStream_t up_stream = nullptr;   // map uploads: colours / semantic rows (sgm_map_upload)
    sgm_map* rows_owner = nullptr;      // the map whose rows_thread uses h_rows
    uint64_t list_budget = uint64_t(2) << 30;  // u32 tile-list entries per group of views
    std::unique_ptr<HostPool> workers;  // upload staging workers (created on the first large upload)
    cudaEvent_t ev_hstage = nullptr;    // the last copy out of h_stage (geometry) / h_rows
    cudaEvent_t ev_hrows = nullptr;
    cudaEvent_t ev_ready = nullptr;
    cudaEvent_t ev_binned[2] = {nullptr, nullptr};
    cudaEvent_t ev_r[32] = {};  // raster start/stop pairs of one group (profiling)

    // scratch
    DevBuf poses, vcount, pcount, keys, vals, keys_alt, vals_alt, packed, counts, offsets, rects,
        bounds, bdiff, rranges, rvals, segs, segcnt, rcbuf;
    DevBuf tkeys, tvals, tkeys_alt, tvals_alt, ranges, ent_part, miss_part, views, out,
        contributors, cub_tmp, sort_tmp, scan_tmp, franges, trunc8, bmask, incomplete, redo,
        dense_tot, list2, cdiff, csat, planes, dbg, ccount, coffset, contrib, fis_part, bw_frame,
        bw_flags, bw_part, bw_grad;
    uint64_t last_ncontrib = 0;
    bool last_has_contrib = false;
    int last_px = 0;
    HostBuf h_counts, h_views, h_poses, h_out, h_stage, h_rows, h_ring;
    cudaEvent_t ev_ring[4] = {nullptr, nullptr, nullptr, nullptr};  // copy_out pinned ring
    DevBuf upload_tmp;
    // device buffers of released maps, reused by the next upload (a map version bump
    // otherwise pays cudaFree + cudaMalloc of ~0.2 KB per Gaussian)
    std::vector<DevBuf> pool;

    void take(DevBuf& dst, size_t want) {
        if (dst.bytes >= want) return;
        size_t best = pool.size();
        for (size_t i = 0; i < pool.size(); ++i)
            if (pool[i].bytes >= want && (best == pool.size() || pool[i].bytes < pool[best].bytes))
                best = i;
        if (best == pool.size()) return;
        dst = std::move(pool[best]);
        pool.erase(pool.begin() + static_cast<long>(best));
    }
    void give(DevBuf&& b) {
        if (!b.p) return;
        pool.push_back(std::move(b));
        while (pool.size() > 16) pool.erase(pool.begin());  // bounded: oldest first
    }

    // state of the last render (for sgm_last_*)
    bool last_valid = false;
    uint32_t last_V = 0;
    uint64_t last_P = 0;
    int last_bin_tiles = 0;
    const sgm_map* last_map = nullptr;
    CamParams last_cam{};
    OptParams last_opt{};
    PoseParams last_pose{};
};

namespace sgm {

// The map's semantic rows (and colours, group bounds) are on the device: joins the upload's
// staging thread (failing with its error) and makes the ctx stream wait for the rows' copies.
void map_ready(sgm_ctx* ctx, const sgm_map* map);
// Channel-group bounds of a map whose rows are sorted on the device (stream s).
void map_group_bounds(sgm_ctx* ctx, sgm_map* map, cudaStream_t s);
// builds DevMap::sem_rec on ctx->stream unless still valid (after map_ready)
void map_records(sgm_ctx* ctx, const sgm_map* map);
CamParams to_cam(const sgm_camera* c);
OptParams to_opt(const sgm_options* o, const CamParams& cam);
PoseParams to_pose(const sgm_pose& p);
// runs fn, mapping SgmError / CUDA / allocation failures to status codes and ctx->err
int guard(sgm_ctx* ctx, const std::function<void()>& fn);
void need_ctx(sgm_ctx* ctx);
unsigned tile_bits(uint64_t tiles);

enum class Mode { Score, Render };
enum class Fisher { None, Prior, Gain };

struct RenderTargets {
    double* color = nullptr;
    double* depth = nullptr;
    double* sil = nullptr;
    double* sem = nullptr;
    uint32_t channels = 0;
    uint32_t* contrib = nullptr;            // retain_contributors
    uint32_t* contrib_count = nullptr;      // pass 1
    const unsigned long long* contrib_offset = nullptr;  // pass 2
};

// Runs n views. Score mode writes n_missing/entropy_sum (host); render mode (n == 1)
// writes planes to device targets. Binning of sub-batch i+1 (on ctx->bin_stream)
// overlaps the raster of sub-batch i (on ctx->stream).
void run_views(sgm_ctx* ctx, const sgm_map* map, const CamParams& cam, const OptParams& o,
               uint64_t n, const PoseParams* poses, Mode mode, const RenderTargets& rt,
               double* h_missing, double* h_entropy, Fisher fk = Fisher::None,
               double* h_fisher = nullptr, double* d_H = nullptr);
// One render into device planes (retain_contributors: two raster passes).
void do_render(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera, const sgm_pose* pose,
               uint32_t channels, const sgm_options* opt, double* d_color, double* d_depth,
               double* d_sil, double* d_sem, uint64_t* n_proj, bool reference_form = false);
// The mapping step on device-resident frame planes (see sgm_pipeline.cu).
void backward_core(sgm_ctx* ctx, const sgm_map* map, const CamParams& cam, const OptParams& o,
                   const PoseParams& p, const float* f_rgb, const float* f_depth,
                   const float* f_sem, const double weights[7], int include_mapping,
                   int include_semantic, double report[7]);

struct CopyOut {
    void* dst;        // host (pageable) destination
    const void* src;  // device source
    size_t bytes;
};
void copy_out(sgm_ctx* ctx, const std::vector<CopyOut>& segs);

}  // namespace sgm
