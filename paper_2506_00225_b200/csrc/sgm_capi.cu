// C ABI (include/sgm.h) and the host pipeline that drives the sm_100a kernels.
//
// Pipeline for a batch of views (all on the ctx stream):
//   1. K1 k_preprocess over (Gaussian, view): compact visible (z, index), count V, P and
//      the row pairs R (tile rows spanned)
//   2. one D2H of the per-view V/P/R counts (the only host sync before the results)
//   3. per view (binning stream): CUB radix sort on fp32(z) -> k_tiefix -> k_pack ->
//      k_bin_hist + k_bin_scan (tile ranges) -> k_emit_rows + CUB stable row sort ->
//      k_row_segs / k_seg_pass x2 / k_seg_scan (ordered scatter into the tile lists)
//   4. one batched raster launch over (8x8 tile, view)
//   5. k_reduce_scores (score) / planes already written (render)
// Views whose pair lists do not fit the scratch budget together are split into
// sub-batches; results do not depend on the split (per-view work is independent).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sgm.h"
#include "sgm_internal.h"

using namespace sgm;

namespace {

thread_local std::string g_create_error;

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

[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    throw SgmError{code, buf};
}

#define CK(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            fail(e_ == cudaErrorMemoryAllocation ? SGM_ERR_OOM : SGM_ERR_CUDA,         \
                 "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,     \
                 __LINE__);                                                            \
    } while (0)

}  // namespace

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
};

struct sgm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    sgm_stats stats{};
    bool profiling = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaStream_t bin_stream = nullptr;  // binning of the next sub-batch overlaps the raster
    cudaEvent_t ev_ready = nullptr;
    cudaEvent_t ev_binned[2] = {nullptr, nullptr};
    cudaEvent_t ev_r[16] = {};  // raster start/stop pairs of one group (profiling)

    // scratch
    DevBuf poses, vcount, pcount, keys, vals, keys_alt, vals_alt, packed, counts, offsets, rects,
        bounds, bdiff, rranges, rvals, segs, segcnt, rcbuf;
    DevBuf tkeys, tvals, tkeys_alt, tvals_alt, ranges, ent_part, miss_part, views, out,
        contributors, cub_tmp, planes, dbg, ccount, coffset, contrib, fis_part, bw_frame,
        bw_flags, bw_part, bw_grad;
    uint64_t last_ncontrib = 0;
    bool last_has_contrib = false;
    int last_px = 0;
    HostBuf h_counts, h_views, h_poses, h_out, h_stage, h_ring;
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

namespace {

CamParams to_cam(const sgm_camera* c) {
    if (!c) fail(SGM_ERR_INVALID, "camera is null");
    if (c->width <= 0 || c->height <= 0) fail(SGM_ERR_INVALID, "camera: resolution must be positive");
    return CamParams{c->width, c->height, c->fx, c->fy, c->cx, c->cy};
}

OptParams to_opt(const sgm_options* o, const CamParams& cam) {
    sgm_options d{1, 1e-4, 0.01, 3.0, 8};
    const sgm_options& s = o ? *o : d;
    if (s.tile_size <= 0 || s.tile_size % kTile != 0)
        fail(SGM_ERR_UNSUPPORTED, "tile_size %d: this build bins at multiples of %d", s.tile_size,
             kTile);
    OptParams p;
    p.early_exit = s.early_exit ? 1 : 0;
    p.eps = s.transmittance_eps;
    p.z_near = s.z_near;
    p.trunc = s.truncation_sigmas;
    p.cut_sq = s.truncation_sigmas * s.truncation_sigmas;
    p.ts = s.tile_size;
    p.tiles_x = (cam.W + s.tile_size - 1) / s.tile_size;
    p.tiles_y = (cam.H + s.tile_size - 1) / s.tile_size;
    return p;
}

PoseParams to_pose(const sgm_pose& p) {
    PoseParams q;
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) q.Rcw[3 * i + k] = p.R[3 * k + i];  // R_cw = R^T
    for (int i = 0; i < 3; ++i) q.t[i] = p.t[i];
    return q;
}

int guard(sgm_ctx* ctx, const std::function<void()>& fn);

unsigned tile_bits(uint64_t tiles) {
    unsigned b = 1;
    while ((1ull << b) < tiles) ++b;
    return b;
}

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

// Bins one view (step 3). Writes ranges / sorted list / packed into the per-view
// slices and returns via the slice pointers. vals/keys hold the compacted (z, idx).
void bin_view(sgm_ctx* ctx, cudaStream_t s, const sgm_map* map, const CamParams& cam,
              const OptParams& o, const PoseParams* d_pose, uint32_t* keys, uint32_t* vals,
              uint32_t V, uint64_t P, uint64_t R, PackedSplat* packed, uint4* bounds, uint32_t* list,
              uint2* ranges, int bin_tiles) {
    CK(cudaMemsetAsync(ranges, 0, sizeof(uint2) * bin_tiles, s));
    if (V == 0) return;
    // K2: depth rank (radix sort on the monotone fp32 key; runs fixed below)
    cub::DoubleBuffer<uint32_t> dk(keys, ctx->keys_alt.as<uint32_t>());
    cub::DoubleBuffer<uint32_t> dv(vals, ctx->vals_alt.as<uint32_t>());
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, V, 0, 32, s));
    CK(ctx->cub_tmp.reserve(tmp));
    CK(cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.p, tmp, dk, dv, V, 0, 32, s));
    ctx->stats.kernel_launches += 1;  // counted as one library sort call
    launch_tiefix(map->dev, d_pose, cam, o, dk.Current(), dv.Current(), V, s);
    launch_pack(map->dev, d_pose, cam, o, map->groups, dv.Current(), V, packed,
                ctx->counts.as<unsigned long long>(), ctx->rects.as<int4>(), bounds, s);
    ctx->stats.kernel_launches += (V >= 2 ? 1 : 0) + 1;
    // keep the sorted indices for sgm_last_projections
    if (dv.Current() != vals) CK(cudaMemcpyAsync(vals, dv.Current(), 4ull * V, cudaMemcpyDeviceToDevice, s));
    if (P == 0) return;
    // K3 (row-bucketed, no sort of the P pairs): tile ranges from the rectangles' 2D
    // difference array; each tile row's ranks in rank order (R = sum of rows spanned pairs,
    // stably sorted by row); then one CTA per tile row scatters its ranks into the tile lists
    // in rank order (sgm_kernels.cu)
    const int X = o.tiles_x + 1, Y = o.tiles_y + 1;
    int* diff = ctx->bdiff.as<int>();
    CK(cudaMemsetAsync(diff, 0, sizeof(int) * X * Y, s));
    unsigned long long* rows = ctx->counts.as<unsigned long long>();
    unsigned long long* roff = ctx->offsets.as<unsigned long long>();
    launch_bin_hist(ctx->rects.as<int4>(), V, o.tiles_x, diff, rows, s);
    launch_bin_scan(diff, o.tiles_x, o.tiles_y, ranges, s);
    CK(cudaMemsetAsync(rows + V, 0, sizeof(unsigned long long), s));
    size_t tmp2 = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, rows, roff, V + 1, s));
    CK(ctx->cub_tmp.reserve(tmp2));
    CK(cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, tmp2, rows, roff, V + 1, s));
    uint32_t* rk = ctx->tkeys.as<uint32_t>();
    unsigned long long* rv = ctx->rvals.as<unsigned long long>();
    launch_emit_rows(roff, ctx->rects.as<int4>(), V, R, rk, rv, s);
    cub::DoubleBuffer<uint32_t> qk(rk, ctx->tkeys_alt.as<uint32_t>());
    cub::DoubleBuffer<unsigned long long> qv(rv, ctx->tvals_alt.as<unsigned long long>());
    tmp2 = 0;
    const int rbits = static_cast<int>(tile_bits(static_cast<uint64_t>(o.tiles_y)));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, qk, qv, R, 0, rbits, s));
    CK(ctx->cub_tmp.reserve(tmp2));
    CK(cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.p, tmp2, qk, qv, R, 0, rbits, s));
    uint2* rranges = ctx->rranges.as<uint2>();
    CK(cudaMemsetAsync(rranges, 0, sizeof(uint2) * o.tiles_y, s));
    launch_ranges(qk.Current(), R, rranges, s);
    const uint64_t G = row_scatter_segments(R, o.tiles_y);  // buffers sized per group (run_views)
    launch_row_scatter(qv.Current(), rranges, ranges, o.tiles_x, o.tiles_y, R,
                       ctx->segs.as<uint4>(), reinterpret_cast<uint32_t*>(ctx->segs.as<char>() + sizeof(uint4) * G),
                       ctx->segcnt.as<uint32_t>(), list, s);
    ctx->stats.kernel_launches += 7;
}

// Runs n views. Score mode writes n_missing/entropy_sum (host); render mode (n == 1)
// writes planes to device targets. Binning of sub-batch i+1 (on ctx->bin_stream)
// overlaps the raster of sub-batch i (on ctx->stream).
void run_views(sgm_ctx* ctx, const sgm_map* map, const CamParams& cam, const OptParams& o,
               uint64_t n, const PoseParams* poses, Mode mode, const RenderTargets& rt,
               double* h_missing, double* h_entropy, Fisher fk = Fisher::None,
               double* h_fisher = nullptr, double* d_H = nullptr) {
    cudaStream_t s = ctx->stream;
    cudaStream_t sb = ctx->bin_stream;
    const uint64_t N = map->dev.n;
    const int bin_tiles = o.tiles_x * o.tiles_y;
    const int rtx = (cam.W + kTile - 1) / kTile;
    const int rty = (cam.H + kTile - 1) / kTile;
    const int rtiles = rtx * rty;
    ctx->last_valid = false;

    // batch size bounded by a scratch budget for the per-view N-sized arrays
    const size_t per_view = std::max<uint64_t>(N, 1) * (4 + 4 + sizeof(PackedSplat) + 16) +
                            static_cast<size_t>(bin_tiles) * sizeof(uint2) +
                            static_cast<size_t>(rtiles) * 12 + 256;
    const size_t budget = size_t(12) << 30;
    uint64_t B = std::max<uint64_t>(1, std::min<uint64_t>(n, std::max<size_t>(1, budget / per_view)));
    B = std::min<uint64_t>(B, 64);
    if (mode == Mode::Render) B = 1;

    const size_t NS = std::max<uint64_t>(N, 1);
    CK(ctx->poses.reserve(sizeof(PoseParams) * B));
    CK(ctx->vcount.reserve(4 * B));
    CK(ctx->pcount.reserve(16 * B));  // pairs P | row pairs R per view
    CK(ctx->bdiff.reserve(sizeof(int) * (o.tiles_x + 1) * (o.tiles_y + 1)));
    CK(ctx->rranges.reserve(sizeof(uint2) * o.tiles_y));
    CK(ctx->keys.reserve(4 * NS * B));
    CK(ctx->vals.reserve(4 * NS * B));
    CK(ctx->keys_alt.reserve(4 * NS));
    CK(ctx->rects.reserve(sizeof(int4) * NS));
    CK(ctx->vals_alt.reserve(4 * NS));
    CK(ctx->packed.reserve(sizeof(PackedSplat) * NS * B));
    CK(ctx->bounds.reserve(sizeof(uint4) * NS * B));
    CK(ctx->counts.reserve(8 * (NS + 1)));
    CK(ctx->offsets.reserve(8 * (NS + 1)));
    CK(ctx->ranges.reserve(sizeof(uint2) * bin_tiles * B));
    CK(ctx->ent_part.reserve(8ull * rtiles * B));
    CK(ctx->miss_part.reserve(4ull * rtiles * B));
    CK(ctx->views.reserve(sizeof(ViewDesc) * B));
    CK(ctx->out.reserve(24 * B));
    if (fk == Fisher::Gain) {
        CK(ctx->fis_part.reserve(8ull * rtiles * B));
        // rendered colour / depth per view for the gain's Jacobian pass (written by the
        // score raster, so k_fisher skips its own pass 0)
        CK(ctx->rcbuf.reserve(32ull * cam.W * cam.H * B));
    }
    CK(ctx->contributors.reserve(8));
    CK(ctx->h_counts.reserve(32 * B + 16));  // V (u32) | P | R | contributors
    CK(ctx->h_views.reserve(sizeof(ViewDesc) * B));
    CK(ctx->h_poses.reserve(sizeof(PoseParams) * B));
    CK(ctx->h_out.reserve(24 * B));

    const int kSub = 8;  // views per raster launch (binning of the next 8 overlaps)
    for (uint64_t b0 = 0; b0 < n; b0 += B) {
        const int nb = static_cast<int>(std::min<uint64_t>(B, n - b0));
        if (ctx->profiling) CK(cudaEventRecord(ctx->ev[0], s));
        std::memcpy(ctx->h_poses.p, poses + b0, sizeof(PoseParams) * nb);
        CK(cudaMemcpyAsync(ctx->poses.p, ctx->h_poses.p, sizeof(PoseParams) * nb,
                           cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(ctx->vcount.p, 0, 4 * nb, s));
        CK(cudaMemsetAsync(ctx->pcount.p, 0, 16 * nb, s));
        CK(cudaMemsetAsync(ctx->contributors.p, 0, 8, s));
        launch_preprocess(map->dev, ctx->poses.as<PoseParams>(), cam, o, nb, ctx->keys.as<uint32_t>(),
                          ctx->vals.as<uint32_t>(), NS, ctx->vcount.as<uint32_t>(),
                          ctx->pcount.as<unsigned long long>(),
                          ctx->pcount.as<unsigned long long>() + nb, s);
        ctx->stats.kernel_launches += (N > 0) ? 1 : 0;
        uint32_t* hv = ctx->h_counts.as<uint32_t>();
        unsigned long long* hp = reinterpret_cast<unsigned long long*>(ctx->h_counts.as<char>() + 8 * B);
        CK(cudaMemcpyAsync(hv, ctx->vcount.p, 4 * nb, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hp, ctx->pcount.p, 16 * nb, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<uint32_t> V(hv, hv + nb);
        std::vector<uint64_t> P(hp, hp + nb);
        std::vector<uint64_t> R(hp + nb, hp + 2 * nb);  // (row, rank) pairs of the binning
        for (int v = 0; v < nb; ++v)
            if (P[v] >= (1ull << 32)) fail(SGM_ERR_UNSUPPORTED, "view has %llu tile pairs (>= 2^32)",
                                          static_cast<unsigned long long>(P[v]));

        // groups of views whose pair lists fit the budget together
        const uint64_t pair_budget = (uint64_t(8) << 30) / 4;  // u32 list entries
        int v0 = 0;
        while (v0 < nb) {
            int v1 = v0;
            uint64_t sumP = 0, maxP = 0;
            while (v1 < nb && (v1 == v0 || sumP + P[v1] <= pair_budget)) {
                sumP += P[v1];
                maxP = std::max<uint64_t>(maxP, P[v1]);
                ++v1;
            }
            uint64_t maxR = 1;
            for (int v = v0; v < v1; ++v) maxR = std::max<uint64_t>(maxR, R[v]);
            CK(ctx->tvals.reserve(4 * std::max<uint64_t>(sumP, 1)));
            CK(ctx->tkeys.reserve(4 * maxR));
            CK(ctx->tkeys_alt.reserve(4 * maxR));
            CK(ctx->tvals_alt.reserve(8 * maxR));
            CK(ctx->rvals.reserve(8 * maxR));
            // row-scatter segments of the largest view (reserved here, not between the
            // views' binning launches: a reallocation would synchronise the device)
            const uint64_t maxG = row_scatter_segments(maxR, o.tiles_y);
            CK(ctx->segs.reserve(sizeof(uint4) * maxG + 16));
            CK(ctx->segcnt.reserve(sizeof(uint32_t) * maxG * o.tiles_x));
            // descriptors for the whole group (list offsets known from the counts)
            ViewDesc* hvd = ctx->h_views.as<ViewDesc>();
            uint64_t list_off = 0;
            for (int v = v0; v < v1; ++v) {
                ViewDesc d{};
                d.order = ctx->vals.as<uint32_t>() + NS * v;
                d.pose = ctx->poses.as<PoseParams>() + v;
                d.fis_partial = fk == Fisher::Gain ? ctx->fis_part.as<double>() + static_cast<size_t>(rtiles) * v
                                                   : nullptr;
                d.ranges = ctx->ranges.as<uint2>() + static_cast<size_t>(bin_tiles) * v;
                d.list = ctx->tvals.as<uint32_t>() + list_off;
                d.packed = ctx->packed.as<PackedSplat>() + NS * v;
                d.bounds = ctx->bounds.as<uint4>() + NS * v;
                d.ent_partial = ctx->ent_part.as<double>() + static_cast<size_t>(rtiles) * v;
                d.miss_partial = ctx->miss_part.as<uint32_t>() + static_cast<size_t>(rtiles) * v;
                d.color = rt.color;
                d.depth = rt.depth;
                d.sil = rt.sil;
                d.sem = rt.sem;
                d.contributors = ctx->contributors.as<unsigned long long>();
                d.contrib = rt.contrib;
                d.contrib_count = rt.contrib_count;
                d.contrib_offset = rt.contrib_offset;
                d.rc4 = fk == Fisher::Gain
                            ? ctx->rcbuf.as<double>() + 4ull * cam.W * cam.H * static_cast<size_t>(v)
                            : nullptr;
                hvd[v - v0] = d;
                list_off += P[v];
                ctx->stats.visible += V[v];
                ctx->stats.pairs += P[v];
            }
            const int ngroup = v1 - v0;
            CK(cudaMemcpyAsync(ctx->views.p, hvd, sizeof(ViewDesc) * ngroup, cudaMemcpyHostToDevice, s));
            // the binning stream starts after everything already queued on s
            CK(cudaEventRecord(ctx->ev_ready, s));
            CK(cudaStreamWaitEvent(sb, ctx->ev_ready, 0));
            RasterParams rp{};
            rp.map = map->dev;
            rp.cam = cam;
            rp.opt = o;
            rp.tiles_per_view = rtiles;
            rp.raster_tiles_x = rtx;
            rp.channels = rt.channels;
            rp.groups = map->groups;
            rp.want_rc = fk == Fisher::Gain ? 1 : 0;
            for (int s0 = v0; s0 < v1; s0 += kSub) {
                const int s1 = std::min(v1, s0 + kSub);
                for (int v = s0; v < s1; ++v) {
                    const ViewDesc& d = hvd[v - v0];
                    bin_view(ctx, sb, map, cam, o, ctx->poses.as<PoseParams>() + v,
                             ctx->keys.as<uint32_t>() + NS * v, const_cast<uint32_t*>(d.order), V[v],
                             P[v], R[v], const_cast<PackedSplat*>(d.packed), const_cast<uint4*>(d.bounds),
                             const_cast<uint32_t*>(d.list), const_cast<uint2*>(d.ranges), bin_tiles);
                }
                const int slot = (s0 / kSub) & 1;
                CK(cudaEventRecord(ctx->ev_binned[slot], sb));
                CK(cudaStreamWaitEvent(s, ctx->ev_binned[slot], 0));
                rp.views = ctx->views.as<ViewDesc>() + (s0 - v0);
                const int pr = ((s0 - v0) / kSub) % 8;  // profiling event pair
                if (ctx->profiling) CK(cudaEventRecord(ctx->ev_r[2 * pr], s));
                FisherParams fp{};
                fp.H = d_H;
                fp.invp = map->fisher_invp.as<double>();
                if (fk == Fisher::Prior) {
                    launch_fisher_prior(rp, fp, s1 - s0, s);
                } else {
                    if (mode == Mode::Score)
                        launch_raster_score(rp, s1 - s0, s);
                    else
                        launch_raster_render(rp, s1 - s0, s);
                    if (fk == Fisher::Gain) {
                        launch_fisher_gain(rp, fp, s1 - s0, s);
                        ctx->stats.kernel_launches += 1;
                    }
                }
                CK(cudaGetLastError());
                if (ctx->profiling) CK(cudaEventRecord(ctx->ev_r[2 * pr + 1], s));
                ctx->stats.kernel_launches += 1;
                ctx->stats.raster_launches += 1;
            }
            if (mode == Mode::Score && fk != Fisher::Prior) {
                double* dfis = fk == Fisher::Gain ? ctx->out.as<double>() + 2 * ngroup : nullptr;
                launch_reduce_scores(ctx->views.as<ViewDesc>(), ngroup, rtiles, ctx->out.as<double>(),
                                     ctx->out.as<double>() + ngroup, dfis, s);
                ctx->stats.kernel_launches += 1;
                double* ho = ctx->h_out.as<double>();
                CK(cudaMemcpyAsync(ho, ctx->out.p, 24 * ngroup, cudaMemcpyDeviceToHost, s));
                unsigned long long* kc = hp + 2 * B;
                CK(cudaMemcpyAsync(kc, ctx->contributors.p, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaMemsetAsync(ctx->contributors.p, 0, 8, s));
                CK(cudaStreamSynchronize(s));
                for (int v = 0; v < ngroup; ++v) {
                    h_missing[b0 + v0 + v] = ho[v];
                    h_entropy[b0 + v0 + v] = ho[ngroup + v];
                    if (h_fisher) h_fisher[b0 + v0 + v] = ho[2 * ngroup + v];
                }
                ctx->stats.contributors += *kc;
            } else {
                unsigned long long* kc = hp + 2 * B;
                CK(cudaMemcpyAsync(kc, ctx->contributors.p, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaMemsetAsync(ctx->contributors.p, 0, 8, s));
                CK(cudaStreamSynchronize(s));
                ctx->stats.contributors += *kc;
            }
            if (ctx->profiling) {
                const int nsub = std::min(8, (ngroup + kSub - 1) / kSub);
                for (int q = 0; q < nsub; ++q) {
                    float ms = 0;
                    CK(cudaEventElapsedTime(&ms, ctx->ev_r[2 * q], ctx->ev_r[2 * q + 1]));
                    ctx->stats.raster_ms += ms;
                }
            }
            v0 = v1;
        }
        if (ctx->profiling) {
            CK(cudaEventRecord(ctx->ev[3], s));
            CK(cudaEventSynchronize(ctx->ev[3]));
            float total = 0;
            CK(cudaEventElapsedTime(&total, ctx->ev[0], ctx->ev[3]));
            ctx->stats.binning_ms += total;  // whole-batch span; raster share in raster_ms
        }
        ctx->stats.views += nb;
        if (mode == Mode::Render) {
            ctx->last_valid = true;
            ctx->last_V = V[0];
            ctx->last_P = P[0];
            ctx->last_bin_tiles = bin_tiles;
            ctx->last_map = map;
            ctx->last_cam = cam;
            ctx->last_opt = o;
            ctx->last_pose = poses[0];
        }
    }
}

int guard(sgm_ctx* ctx, const std::function<void()>& fn) {
    try {
        fn();
        if (ctx) ctx->err.clear();
        return SGM_OK;
    } catch (const SgmError& e) {
        if (ctx) ctx->err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        if (ctx) ctx->err = "host allocation failed";
        return SGM_ERR_OOM;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return SGM_ERR_INVALID;
    }
}

void need_ctx(sgm_ctx* ctx) {
    if (!ctx) fail(SGM_ERR_INVALID, "ctx is null");
    CK(cudaSetDevice(ctx->device));
}

void do_render(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera, const sgm_pose* pose,
               uint32_t channels, const sgm_options* opt, double* d_color, double* d_depth,
               double* d_sil, double* d_sem, uint64_t* n_proj) {
    need_ctx(ctx);
    if (!map) fail(SGM_ERR_INVALID, "map is null");
    if (!pose) fail(SGM_ERR_INVALID, "pose is null");
    const CamParams cam = to_cam(camera);
    const OptParams o = to_opt(opt, cam);
    const PoseParams p = to_pose(*pose);
    RenderTargets rt;
    rt.channels = channels;
    rt.color = (channels & SGM_COLOR) ? d_color : nullptr;
    rt.depth = (channels & SGM_DEPTH) ? d_depth : nullptr;
    rt.sem = (channels & SGM_SEMANTICS) ? d_sem : nullptr;
    rt.sil = d_sil;
    ctx->last_has_contrib = false;
    if (channels & SGM_RETAIN_CONTRIBUTORS) {
        // pass 1: per-pixel contributor counts (splat_render.cpp:215-216, 310)
        const size_t px = static_cast<size_t>(cam.W) * cam.H;
        CK(ctx->ccount.reserve(4 * (px + 1)));
        CK(ctx->coffset.reserve(8 * (px + 1)));
        CK(ctx->contrib.reserve(4));
        CK(cudaMemsetAsync(ctx->ccount.p, 0, 4 * (px + 1), ctx->stream));
        rt.contrib = ctx->contrib.as<uint32_t>();
        rt.contrib_count = ctx->ccount.as<uint32_t>();
        run_views(ctx, map, cam, o, 1, &p, Mode::Render, rt, nullptr, nullptr);
        // offsets = exclusive scan (flatten_contributors, :125-137)
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, ctx->ccount.as<uint32_t>(),
                                         ctx->coffset.as<unsigned long long>(), px + 1, ctx->stream));
        CK(ctx->cub_tmp.reserve(tmp));
        CK(cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, tmp, ctx->ccount.as<uint32_t>(),
                                         ctx->coffset.as<unsigned long long>(), px + 1, ctx->stream));
        ctx->stats.kernel_launches += 1;
        unsigned long long total = 0;
        CK(cudaMemcpyAsync(&total, ctx->coffset.as<unsigned long long>() + px, 8,
                           cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (total >= (1ull << 32)) fail(SGM_ERR_UNSUPPORTED, "more than 2^32 contributors");
        CK(ctx->contrib.reserve(4 * std::max<unsigned long long>(total, 1)));
        // pass 2: write the depth-ordered contributor ranks
        rt.contrib = ctx->contrib.as<uint32_t>();
        rt.contrib_offset = ctx->coffset.as<unsigned long long>();
        run_views(ctx, map, cam, o, 1, &p, Mode::Render, rt, nullptr, nullptr);
        ctx->last_ncontrib = total;
        ctx->last_has_contrib = true;
        ctx->last_px = static_cast<int>(px);
    } else {
        run_views(ctx, map, cam, o, 1, &p, Mode::Render, rt, nullptr, nullptr);
    }
    if (n_proj) *n_proj = ctx->last_V;
}

}  // namespace

namespace {

// The mapping step on device-resident frame planes: render(all(true)) with contributor
// counts, mapping_loss + semantic_loss, backward, projection->world chain, KL clip and the
// finiteness check (losses.cpp:40-362). Gradients stay in ctx->bw_grad:
//   center 3NS | log_radius NS | opacity_logit NS | color 3NS | sem k*NS | proj 5NS
// (NS = max(N, 1)); report = LossReport fields. Throws like the reference on a non-finite
// gradient.
void backward_core(sgm_ctx* ctx, const sgm_map* map, const CamParams& cam, const OptParams& o,
                   const PoseParams& p, const float* f_rgb, const float* f_depth,
                   const float* f_sem, const double weights[7], int include_mapping,
                   int include_semantic, double report[7]) {
    cudaStream_t s = ctx->stream;
    const size_t px = static_cast<size_t>(cam.W) * cam.H;
    const int C = map->dev.C, k = map->dev.k;
    const uint64_t N = map->dev.n;
    const size_t NS = std::max<uint64_t>(N, 1);
    // device planes: rendered (sil, color, depth, sem) + frame (rgb, depth, sem)
    const size_t rend_b = 8 * px * (5 + C);
    CK(ctx->planes.reserve(rend_b));
    CK(ctx->ccount.reserve(4 * (px + 1)));
    CK(ctx->contrib.reserve(4));
    CK(ctx->bw_flags.reserve(px + 16));
    const size_t nlb = backward_loss_blocks(cam.W, cam.H);
    CK(ctx->bw_part.reserve(64 * nlb + 64 + 64));
    CK(ctx->bw_grad.reserve(8 * (NS * (8 + k) + 5 * NS) + 64));
    double* d_sil = ctx->planes.as<double>();
    double* d_color = d_sil + px;
    double* d_depth = d_color + 3 * px;
    double* d_sem = d_depth + px;
    CK(cudaMemsetAsync(ctx->ccount.p, 0, 4 * (px + 1), s));
    // 1. forward render + contributor counts (the reference's render(..., all(true)))
    RenderTargets rt;
    rt.channels = SGM_COLOR | SGM_DEPTH | SGM_SEMANTICS;
    rt.color = d_color;
    rt.depth = d_depth;
    rt.sil = d_sil;
    rt.sem = d_sem;
    rt.contrib = ctx->contrib.as<uint32_t>();
    rt.contrib_count = ctx->ccount.as<uint32_t>();
    run_views(ctx, map, cam, o, 1, &p, Mode::Render, rt, nullptr, nullptr);
    const uint32_t V = ctx->last_V;
    // 2. loss masks, reports and mask counts
    double* g = ctx->bw_grad.as<double>();
    BackwardParams b{};
    b.W = cam.W;
    b.H = cam.H;
    b.C = C;
    b.color = d_color;
    b.depth = d_depth;
    b.sil = d_sil;
    b.sem = d_sem;
    b.ccount = ctx->ccount.as<uint32_t>();
    b.rgb = f_rgb;
    b.fdepth = f_depth;
    b.fsem = f_sem;
    b.flags = ctx->bw_flags.as<uint8_t>();
    b.tau = std::log(weights[2]);
    b.lambda_hd = weights[0];
    b.lambda_cos = weights[1];
    b.use_hd = weights[3] != 0.0;
    b.use_cos = weights[4] != 0.0;
    b.use_kl = weights[5] != 0.0;
    b.include_mapping = include_mapping != 0;
    b.include_semantic = include_semantic != 0;
    double* totals = ctx->bw_part.as<double>() + 8 * nlb;
    b.totals = totals;
    b.gcenter = g;
    b.glogr = g + 3 * NS;
    b.glogit = g + 4 * NS;
    b.gcolor = g + 5 * NS;
    b.gsem = g + 8 * NS;
    b.gproj = g + (8 + k) * NS;
    b.sem_perm = map->dev.sem_perm;
    CK(cudaMemsetAsync(g, 0, 8 * (NS * (8 + k) + 5 * NS), s));
    launch_loss_pixels(b, ctx->bw_part.as<double>(), totals, s);
    // 3. backward over the block lists of the render above (same binning)
    RasterParams rp{};
    rp.map = map->dev;
    rp.cam = cam;
    rp.opt = o;
    rp.views = ctx->views.as<ViewDesc>();
    rp.tiles_per_view = ((cam.W + kTile - 1) / kTile) * ((cam.H + kTile - 1) / kTile);
    rp.raster_tiles_x = (cam.W + kTile - 1) / kTile;
    rp.channels = rt.channels;
    rp.groups = map->groups;
    launch_backward(rp, b, s);
    // 4. projection -> world, KL clipping, finiteness
    launch_chain(map->dev, ctx->poses.as<PoseParams>(), cam, o, ctx->vals.as<uint32_t>(), V,
                 b.gproj, b, s);
    if (b.use_kl && b.include_semantic && weights[6] > 0.0)
        launch_kl_clip(b.gsem, N, k, weights[6], s);
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(totals + 8);
    CK(cudaMemsetAsync(bad, 0xff, 5 * 8, s));
    const double* arrs[5] = {b.gcenter, b.glogr, b.glogit, b.gcolor, b.gsem};
    const uint64_t lens[5] = {3 * N, N, N, 3 * N, static_cast<uint64_t>(k) * N};
    for (int a = 0; a < 5; ++a) launch_finite(arrs[a], lens[a], bad + a, s);
    ctx->stats.kernel_launches += 4 + 5;
    CK(cudaGetLastError());
    double h_tot[8];
    unsigned long long h_bad[5];
    CK(cudaMemcpyAsync(h_tot, totals, 64, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h_bad, bad, 40, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    static const char* names[5] = {"center", "log_radius", "opacity_logit", "color", "sem"};
    static const uint64_t stride[5] = {3, 1, 1, 3, 0};
    for (int a = 0; a < 5; ++a)
        if (h_bad[a] != ~0ull)  // losses.cpp:349-360
            fail(SGM_ERR_INVALID, "backward: non-finite gradient for gaussian %llu parameter %s",
                 static_cast<unsigned long long>(h_bad[a] / (a == 4 ? k : stride[a])), names[a]);
    report[0] = h_tot[3] > 0 ? h_tot[0] / h_tot[3] : 0.0;  // photometric (:57)
    report[1] = h_tot[4] > 0 ? h_tot[1] / h_tot[4] : 0.0;  // depth (:58)
    report[2] = h_tot[5] > 0 ? h_tot[2] / h_tot[5] : 0.0;  // semantic (:158)
    report[3] = h_tot[3];
    report[4] = h_tot[4];
    report[5] = h_tot[5];
    report[6] = h_tot[6];
}

}  // namespace

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
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->bin_stream) cudaStreamSynchronize(ctx->bin_stream);
    for (auto& ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
    for (auto& ev : ctx->ev_binned)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev_r)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev_ring)
        if (ev) cudaEventDestroy(ev);
    cudaStream_t s = ctx->stream, s2 = ctx->bin_stream;
    delete ctx;
    if (s) cudaStreamDestroy(s);
    if (s2) cudaStreamDestroy(s2);
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

int sgm_map_upload(sgm_ctx* ctx, uint64_t n, int32_t k, int32_t num_classes, const double* centers,
                   const double* log_radii, const double* opacity_logits, const double* colors,
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
        const int C = num_classes + 1;
        const int kpad = (k + 7) / 8 * 8;
        m = new sgm_map();
        m->num_classes = num_classes;
        const size_t ns = std::max<uint64_t>(n, 1);
        // pinned staging: geo SoA (5 ns), colour (4 ns), raw rows (k ns u16 + k ns f64)
        const size_t geo_b = 8 * 5 * ns, col_b = 8 * 4 * ns, idx_b = 2 * static_cast<size_t>(k) * ns,
                     prob_b = 8 * static_cast<size_t>(k) * ns;
        CK(ctx->h_stage.reserve(geo_b + col_b + prob_b + idx_b + 64));
        char* hs = ctx->h_stage.as<char>();
        double* geo = reinterpret_cast<double*>(hs);
        double* col = reinterpret_cast<double*>(hs + geo_b);
        double* rprob = reinterpret_cast<double*>(hs + geo_b + col_b);
        uint16_t* ridx = reinterpret_cast<uint16_t*>(hs + geo_b + col_b + prob_b);
        // Host side (reference libm, gaussian_map.hpp:36-37) in kChunks chunks over a pool of
        // threads; as soon as every thread has finished chunk c, its slices go to the GPU
        // (async H2D), so the copies overlap the host work on the next chunks.
        const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        const unsigned nth = n > 65536 ? hw : 1;
        const unsigned kChunks = n > 65536 ? 8 : 1;
        std::vector<int> bad(nth, -1), dup(nth, 0);
        std::unique_ptr<std::atomic<unsigned>[]> finished(new std::atomic<unsigned>[kChunks]);
        for (unsigned c = 0; c < kChunks; ++c) finished[c].store(0);
        auto work = [&](unsigned w) {
            std::vector<uint32_t> seen(static_cast<size_t>(C), 0xffffffffu);
            for (unsigned c = 0; c < kChunks; ++c) {
                const uint64_t ca = n * c / kChunks, cb = n * (c + 1) / kChunks;
                const uint64_t a = ca + (cb - ca) * w / nth, b = ca + (cb - ca) * (w + 1) / nth;
                for (uint64_t i = a; i < b; ++i) {
                    geo[i] = centers[3 * i];
                    geo[ns + i] = centers[3 * i + 1];
                    geo[2 * ns + i] = centers[3 * i + 2];
                    geo[3 * ns + i] = std::exp(log_radii[i]);                      // radius()
                    geo[4 * ns + i] = 1.0 / (1.0 + std::exp(-opacity_logits[i]));  // sigmoid
                    for (int q = 0; q < 3; ++q) col[4 * i + q] = std::clamp(colors[3 * i + q], 0.0, 1.0);
                    col[4 * i + 3] = 0.0;
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
                finished[c].fetch_add(1, std::memory_order_release);
            }
        };
        cudaStream_t s = ctx->stream;
        ctx->take(m->geo, geo_b);
        ctx->take(m->color, col_b);
        ctx->take(m->idx, 2 * ns * kpad);
        ctx->take(m->prob, 8 * ns * kpad);
        ctx->take(m->perm, 2 * ns * kpad);
        CK(m->geo.reserve(geo_b));
        CK(m->color.reserve(col_b));
        CK(m->idx.reserve(2 * ns * kpad));
        CK(m->prob.reserve(8 * ns * kpad));
        CK(m->perm.reserve(2 * ns * kpad));
        CK(ctx->upload_tmp.reserve(idx_b + prob_b + 64));
        char* draw = ctx->upload_tmp.as<char>();
        std::vector<std::thread> pool;
        for (unsigned w = 1; w < nth; ++w) pool.emplace_back(work, w);
        std::thread self(work, 0u);
        cudaError_t copy_err = cudaSuccess;
        for (unsigned c = 0; c < kChunks; ++c) {
            while (finished[c].load(std::memory_order_acquire) < nth) std::this_thread::yield();
            const uint64_t ca = n * c / kChunks, cb = n * (c + 1) / kChunks;
            if (cb == ca) continue;
            for (int f = 0; f < 5 && copy_err == cudaSuccess; ++f)
                copy_err = cudaMemcpyAsync(m->geo.as<double>() + f * ns + ca, geo + f * ns + ca,
                                           8 * (cb - ca), cudaMemcpyHostToDevice, s);
            if (copy_err == cudaSuccess)
                copy_err = cudaMemcpyAsync(m->color.as<double>() + 4 * ca, col + 4 * ca, 32 * (cb - ca),
                                           cudaMemcpyHostToDevice, s);
            if (copy_err == cudaSuccess)
                copy_err = cudaMemcpyAsync(draw + 8 * k * ca, rprob + k * ca, 8 * k * (cb - ca),
                                           cudaMemcpyHostToDevice, s);
            if (copy_err == cudaSuccess)
                copy_err = cudaMemcpyAsync(draw + prob_b + 2 * k * ca, ridx + k * ca, 2 * k * (cb - ca),
                                           cudaMemcpyHostToDevice, s);
        }
        self.join();
        for (auto& th : pool) th.join();
        CK(copy_err);
        for (unsigned w = 0; w < nth; ++w)
            if (bad[w] >= 0) {
                cudaStreamSynchronize(s);  // the in-flight copies target this map's buffers
                fail(SGM_ERR_INVALID, "map: semantic index >= channels %d (near gaussian %d)", C, bad[w]);
            }
        int has_dup = 0;
        for (unsigned w = 0; w < nth; ++w) has_dup |= dup[w];
        // rows sorted by class id (stable) and padded to kpad, on the GPU
        launch_sort_rows(reinterpret_cast<const uint16_t*>(draw + prob_b),
                         reinterpret_cast<const double*>(draw), n, k, kpad, m->idx.as<uint16_t>(),
                         m->prob.as<double>(), m->perm.as<uint16_t>(), s);
        ctx->stats.kernel_launches += n ? 1 : 0;
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
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
        d.dup_idx = has_dup;
        m->groups = choose_groups(C, k);
        *out = m;
        m = nullptr;
    });
    delete m;
    return rc;
}

void sgm_map_release(sgm_ctx* ctx, sgm_map* map) {
    if (!map) return;
    if (ctx) {
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->bin_stream);
        if (ctx->last_map == map) ctx->last_valid = false;
        ctx->give(std::move(map->geo));
        ctx->give(std::move(map->color));
        ctx->give(std::move(map->idx));
        ctx->give(std::move(map->prob));
        ctx->give(std::move(map->perm));
        ctx->give(std::move(map->cov));
    }
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

namespace {

struct CopyOut {
    void* dst;        // host (pageable) destination
    const void* src;  // device source
    size_t bytes;
};

// Device -> pageable host copies of large planes (a full render is px (5 + C) doubles:
// 698 MB at cfg1). A plain cudaMemcpy to pageable memory is staged by the driver at about
// 15 GB/s and pays the fresh pages' faults serially; here the planes go through a ring of
// pinned buffers in kChunk pieces (DMA at full PCIe rate) while a pool of host threads
// copies the finished pieces out in parallel.
void copy_out(sgm_ctx* ctx, const std::vector<CopyOut>& segs) {
    constexpr size_t kChunk = size_t(16) << 20;
    constexpr int kSlots = 4;
    cudaStream_t s = ctx->stream;
    size_t total = 0;
    for (const auto& g : segs) total += g.bytes;
    if (total <= 2 * kChunk) {  // small: direct copies
        for (const auto& g : segs)
            CK(cudaMemcpyAsync(g.dst, g.src, g.bytes, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return;
    }
    struct Piece {
        char* dst;
        const char* src;
        size_t bytes;
    };
    std::vector<Piece> pieces;
    for (const auto& g : segs)
        for (size_t o = 0; o < g.bytes; o += kChunk)
            pieces.push_back({static_cast<char*>(g.dst) + o, static_cast<const char*>(g.src) + o,
                              std::min(kChunk, g.bytes - o)});
    CK(ctx->h_ring.reserve(kSlots * kChunk));
    for (int k = 0; k < kSlots; ++k)
        if (!ctx->ev_ring[k]) CK(cudaEventCreateWithFlags(&ctx->ev_ring[k], cudaEventDisableTiming));
    const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const size_t np = pieces.size();
    std::unique_ptr<std::atomic<unsigned>[]> copied(new std::atomic<unsigned>[np]);
    for (size_t j = 0; j < np; ++j) copied[j].store(0);
    std::atomic<size_t> issued{0};  // pieces whose D2H + event are enqueued
    std::atomic<int> err{0};
    auto worker = [&](unsigned w) {
        for (size_t j = 0; j < np; ++j) {
            while (issued.load(std::memory_order_acquire) <= j && !err.load()) std::this_thread::yield();
            if (err.load()) return;
            const int slot = static_cast<int>(j % kSlots);
            if (cudaEventSynchronize(ctx->ev_ring[slot]) != cudaSuccess) err.store(1);
            const Piece& pc = pieces[j];
            const size_t a = pc.bytes * w / nth, b = pc.bytes * (w + 1) / nth;
            std::memcpy(pc.dst + a, ctx->h_ring.as<char>() + slot * kChunk + a, b - a);
            copied[j].fetch_add(1, std::memory_order_release);
        }
    };
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nth; ++w) pool.emplace_back(worker, w);
    cudaError_t e = cudaSuccess;
    for (size_t j = 0; j < np && e == cudaSuccess; ++j) {
        const int slot = static_cast<int>(j % kSlots);
        if (j >= kSlots)  // the slot's previous piece must be copied out first
            while (copied[j - kSlots].load(std::memory_order_acquire) < nth && !err.load())
                std::this_thread::yield();
        e = cudaMemcpyAsync(ctx->h_ring.as<char>() + slot * kChunk, pieces[j].src, pieces[j].bytes,
                            cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_ring[slot], s);
        issued.store(j + 1, std::memory_order_release);
    }
    if (e != cudaSuccess) err.store(1);
    for (auto& th : pool) th.join();
    CK(e);
    if (err.load()) fail(SGM_ERR_CUDA, "device-to-host copy failed");
    CK(cudaStreamSynchronize(s));
}

}  // namespace

int sgm_render(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera, const sgm_pose* pose,
               uint32_t channels, const sgm_options* opt, double* color, double* depth,
               double* silhouette, double* sem, uint64_t* n_projections) {
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
        do_render(ctx, map, camera, pose, ch, opt, d_color, d_depth, d_sil, d_sem, n_projections);
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
